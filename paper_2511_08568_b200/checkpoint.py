"""Model checkpoints (neural/checkpoint.py of the reference): the same .npz
container, header and errors, so checkpoints move between the two packages
unchanged, plus a shard reader for vocabularies too large to load whole.

Container (checkpoint.py:1-8, 27-45): a numpy .npz archive whose reserved
``__meta__`` entry is a JSON header (format tag, hyperparameters, table
sizes, sha256 of the vocabulary, array shapes); loading for a different
vocabulary raises VocabularyMismatchError (checkpoint.py:66-76).
"""
from __future__ import annotations

import hashlib
import json
import os
import zipfile

import numpy as np

from .errors import CheckpointError, MissingArtifactError, VocabularyMismatchError
from .model import ModelParameters

_META_KEY = "__meta__"
_FORMAT = "embcache-checkpoint-v1"


def vocabulary_hash(table_sizes) -> str:
    """checkpoint.py:22-24."""
    text = ",".join(str(int(s)) for s in table_sizes)
    return hashlib.sha256(text.encode("utf-8")).hexdigest()


def save_checkpoint(params: ModelParameters, path: str):
    """checkpoint.py:27-45 (np.savez: members stored, so shards can be read
    row-range by row-range)."""
    meta = {
        "format": _FORMAT,
        "kind": params.kind,
        "dim": params.dim,
        "stacks": params.stacks,
        "l_in": params.l_in,
        "l_out": params.l_out,
        "table_sizes": [int(s) for s in params.table_sizes],
        "vocab_hash": vocabulary_hash(params.table_sizes),
        "arrays": {name: list(a.shape) for name, a in params.arrays.items()},
    }
    payload = {name: a for name, a in params.arrays.items()}
    payload[_META_KEY] = np.array(json.dumps(meta))
    with open(path, "wb") as f:
        np.savez(f, **payload)


def _read_meta(archive, path):
    if _META_KEY not in archive:
        raise CheckpointError(f"{path!r} has no header entry")
    try:
        return json.loads(str(archive[_META_KEY]))
    except json.JSONDecodeError as e:
        raise CheckpointError(f"{path!r} header is not valid JSON: {e}")


def _check_meta(meta, shapes, path, table_sizes):
    """checkpoint.py:62-76: format, declared shapes, vocabulary hash."""
    if meta.get("format") != _FORMAT:
        raise CheckpointError(f"{path!r} has unknown format {meta.get('format')!r}")
    for name, shape in meta.get("arrays", {}).items():
        if name not in shapes or list(shapes[name]) != shape:
            raise CheckpointError(f"{path!r} array {name!r} missing or misshaped")
    stored = meta.get("table_sizes")
    if stored is None or meta.get("vocab_hash") != vocabulary_hash(stored):
        raise CheckpointError(f"{path!r} vocabulary hash does not match header")
    if table_sizes is not None and vocabulary_hash(table_sizes) != meta["vocab_hash"]:
        raise VocabularyMismatchError(
            f"checkpoint vocabulary {stored} does not match expected {list(table_sizes)}")
    return stored


def load_checkpoint(path: str, table_sizes=None) -> ModelParameters:
    """checkpoint.py:48-79, same checks in the same order and the same errors."""
    if not os.path.exists(path):
        raise MissingArtifactError(f"checkpoint {path!r} does not exist")
    try:
        with np.load(path, allow_pickle=False) as archive:
            meta = _read_meta(archive, path)
            arrays = {name: archive[name] for name in archive.files if name != _META_KEY}
    except (zipfile.BadZipFile, OSError, ValueError) as e:
        raise CheckpointError(f"{path!r} is not a readable checkpoint: {e}")
    stored = _check_meta(meta, {k: v.shape for k, v in arrays.items()}, path, table_sizes)
    return ModelParameters(meta["kind"], stored, meta["dim"], meta["stacks"], meta["l_in"],
                           meta["l_out"], arrays)


def load_checkpoint_shard(path: str, shard, table_sizes=None, device=True):
    """A table shard of a checkpoint: the dense arrays whole,
    embed_table's rows of the shard's tables, and only the shard's embed_id
    rows -- read row-range by row-range from the stored .npz member, never
    the whole [V, d] float64 array (43.8 GB at config 3).  Returns what
    shard.init_params_shard returns: (ModelParameters over the shard's local
    vocabulary without "embed_id", the local embed_id rows as fp32 on the
    GPU when device else numpy)."""
    from .shard import TableShard
    if not os.path.exists(path):
        raise MissingArtifactError(f"checkpoint {path!r} does not exist")
    try:
        zf = zipfile.ZipFile(path)
    except (zipfile.BadZipFile, OSError) as e:
        raise CheckpointError(f"{path!r} is not a readable checkpoint: {e}")
    with zf:
        try:
            with np.load(path, allow_pickle=False) as archive:
                meta = _read_meta(archive, path)
                names = [n for n in archive.files if n != _META_KEY]
                dense = {n: archive[n] for n in names if n != "embed_id"}
            shapes = {n: v.shape for n, v in dense.items()}
            with zf.open("embed_id.npy") as f:
                version = np.lib.format.read_magic(f)
                if version == (1, 0):
                    shape, fortran, dtype = np.lib.format.read_array_header_1_0(f)
                else:
                    shape, fortran, dtype = np.lib.format.read_array_header_2_0(f)
                shapes["embed_id"] = shape
                stored = _check_meta(meta, shapes, path, table_sizes)
                sh = shard if isinstance(shard, TableShard) else TableShard(stored, shard)
                if list(sh.table_sizes) != list(stored):
                    raise VocabularyMismatchError("shard layout does not match the checkpoint")
                if fortran or len(shape) != 2:
                    raise CheckpointError(f"{path!r} embed_id is not a C-order matrix")
                d = int(shape[1])
                emb = _read_rows(f, dtype, d, sh, device)
        except KeyError as e:
            raise CheckpointError(f"{path!r} array {e} missing or misshaped")
        except (zipfile.BadZipFile, OSError, ValueError) as e:
            raise CheckpointError(f"{path!r} is not a readable checkpoint: {e}")
    dense["embed_table"] = np.ascontiguousarray(dense["embed_table"][sh.tables])
    return ModelParameters(meta["kind"], list(sh.local_sizes), meta["dim"], meta["stacks"],
                           meta["l_in"], meta["l_out"], dense), emb


def _read_rows(f, dtype, d, sh, device, block_rows=1 << 18):
    """Rows of sh.tables from the open .npy member f (positioned at the data)."""
    item = np.dtype(dtype).itemsize
    base = f.tell()
    if device:
        from . import _native
        torch = _native.torch_cuda()
        emb = torch.empty((sh.local_ids, d), dtype=torch.float32, device="cuda")
    else:
        emb = np.empty((sh.local_ids, d), dtype=np.float32)
    for lt, t in enumerate(sh.tables):
        r0, rows, l0 = int(sh.offsets[t]), sh.table_sizes[t], int(sh.local_offsets[lt])
        for b in range(0, rows, block_rows):
            nb = min(block_rows, rows - b)
            f.seek(base + (r0 + b) * d * item)
            blk = np.frombuffer(f.read(nb * d * item), dtype=dtype).reshape(nb, d)
            blk = blk.astype(np.float32)
            if device:
                emb[l0 + b:l0 + b + nb].copy_(torch.from_numpy(blk))
            else:
                emb[l0 + b:l0 + b + nb] = blk
    return emb
