"""Artifact ingest: checkpoints and trace files written
by the reference itself (tests/golden/make_golden.py --only artifacts) read
back identically, with the reference's errors; the shard readers return the
same arrays as the whole-file readers restricted to the shard."""
import json
import os
import zipfile

import numpy as np
import pytest

import paper_2511_08568_b200 as rb
from paper_2511_08568_b200 import checkpoint as ck
from paper_2511_08568_b200 import errors, shard
from paper_2511_08568_b200 import trace as tr
from conftest import GOLDEN

SIZES = [30, 5, 70, 12]


def test_reference_checkpoint_loads_bit_exact():
    p = ck.load_checkpoint(os.path.join(GOLDEN, "ref_ckpt_prefetch.npz"), SIZES)
    want = rb.init_params("prefetch", SIZES, dim=8, seed=9, init_scale=0.4)
    assert (p.kind, p.dim, p.stacks, p.l_in, p.l_out, p.table_sizes) == \
        ("prefetch", 8, 2, 15, 5, SIZES)
    assert list(p.arrays) == list(want.arrays)
    for k in want.arrays:
        assert np.array_equal(p.arrays[k], want.arrays[k]), k


def test_save_matches_reference_container(tmp_path):
    want = rb.init_params("prefetch", SIZES, dim=8, seed=9, init_scale=0.4)
    path = str(tmp_path / "mine.npz")
    ck.save_checkpoint(want, path)
    ref = np.load(os.path.join(GOLDEN, "ref_ckpt_prefetch.npz"))
    mine = np.load(path)
    assert ref.files == mine.files
    assert json.loads(str(ref["__meta__"])) == json.loads(str(mine["__meta__"]))
    for k in ref.files:
        assert np.array_equal(ref[k], mine[k]), k


def test_checkpoint_errors(tmp_path):
    src = os.path.join(GOLDEN, "ref_ckpt_prefetch.npz")
    with pytest.raises(errors.MissingArtifactError):
        ck.load_checkpoint(str(tmp_path / "nope.npz"))
    with pytest.raises(errors.VocabularyMismatchError):
        ck.load_checkpoint(src, [30, 5, 70, 13])
    bad = tmp_path / "bad.npz"
    bad.write_bytes(b"not a zip")
    with pytest.raises(errors.CheckpointError):
        ck.load_checkpoint(str(bad))
    nometa = tmp_path / "nometa.npz"
    with zipfile.ZipFile(src) as zin, zipfile.ZipFile(nometa, "w") as zout:
        for item in zin.infolist():
            if item.filename != "__meta__.npy":
                zout.writestr(item, zin.read(item.filename))
    with pytest.raises(errors.CheckpointError):
        ck.load_checkpoint(str(nometa))
    for loader in (ck.load_checkpoint, lambda p: ck.load_checkpoint_shard(p, [0], device=False)):
        with pytest.raises(errors.CheckpointError):
            loader(str(nometa))


def test_checkpoint_shard_reader(tmp_path):
    src = os.path.join(GOLDEN, "ref_ckpt_prefetch.npz")
    full = ck.load_checkpoint(src)
    for tables in ([2], [0, 3], [3, 1, 2]):
        sh = shard.TableShard(SIZES, tables)
        p, emb = ck.load_checkpoint_shard(src, sh, SIZES, device=False)
        q, emb2 = shard.init_params_shard("prefetch", SIZES, sh, dim=8, seed=9, init_scale=0.4,
                                          device=False)
        rows = np.concatenate([np.arange(sh.offsets[t], sh.offsets[t + 1]) for t in sh.tables])
        assert np.array_equal(emb, full.arrays["embed_id"][rows].astype(np.float32))
        assert np.array_equal(emb, emb2)
        assert p.table_sizes == q.table_sizes
        for k in q.arrays:
            assert np.array_equal(p.arrays[k], q.arrays[k]), k
    with pytest.raises(errors.VocabularyMismatchError):
        ck.load_checkpoint_shard(src, [0], [30, 5, 70, 11], device=False)


def test_reference_trace_file_reads_identically(tmp_path):
    t = tr.read_trace(os.path.join(GOLDEN, "ref_trace.txt"))
    want = rb.generate_trace(rb.TraceGenConfig([300, 50, 7], 3000, 1.05, 0.4, 32, 1))
    assert t == want
    out = str(tmp_path / "w.txt")
    tr.write_trace(want, out)
    assert open(out).read() == open(os.path.join(GOLDEN, "ref_trace.txt")).read()


def test_trace_parse_cases_match_reference(tmp_path):
    cases = json.load(open(os.path.join(GOLDEN, "ref_trace_cases.json")))
    for name, c in cases.items():
        path = tmp_path / f"{name}.txt"
        path.write_bytes(c["body"].encode("utf-8"))
        if "error" in c:
            with pytest.raises(getattr(errors, c["error"])) as ei:
                tr.read_trace(str(path))
            assert str(ei.value) == c["msg"], name
        else:
            t = tr.read_trace(str(path))
            assert t.gid_array.tolist() == c["ok"] and t.table_sizes == c["sizes"], name


def test_binary_trace_round_trip(tmp_path):
    want = rb.generate_trace(rb.TraceGenConfig([300, 50, 7], 3000, 1.05, 0.4, 32, 1))
    p = str(tmp_path / "t.bin")
    tr.write_trace_binary(want, p)
    assert tr.read_trace_binary(p) == want
    g, sizes = tr.read_trace_binary(p, mmap=True)
    assert np.array_equal(np.asarray(g), want.gid_array) and sizes == want.table_sizes
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXXXXXX" + b"\0" * 16)
    with pytest.raises(errors.TraceParseError):
        tr.read_trace_binary(str(bad))
