"""ORACLE — TEST INFRASTRUCTURE ONLY.

float64 numpy restatement of the reference model forwards, returning the
pre-sigmoid logits (the reference returns sigmoid(logit) as ``Tensor.value``).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product path never does.

Pinned: tests/golden/models.npz holds reference ``forward_*_batch`` outputs
(made by tests/golden/make_golden.py from /root/reference); the restatement
matches them to max |dp| = 0.0 (tests/test_oracle.py).

Citations are relative to /root/reference/pkg/src/embcache/neural/.
"""
from __future__ import annotations

import numpy as np


def _sigmoid(x):
    # autodiff.py:183-185
    return 1.0 / (1.0 + np.exp(-x))


def _softmax(a):
    # autodiff.py:226-236 (max-shift along axis 1)
    shifted = a - a.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=1, keepdims=True)


def _lstm_step(x, h, c, wx, wh, b, d):
    # model.py:103-112
    z = (x @ wx + h @ wh) + b
    i = _sigmoid(z[:, 0 * d:1 * d])
    f = _sigmoid(z[:, 1 * d:2 * d])
    g = np.tanh(z[:, 2 * d:3 * d])
    o = _sigmoid(z[:, 3 * d:4 * d])
    c_new = f * c + i * g
    h_new = o * np.tanh(c_new)
    return h_new, c_new


def _attend(h_prev, enc_pre, enc_stack, att_dec, att_v, mask, batch, length):
    # model.py:115-124
    query = (h_prev @ att_dec).reshape((batch, 1, -1))
    scores = (np.tanh(enc_pre + query) @ att_v).reshape((batch, length))
    if mask is not None:
        scores = scores + mask
    attn = _softmax(scores)
    return (attn.reshape((batch, length, 1)) * enc_stack).sum(axis=1)


def _encode(p, tokens, stacks, d, batch):
    # model.py:131-145
    zero = np.zeros((batch, d))
    hs = [zero] * stacks
    cs = [zero] * stacks
    top = []
    for x in tokens:
        inp = x
        for k in range(stacks):
            hs[k], cs[k] = _lstm_step(inp, hs[k], cs[k], p[f"enc{k}_wx"],
                                      p[f"enc{k}_wh"], p[f"enc{k}_b"], d)
            inp = hs[k]
        top.append(hs[-1])
    return top


def _tokens(p, gid, tid, length):
    # model.py:148-153 + autodiff.py:273-283
    tok = np.concatenate([p["embed_id"][gid], p["embed_table"][tid]], axis=2)
    return [tok[:, t, :] for t in range(length)]


def _decode_logits(p, dec_inputs, enc_states, stacks, d, batch, causal):
    # model.py:156-181, stopping before the final sigmoid (:179)
    length = len(enc_states)
    enc_stack = np.concatenate([h.reshape((batch, 1, d)) for h in enc_states], axis=1)
    enc_pre = enc_stack @ p["att_enc"]
    zero = np.zeros((batch, d))
    hs = [zero] * stacks
    cs = [zero] * stacks
    outs = []
    for t, x in enumerate(dec_inputs):
        mask = None
        if causal and t + 1 < length:
            mask = np.zeros((1, length))
            mask[:, t + 1:] = -1e9
        ctx = _attend(hs[-1], enc_pre, enc_stack, p["att_dec"], p["att_v"], mask,
                      batch, length)
        inp = np.concatenate([x, ctx], axis=1)
        for k in range(stacks):
            hs[k], cs[k] = _lstm_step(inp, hs[k], cs[k], p[f"dec{k}_wx"],
                                      p[f"dec{k}_wh"], p[f"dec{k}_b"], d)
            inp = hs[k]
        comb = np.tanh(np.concatenate([hs[-1], ctx], axis=1) @ p["comb_w"] + p["comb_b"])
        outs.append((comb @ p["head_w"] + p["head_b"]).reshape((batch,)))
    return np.stack(outs, axis=1)


def caching_logits(arrays, dim, stacks, gid, tid):
    """forward_caching_batch (model.py:184-196) as logits [B, L]."""
    gid = np.asarray(gid)
    batch, length = gid.shape
    toks = _tokens(arrays, gid, np.asarray(tid), length)
    enc = _encode(arrays, toks, stacks, dim, batch)
    return _decode_logits(arrays, toks, enc, stacks, dim, batch, causal=True)


def prefetch_logits(arrays, dim, stacks, l_out, gid, tid):
    """forward_prefetch_batch (model.py:199-212) as logits [B, l_out]."""
    gid = np.asarray(gid)
    batch, length = gid.shape
    toks = _tokens(arrays, gid, np.asarray(tid), length)
    enc = _encode(arrays, toks, stacks, dim, batch)
    zeros = np.zeros((batch, 2 * dim))
    dec_inputs = [arrays["slot_embed"][j, :] + zeros for j in range(l_out)]
    return _decode_logits(arrays, dec_inputs, enc, stacks, dim, batch, causal=False)


def sigmoid(logits):
    return _sigmoid(np.asarray(logits, dtype=np.float64))


def decode_gids(po, total_ids):
    """decode_indices (model.py:250-258) on the flat id scale."""
    g = np.floor(np.asarray(po, dtype=np.float64) * (total_ids - 1) + 0.5)
    return np.clip(g, 0, total_ids - 1).astype(np.int64)


def init_arrays(kind, table_sizes, dim, stacks=None, l_out=5, seed=0, init_scale=0.08):
    """init_params (model.py:83-100): uniform(-s, s) per array in _shapes order
    (model.py:54-80), one default_rng(seed) stream."""
    if stacks is None:
        stacks = 1 if kind == "caching" else 2
    d = dim
    total = int(sum(table_sizes))
    shapes = {
        "embed_id": (total, d), "embed_table": (len(table_sizes), d),
        "att_enc": (d, d), "att_dec": (d, d), "att_v": (d, 1),
        "comb_w": (2 * d, d), "comb_b": (d,), "head_w": (d, 1), "head_b": (1,),
    }
    for k in range(stacks):
        shapes[f"enc{k}_wx"] = (2 * d if k == 0 else d, 4 * d)
        shapes[f"enc{k}_wh"] = (d, 4 * d)
        shapes[f"enc{k}_b"] = (4 * d,)
        shapes[f"dec{k}_wx"] = (3 * d if k == 0 else d, 4 * d)
        shapes[f"dec{k}_wh"] = (d, 4 * d)
        shapes[f"dec{k}_b"] = (4 * d,)
    if kind == "prefetch":
        shapes["slot_embed"] = (l_out, 2 * d)
    rng = np.random.default_rng(seed)
    return {n: rng.uniform(-init_scale, init_scale, size=s) for n, s in shapes.items()}
