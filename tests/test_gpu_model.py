"""K1 / K2 (fp32 LSTM forwards) on the B200 vs the float64 oracle and the
reference's own outputs.  Tolerance (north star / SURVEY.md §8c): logits
within 1e-3 relative, measured as |d| <= 1e-3 * max(|ref|, 1e-2) because
relative error is meaningless at logits ~1e-6."""
import numpy as np
import pytest

import paper_2511_08568_b200 as rb
from oracle import model_oracle as mo
from conftest import golden

pytestmark = pytest.mark.gpu
RTOL = 1e-3
FLOOR = 1e-2


def _check(got, ref):
    err = np.abs(got - ref) / np.maximum(np.abs(ref), FLOOR)
    assert err.max() <= RTOL, f"max scaled error {err.max():.3e}"
    return err.max()


def test_models_vs_reference_fixture():
    m = golden("models.npz")
    sizes = [int(s) for s in m["table_sizes"]]
    for kind, dim, seed, scale in m["cases"]:
        kind = "caching" if kind == 0 else "prefetch"
        dim, seed = int(dim), int(seed)
        p = rb.init_params(kind, sizes, dim=dim, seed=seed, init_scale=float(scale))
        fwd = rb.forward_caching_batch if kind == "caching" else rb.forward_prefetch_batch
        res = fwd(p, m["gid"], m["tid"])
        probs = m[f"{kind}_{dim}_{seed}_probs"]
        ref_logit = np.log(probs) - np.log1p(-probs)
        _check(res.logits, ref_logit)
        assert np.abs(res.value - probs).max() < 1e-5


@pytest.mark.parametrize("dim", [32, 64])
@pytest.mark.parametrize("precision", ["fp32", "tc32"])
@pytest.mark.parametrize("scale", [0.08, 0.4, 0.6])
def test_config1_shapes_vs_oracle(scale, precision, dim):
    """d = 64 and the reference default d = 32 (model.py:34; tc32 runs it
    zero-padded on the d = 64 tcgen05 kernels), config-1 layout, 300 chunks
    (a ragged tile) of a config-1 style trace."""
    from paper_2511_08568_b200 import model as mdl
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 300 * 15 + 30, 1.05, 0.4, 32, 0))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    cp = rb.init_params("caching", t.table_sizes, dim=dim, seed=0, init_scale=scale)
    pp = rb.init_params("prefetch", t.table_sizes, dim=dim, seed=1, init_scale=scale)
    assert mdl.device_model(cp, precision=precision).precision == precision
    lc = rb.forward_caching_batch(cp, gid, tid, precision).logits
    lp = rb.forward_prefetch_batch(pp, gid, tid, precision).logits
    rc = mo.caching_logits(cp.arrays, dim, 1, gid, tid)
    rp = mo.prefetch_logits(pp.arrays, dim, 2, 5, gid, tid)
    _check(lc, rc)
    _check(lp, rp)
    # decisions: bit flips only where the reference logit is ~0
    flips = (lc >= 0) != (rc >= 0)
    assert np.all(np.abs(rc[flips]) < 1e-4)


@pytest.mark.parametrize("precision", ["fp32", "tc32"])
@pytest.mark.parametrize("which", ["att_enc", "att_dec", "both"])
def test_attention_exponent_range(which, precision):
    """Attention keys / queries beyond the e^(2x) fast path's range (|x| > 40)
    take the direct tanh form (lstm_tc.cu store_keys / attn_scores)."""
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 300 * 15 + 30, 1.05, 0.4, 32, 0))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    for kind, seed in (("caching", 0), ("prefetch", 1)):
        p = rb.init_params(kind, t.table_sizes, dim=64, seed=seed, init_scale=0.4)
        for name in ("att_enc", "att_dec"):
            if which in (name, "both"):
                p.arrays[name] = (p.arrays[name] * 60.0).astype(p.arrays[name].dtype)
        if kind == "caching":
            got = rb.forward_caching_batch(p, gid, tid, precision).logits
            ref = mo.caching_logits(p.arrays, 64, 1, gid, tid)
        else:
            got = rb.forward_prefetch_batch(p, gid, tid, precision).logits
            ref = mo.prefetch_logits(p.arrays, 64, 2, 5, gid, tid)
        _check(got, ref)


@pytest.mark.parametrize("vscale", [1.0, 10.0])
def test_softmax_shift_paths(vscale):
    """The tc kernels shift the attention softmax by sum|att_v| (a bound on
    every score) while that stays <= 40, and by the running max beyond
    (lstm_tc.cu attn_context): both paths against the float64 oracle."""
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 300 * 15 + 30, 1.05, 0.4, 32, 0))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    for kind, seed in (("caching", 0), ("prefetch", 1)):
        p = rb.init_params(kind, t.table_sizes, dim=64, seed=seed, init_scale=0.4)
        p.arrays["att_v"] = (p.arrays["att_v"] * vscale).astype(p.arrays["att_v"].dtype)
        assert (np.abs(p.arrays["att_v"]).sum() > 40.0) == (vscale > 1.0)
        if kind == "caching":
            got = rb.forward_caching_batch(p, gid, tid, "tc32").logits
            ref = mo.caching_logits(p.arrays, 64, 1, gid, tid)
        else:
            got = rb.forward_prefetch_batch(p, gid, tid, "tc32").logits
            ref = mo.prefetch_logits(p.arrays, 64, 2, 5, gid, tid)
        _check(got, ref)


@pytest.mark.parametrize("precision", ["fp32", "tc32"])
def test_batch_equals_single_bit_exact(precision):
    """test_model.py:89-96 (batch == single at rel 1e-12), held bit-exactly:
    a chunk's logits do not depend on its tile, its row in the tile or the
    batch size (one chunk alone, a permuted batch, a ragged tail)."""
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 300 * 15 + 30, 1.05, 0.4, 32, 0))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    perm = np.random.default_rng(5).permutation(K)
    for kind, seed, fwd in (("caching", 0, rb.forward_caching_batch),
                            ("prefetch", 1, rb.forward_prefetch_batch)):
        p = rb.init_params(kind, t.table_sizes, dim=64, seed=seed, init_scale=0.4)
        full = fwd(p, gid, tid, precision).logits
        shuf = fwd(p, gid[perm], tid[perm], precision).logits
        assert np.array_equal(shuf, full[perm]), kind
        for k in (0, 129, K - 1):
            one = fwd(p, gid[k:k + 1], tid[k:k + 1], precision).logits
            assert np.array_equal(one[0], full[k]), (kind, k)
        tail = fwd(p, gid[K - 45:], tid[K - 45:], precision).logits
        assert np.array_equal(tail, full[K - 45:]), kind


def test_gpu_decisions_in_replay_path():
    """bits / decoded prefetch ids emitted by the kernel (runtime.py:192,
    model.py:250-258) vs the oracle's, through the replay entry point."""
    import torch
    from paper_2511_08568_b200.model import DeviceModel
    t = rb.generate_trace(rb.TraceGenConfig([250] * 8, 3000 * 15 + 30, 1.05, 0.4, 32, 3))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    g = torch.from_numpy(gid.astype(np.int32)).cuda()
    dm = DeviceModel(cp)
    tt = dm.table_ids(g)
    assert np.array_equal(tt.cpu().numpy(), tid)
    bits = torch.empty((K, 15), dtype=torch.uint8, device="cuda")
    lc = dm.forward(g, tt, bits=bits).cpu().numpy()
    assert np.array_equal(bits.cpu().numpy(), (lc >= 0).astype(np.uint8))
    dp = DeviceModel(pp)
    pf = torch.empty((K, 5), dtype=torch.int32, device="cuda")
    lp = dp.forward(g, tt, pf_gid=pf).cpu().numpy()
    want = mo.decode_gids(mo.sigmoid(lp.astype(np.float64)), t.total_ids)
    assert np.array_equal(pf.cpu().numpy(), want)
    rp = mo.prefetch_logits(pp.arrays, 64, 2, 5, gid, tid)
    agree = np.mean(pf.cpu().numpy() == mo.decode_gids(mo.sigmoid(rp), t.total_ids))
    assert agree > 0.97, agree


def test_zero_weights_and_causality():
    sizes = [6, 10]
    # test_model.py:45-58
    p = rb.init_params("caching", sizes, dim=4, l_in=5, seed=0)
    for a in p.arrays.values():
        a[:] = 0.0
    probs = rb.forward_caching(p, rb.trace_from_gids([0, 3, 7, 7, 1], sizes).accesses)
    assert probs == [0.5] * 5
    p = rb.init_params("prefetch", sizes, dim=4, l_in=4, l_out=3, seed=0)
    for a in p.arrays.values():
        a[:] = 0.0
    po = rb.forward_prefetch(p, rb.trace_from_gids([0, 1, 2, 3], sizes).accesses)
    assert po == [po[0]] * 3
    # test_model.py:71-77 (causal attention)
    p = rb.init_params("caching", sizes, dim=6, l_in=6, seed=8)
    a = rb.forward_caching(p, rb.trace_from_gids([0, 3, 7, 2, 5, 9], sizes).accesses)
    b = rb.forward_caching(p, rb.trace_from_gids([0, 3, 7, 8, 8, 8], sizes).accesses)
    assert a[:3] == b[:3]
    assert all(abs(x - y) > 1e-9 for x, y in zip(a[3:], b[3:]))


def test_replay_with_gpu_models_end_to_end():
    """replay(caching_params, prefetch_params): decisions from K1/K2 feed K3;
    the result equals the oracle replay of the kernel's own decisions."""
    import oracle
    import torch
    from paper_2511_08568_b200.model import DeviceModel
    t = rb.generate_trace(rb.TraceGenConfig([250] * 8, 20000, 1.05, 0.4, 32, 9))
    cp = rb.init_params("caching", t.table_sizes, dim=32, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=32, seed=1, init_scale=0.4)
    C = int(0.2 * t.unique_count)
    rep = rb.replay(t, rb.BufferConfig(C), cp, pp)
    K = rb.num_chunks(len(t))
    g = torch.from_numpy(t.gid_array[:K * 15].reshape(K, 15).astype(np.int32)).cuda()
    dc, dp = DeviceModel(cp), DeviceModel(pp)
    tt = dc.table_ids(g)
    bits = torch.empty((K, 15), dtype=torch.uint8, device="cuda")
    pf = torch.empty((K, 5), dtype=torch.int32, device="cuda")
    dc.forward(g, tt, bits=bits)
    dp.forward(g, tt, pf_gid=pf)
    ref, cov = oracle.replay(t.gid_array, t.total_ids, C, 0, 4, bits=bits.cpu().numpy(),
                             pf=pf.cpu().numpy().astype(np.int64))
    assert (rep.cache_hits, rep.prefetch_hits, rep.on_demand, rep.prefetch_useful) == \
        (ref["cache_hits"], ref["prefetch_hits"], ref["on_demand"], ref["prefetch_useful"])
    assert rep.coverage == cov


def test_hotpath_pipelined_equals_single_replay():
    """HotPath with the replay pipelined in chunk pieces on a side stream (and
    the LRU on a third) reports exactly what one replay reports."""
    from paper_2511_08568_b200.pipeline import HotPath
    t = rb.generate_trace(rb.TraceGenConfig([5000] * 16, 300_000, 1.05, 0.4, 32, 4))
    cp = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    pp = rb.init_params("prefetch", t.table_sizes, dim=64, seed=1, init_scale=0.4)
    C = int(0.2 * t.unique_count)
    C32 = C - C % 32
    reps = []
    for pieces in (1, 4, 7):
        hp = HotPath(cp, pp, t.table_sizes, C32, len(t), ways=32, lru_capacity=C32,
                     lru_ways=32, pieces=pieces)
        reps.append(hp.replay_host(t.gid_array.astype(np.int32)))
    assert reps[0] == reps[1] == reps[2]
    rep, (h, m) = reps[0]
    assert rep.total == len(t) and h + m == len(t)
    ref = rb.replay(t, rb.BufferConfig(C32, 4, 32), cp, pp)
    assert ref == rep and ref.evictions == rep.evictions
    assert m == rb.simulate(t, rb.CacheConfig(C32, rb.Policy.LRU, 32), per_access=False).misses


def test_tc16_variant_bounded_and_reported():
    """RECMG_PREC_TC16 (one fp16 product per GEMM, the reduced-precision
    variant reported separately): bounded logit error, caching bits agree
    with the float64 reference on >= 99.5% of accesses at init 0.4."""
    t = rb.generate_trace(rb.TraceGenConfig([2000] * 8, 1000 * 15 + 30, 1.05, 0.4, 32, 0))
    K = rb.num_chunks(len(t))
    gid = t.gid_array[:K * 15].reshape(K, 15)
    tid = t.table_ids[:K * 15].reshape(K, 15)
    p = rb.init_params("caching", t.table_sizes, dim=64, seed=0, init_scale=0.4)
    ref = mo.caching_logits(p.arrays, 64, 1, gid, tid)
    got = rb.forward_caching_batch(p, gid, tid, precision="tc16").logits
    tc32 = rb.forward_caching_batch(p, gid, tid, precision="tc32").logits
    e16 = (np.abs(got - ref) / np.maximum(np.abs(ref), FLOOR)).max()
    e32 = (np.abs(tc32 - ref) / np.maximum(np.abs(ref), FLOOR)).max()
    assert e32 <= RTOL < e16 < 1.0, (e32, e16)
    assert ((got >= 0) == (ref >= 0)).mean() >= 0.995
