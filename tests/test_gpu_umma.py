"""tcgen05 building blocks (descriptors, TMEM ld/st, A from TMEM) vs numpy."""
import ctypes

import numpy as np
import pytest

from paper_2511_08568_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("a_in_tmem", [0, 1])
@pytest.mark.parametrize("N,K", [(16, 16), (64, 64), (256, 64), (128, 256), (256, 256)])
def test_umma_gemm(N, K, a_in_tmem):
    import torch
    rng = np.random.default_rng(N * 1000 + K + a_in_tmem)
    # small integers / 8: every product and partial sum is exact in fp32
    A = (rng.integers(-8, 9, (128, K)) / 8).astype(np.float16)
    B = (rng.integers(-8, 9, (N, K)) / 8).astype(np.float16)
    a = torch.from_numpy(A).cuda()
    b = torch.from_numpy(B).cuda()
    d = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    rc = _native.lib().recmg_selftest_umma(_native.ptr(a), _native.ptr(b), _native.ptr(d), N, K,
                                           a_in_tmem, _native.stream_handle(torch))
    assert rc == 0
    got = d.cpu().numpy()
    want = A.astype(np.float64) @ B.astype(np.float64).T
    assert np.array_equal(got, want), np.abs(got - want).max()
