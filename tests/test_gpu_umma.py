"""K0: one tcgen05 GEMM per shape / kind used by the sweep, against a float64
GEMM of the same operand-rounded inputs."""

import numpy as np
import pytest

from tests.helpers import need_gpu

pytestmark = pytest.mark.gpu


def _bf16(x):
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def _tf32(x):  # round to nearest even (cvt.rn.tf32.f32)
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0xFFF + ((a >> 13) & 1)) >> 13) << 13
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("prec,n,k", [("bf16", 32, 16), ("bf16", 128, 16), ("bf16", 128, 128),
                                      ("bf16", 64, 64), ("bf16", 256, 32), ("tf32", 128, 8),
                                      ("tf32", 128, 128), ("tf32", 32, 16), ("tf32", 64, 64)])
def test_umma_gemm(prec, n, k):
    pk = need_gpu()
    rng = np.random.default_rng(n * 1000 + k)
    A = rng.normal(size=(128, k)).astype(np.float32)
    B = rng.normal(size=(k, n)).astype(np.float32)
    D = pk.selftest_umma(prec, A, B)
    r = _bf16 if prec == "bf16" else _tf32
    ref = r(A) @ r(B)
    err = np.abs(D - ref) / (np.abs(r(A)) @ np.abs(r(B)) + 1e-30)
    assert err.max() < 1e-5, f"max scaled err {err.max():.3e}"
