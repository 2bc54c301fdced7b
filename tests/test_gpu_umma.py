"""tcgen05 3-pass GEMMs (csrc/umma_gemm.cuh: 3xTF32, 3xBF16 and 3xFP16 operand pairs) against an fp64 numpy product,
all operand majorness combinations, partial tiles and split-K."""
import ctypes as C

import numpy as np
import pytest

from paper_2106_13308_b200 import _capi as K

pytestmark = pytest.mark.gpu
K.lib.vqmc_test_umma_gemm.argtypes = [C.c_int] * 8 + [C.c_void_p] * 3
K.lib.vqmc_test_umma_gemm.restype = C.c_int


@pytest.mark.parametrize("ek", [0, 1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,Kd,bn,splits", [(128, 128, 32, 128, 1), (200, 300, 424, 128, 1),
                                               (1024, 424, 1000, 256, 3), (300, 425, 96, 256, 1)])
def test_umma_3pass(a_mn, b_mn, M, N, Kd, bn, splits, ek):
    rng = np.random.default_rng(M + N + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    Ah = np.ascontiguousarray(A.T if a_mn else A)
    Bh = np.ascontiguousarray(B.T if b_mn else B)
    Cout = np.empty((splits, M, N), np.float32)
    K.check(K.lib.vqmc_test_umma_gemm(M, N, Kd, a_mn, b_mn, bn, splits, ek, K.ptr(Ah), K.ptr(Bh), K.ptr(Cout)))
    got = Cout.sum(axis=0, dtype=np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.sqrt(Kd)
    err = np.abs(got - ref).max() / scale
    # 3xTF32 and 3xFP16: fp32-grade (products ~2^-21); 3xBF16: products ~2^-16 relative
    assert err < (2e-4 if ek == 1 else 2e-5), err


K.lib.vqmc_test_umma2_gemm.argtypes = [C.c_int] * 8 + [C.c_void_p] * 3
K.lib.vqmc_test_umma2_gemm.restype = C.c_int


@pytest.mark.parametrize("ek", [1, 2])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,Kd,bn,splits", [(256, 256, 64, 256, 1), (512, 424, 1000, 256, 3),
                                               (300, 425, 96, 192, 1), (1024, 640, 448, 128, 1),
                                               (425, 1000, 1024, 256, 2)])
def test_umma_pair_3pass(a_mn, b_mn, M, N, Kd, bn, splits, ek):
    """CTA-pair (cta_group::2, M = 256) kernel: same products as the single-CTA one."""
    if bn == 192 and b_mn:
        pytest.skip("bn 192 halves are 96 columns: MN-major B needs whole 64-element atoms")
    rng = np.random.default_rng(7 * M + N + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    Ah = np.ascontiguousarray(A.T if a_mn else A)
    Bh = np.ascontiguousarray(B.T if b_mn else B)
    Cout = np.empty((splits, M, N), np.float32)
    K.check(K.lib.vqmc_test_umma2_gemm(M, N, Kd, a_mn, b_mn, bn, splits, ek, K.ptr(Ah), K.ptr(Bh), K.ptr(Cout)))
    got = Cout.sum(axis=0, dtype=np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(got - ref).max() / np.sqrt(Kd)
    assert err < (2e-4 if ek == 1 else 2e-5), err
