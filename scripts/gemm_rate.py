"""Throughput of the CTA-pair 3-pass GEMM (test hook) at a few shapes: TFLOP/s of useful (1-pass)
and issued (3-pass) work.  Run on the GPU box:  VQMC_TEST_REPS=20 python scripts/gemm_rate.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_13308_b200 import _capi as K  # noqa: E402

K.lib.vqmc_test_umma2_gemm.argtypes = [C.c_int] * 8 + [C.c_void_p] * 3
K.lib.vqmc_test_last_ms.restype = C.c_float
shapes = [(4096, 4096, 4096, 0, 0, 256, 1), (4096, 4096, 4096, 1, 1, 256, 1), (4096, 4096, 4096, 0, 1, 256, 1),
          (1024, 9584, 448, 0, 0, 192, 1), (1024, 424, 10000, 0, 1, 256, 9), (425, 10000, 1024, 1, 1, 128, 1),
          (425, 10000, 1024, 1, 1, 256, 1)]
for (M, N, Kd, amn, bmn, bn, sp) in shapes:
    A = np.random.default_rng(0).standard_normal((Kd, M) if amn else (M, Kd)).astype(np.float32)
    B = np.random.default_rng(1).standard_normal((Kd, N) if bmn else (N, Kd)).astype(np.float32)
    Cc = np.empty((sp, M, N), np.float32)
    K.check(K.lib.vqmc_test_umma2_gemm(M, N, Kd, amn, bmn, bn, sp, 2, K.ptr(A), K.ptr(B), K.ptr(Cc)))
    ms = K.lib.vqmc_test_last_ms()
    f = 2.0 * M * N * Kd
    print(f"M={M} N={N} K={Kd} a_mn={amn} b_mn={bmn} bn={bn} splits={sp}: {ms*1e3:8.1f} us  "
          f"useful {f/ms/1e9:7.1f} TF/s  issued {3*f/ms/1e9:7.1f} TF/s")
