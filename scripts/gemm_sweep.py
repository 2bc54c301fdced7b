"""Sweep the CTA-pair GEMM over tile width and split-K at the backward shapes (GPU box):
    VQMC_TEST_REPS=10 python scripts/gemm_sweep.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_13308_b200 import _capi as K  # noqa: E402

K.lib.vqmc_test_umma2_gemm.argtypes = [C.c_int] * 8 + [C.c_void_p] * 3
K.lib.vqmc_test_last_ms.restype = C.c_float


def run(M, N, Kd, amn, bmn, bn, sp):
    A = np.random.default_rng(0).standard_normal((Kd, M) if amn else (M, Kd)).astype(np.float32)
    B = np.random.default_rng(1).standard_normal((Kd, N) if bmn else (N, Kd)).astype(np.float32)
    Cc = np.empty((sp, M, N), np.float32)
    K.check(K.lib.vqmc_test_umma2_gemm(M, N, Kd, amn, bmn, bn, sp, 2, K.ptr(A), K.ptr(B), K.ptr(Cc)))
    ms = K.lib.vqmc_test_last_ms()
    print(f"M={M} N={N} K={Kd} a_mn={amn} b_mn={bmn} bn={bn} splits={sp}: {ms*1e3:8.1f} us  "
          f"issued {6*M*N*Kd/ms/1e9:7.1f} TF/s", flush=True)


for bmn in (1, 0):
    for bn in (128, 256):
        for sp in (1, 4, 9, 18):
            run(1024, 424, 10000, 0, bmn, bn, sp)
for sp in (1, 2):
    run(425, 10000, 1024, 1, 1, 128, sp)
    run(425, 10000, 1024, 0, 0, 128, sp)
