#!/usr/bin/env python
"""Stand-alone forward and TIM local-energy throughput on the B200 (device-resident random
configurations; CUDA events on the library's stream; per-kernel events from one extra pass).

    python scripts/forward_rate.py [--out profiles/forward_rate.json]

* log_psi_batch (models.cpp:122-124) at the headline shape N = 10k, h = 424, B = 1024: z1_given
  (SIMT, K = Hd) + the tcgen05 pair GEMM with the given-bits epilogue over all n outputs.  Useful
  FLOPs = 2 B (nnz(M1) + nnz(M2)) (masked); the GEMM issues 3 passes over [G1 | 1] x [W2 | b2].
* local_energy_batch on random_tim(n) (estimator.hpp:43-90) at the paper's TIM shapes (PAPER.md
  Table "samples per GPU": n = 10000 with 4 samples, 1000 with 2^9, 100 with 2^15, ...), and the
  TIM training step (vqmc_gpu_train_step with the spec set) at the same shapes.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_13308_b200 import _capi as K  # noqa: E402
from paper_2106_13308_b200 import api  # noqa: E402

K.lib.vqmc_test_forward_rate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.c_void_p,
                                         C.c_void_p, C.c_int, C.POINTER(C.c_int)]
K.lib.vqmc_test_forward_rate.restype = C.c_int


def handle(n, B, spec=None):
    h = api.default_made_hidden(n)
    m = api.made_init(n, h, 0)
    hd = C.c_void_p()
    e = np.zeros((0, 2), np.int32)
    K.check(K.lib.vqmc_gpu_create(0, n, h, K.ptr(m.degrees), K.ptr(m.parameters()), K.ptr(e), 0, B, C.byref(hd)))
    if spec is not None:
        K.check(K.lib.vqmc_gpu_set_spec(hd, K.ptr(spec.alpha), K.ptr(spec.beta), K.ptr(spec.pair_i),
                                        K.ptr(spec.pair_j), K.ptr(spec.pair_value), len(spec.pair_i)))
    return hd, m


def rate(hd, B, iters, mode):
    ms, cnt = C.c_float(), C.c_int()
    names = C.create_string_buffer(32 * 128)
    kms = (C.c_float * 128)()
    K.check(K.lib.vqmc_test_forward_rate(hd, B, iters, mode, C.byref(ms), names, kms, 128, C.byref(cnt)))
    kern = {}
    for i in range(cnt.value):
        name = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
        kern[name] = round(kern.get(name, 0.0) + kms[i], 5)
    return float(ms.value), kern


def nnz(m):
    deg = m.degrees.astype(np.int64)
    n = m.n
    return int(deg.sum()), int(np.sum(n - deg))  # nnz(M1) = sum_k deg_k, nnz(M2) = sum_k (n - deg_k)


def train_rate(hd, B, steps):
    st = K.StepStats()
    K.check(K.lib.vqmc_gpu_set_phase_timing(hd, 1))
    K.check(K.lib.vqmc_gpu_train_step(hd, B, 1, None, 1, 1, 0, 0.01, 0.9, 0.999, 1e-8, 1, C.byref(st)))
    tot = 0.0
    for s in range(steps):
        K.check(K.lib.vqmc_gpu_train_step(hd, B, 1, None, 1, 1, s + 1, 0.01, 0.9, 0.999, 1e-8, s + 2, C.byref(st)))
        ph = (C.c_float * 5)()
        K.check(K.lib.vqmc_gpu_phase_times(hd, ph))
        tot += ph[0]
    return tot / steps, st.energy_mean


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tim", default=None, help="only these TIM shapes, e.g. 10000:4,1000:1024 (no forward, no step)")
    a = ap.parse_args()
    if a.tim:
        for nb in a.tim.split(","):
            n, B = map(int, nb.split(":"))
            hd, m = handle(n, B, api.random_tim(n, 0))
            ms, kern = rate(hd, B, a.iters, 1)
            print(json.dumps(dict(n=n, B=B, ms=ms, kernels_ms=kern)), flush=True)
            K.lib.vqmc_gpu_destroy(hd)
        return
    res = {"device": "B200", "forward": [], "tim_local_energy": [], "tim_train_step": []}
    for n, B in ((10000, 1024), (5000, 1024), (1000, 1024)):
        hd, m = handle(n, B)
        ms, kern = rate(hd, B, a.iters, 0)
        n1, n2 = nnz(m)
        useful = 2.0 * B * (n1 + n2)
        gemm_ms = kern.get("z2_given_umma", ms)
        dense = 2.0 * B * n * (m.h + 1)
        res["forward"].append(dict(n=n, h=m.h, B=B, ms=ms, samples_per_s=B / ms * 1e3, kernels_ms=kern,
                                   useful_gflop=useful / 1e9,
                                   gemm_tflops_dense_as_stored=dense / (gemm_ms * 1e-3) / 1e12,
                                   note="useful = 2 B (nnz(M1) + nnz(M2)); the GEMM's dense-as-stored work is "
                                        "2 B n (h + 1) per pass (3 fp16-pair passes)"))
        K.lib.vqmc_gpu_destroy(hd)
        print(json.dumps(res["forward"][-1]), flush=True)
    for n, B in ((10000, 4), (5000, 16), (2000, 128), (1000, 512), (500, 2048), (200, 8192), (100, 32768),
                 (20, 32768), (1000, 1024)):
        spec = api.random_tim(n, 0)
        hd, m = handle(n, B, spec)
        ms, kern = rate(hd, B, max(3, a.iters // 4), 1)
        Hd = int(m.degrees.max())
        res["tim_local_energy"].append(dict(n=n, h=m.h, Hd=Hd, B=B, pairs=len(spec.pair_i), ms=ms,
                                            samples_per_s=B / ms * 1e3,
                                            neighbour_rows=B * min(Hd, n), kernels_ms=kern))
        print(json.dumps(res["tim_local_energy"][-1]), flush=True)
        step_ms, e = train_rate(hd, B, 5)
        res["tim_train_step"].append(dict(n=n, B=B, ms=step_ms, steps_per_s=1e3 / step_ms,
                                          samples_per_s=B / step_ms * 1e3, energy=e))
        print(json.dumps(res["tim_train_step"][-1]), flush=True)
        K.lib.vqmc_gpu_destroy(hd)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
