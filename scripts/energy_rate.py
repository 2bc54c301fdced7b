#!/usr/bin/env python
"""Energy-kernel throughput on the B200 ("achieved HBM GB/s for the energy kernel",
with a large-batch microbench since B = 1024 is launch-latency-bound).

    python scripts/energy_rate.py [--out profiles/energy_rate.json]

* edge-list path (3-regular N = 10k, the headline instance): B = 1024 ... 2^20 device-resident
  random spin rows; compulsory bytes = 4 B W (packed spins) + 8 |E| (edge list) + 4 B chunks
  (partial counts written), vs the measured HBM peak (MEASURED_PEAKS.json hbm_gbs);
* dense path (the reference generator's G(10^4, 3/4), |E| ~ 3.75e7): the fp8 tensor-core quadratic
  form; useful FLOPs = 2 B n (n - 1) / 2 (the strictly upper triangle of X U^T) vs the measured
  dense bf16 peak x 2 (fp8 rate; stated).
Kernel time = CUDA events around `iters` back-to-back launches on the library's stream.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_13308_b200 import _capi as K  # noqa: E402
from paper_2106_13308_b200 import api  # noqa: E402

K.lib.vqmc_test_energy_rate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int)]
K.lib.vqmc_test_energy_rate.restype = C.c_int


def handle(n, edges):
    h = api.default_made_hidden(n)
    m = api.made_init(n, h, 0)
    hd = C.c_void_p()
    e = np.ascontiguousarray(edges, np.int32)
    K.check(K.lib.vqmc_gpu_create(0, n, h, K.ptr(m.degrees), K.ptr(m.parameters()), K.ptr(e), len(e), 64,
                                  C.byref(hd)))
    return hd


def rate(hd, B, iters):
    ms, ch = C.c_float(), C.c_int()
    K.check(K.lib.vqmc_test_energy_rate(hd, B, iters, C.byref(ms), C.byref(ch)))
    return float(ms.value), int(ch.value)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--only-b", type=int, default=0, help="edge-list path at this batch only (profiling)")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16 = peaks.get("bf16_tflops", 2250.0)
    n = args.n
    W = (n + 31) // 32
    out = {"edge_list": [], "dense": []}
    g = api.random_regular_graph(n, 3, 0)
    E = len(g.edges)
    hd = handle(n, g.edges)
    for B in ((args.only_b,) if args.only_b else (1024, 1 << 14, 1 << 17, 1 << 20)):
        ms, ch = rate(hd, B, 20 if B <= (1 << 17) else 5)
        byts = 4.0 * B * W + 8.0 * E + 4.0 * B * ch
        gbs = byts / (ms * 1e-3) / 1e9
        rec = {"graph": f"random 3-regular N={n}, |E|={E}", "B": B, "ms": ms, "chunks": ch,
               "compulsory_bytes": byts, "GB_per_s": gbs, "peak_GB_per_s": hbm, "frac": gbs / hbm,
               "samples_per_s": B / (ms * 1e-3)}
        out["edge_list"].append(rec)
        print(json.dumps(rec), flush=True)
    K.lib.vqmc_gpu_destroy(hd)
    if args.only_b:
        return
    gd = api.random_maxcut_graph(n, 0)
    Ed = len(gd.edges)
    hd = handle(n, gd.edges)
    for B in (1024, 4096):
        ms, ch = rate(hd, B, 10)
        fl = 2.0 * B * n * (n - 1) / 2.0
        tf = fl / (ms * 1e-3) / 1e12
        rec = {"graph": f"reference G(n,3/4) N={n}, |E|={Ed}", "B": B, "ms": ms, "partials": ch,
               "useful_flop": fl, "TFLOP_per_s": tf, "peak_TFLOP_per_s": 2 * bf16,
               "peak_src": "MEASURED_PEAKS bf16_tflops x 2 (the fp8 kind::f8f6f4 rate)", "frac": tf / (2 * bf16),
               "samples_per_s": B / (ms * 1e-3), "edge_pairs_per_s": B * Ed / (ms * 1e-3)}
        out["dense"].append(rec)
        print(json.dumps(rec), flush=True)
    K.lib.vqmc_gpu_destroy(hd)
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
