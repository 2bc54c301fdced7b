"""Timeline of the tail sampler GEMM (per CTA: MMA and epilogue start / end per tile) from the
trace build (make trace).  python tools/tail_trace.py [B]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["VQMC_LIB"] = os.path.join(ROOT, "paper_2106_13308_b200", "lib", "trace", "libvqmc_trace.so")
L = C.CDLL(os.environ["VQMC_LIB"])
sys.path.insert(0, ROOT)
from paper_2106_13308_b200 import api  # noqa: E402  (host helpers only)

n = 10000
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
EXP = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # 1: no D stores, 2: no Philox
h = api.default_made_hidden(n)
m = api.made_init(n, h, 0)
hd = C.c_void_p()
e = np.zeros((0, 2), np.int32)
assert L.vqmc_gpu_create(0, n, h, m.degrees.ctypes.data_as(C.c_void_p), m.parameters().ctypes.data_as(C.c_void_p),
                         e.ctypes.data_as(C.c_void_p), C.c_int64(0), B, C.byref(hd)) == 0
out = np.zeros(148 * 32, np.uint64)
rc = L.vqmc_test_tail_trace(hd, B, out.ctypes.data_as(C.c_void_p), EXP)
assert rc == 0, rc
t = out.reshape(148, 32).astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
print("exp", EXP, "kernel span us", (t[:, 31].max() - t0) / 1e3)
for cta in (0, 1, 2, 50, 100, 146, 147):
    r = t[cta]
    s = [f"cta {cta:3d} start {(r[0]-t0)/1e3:6.2f}"]
    for j in range(6):
        ms, me, es, ee = r[1 + 4 * j: 5 + 4 * j]
        if es == 0 and ms == 0:
            continue
        f = lambda v: f"{(v - t0) / 1e3:6.2f}" if v else "   -  "
        s.append(f"| t{j} mma {f(ms)}-{f(me)} epi {f(es)}-{f(ee)}")
    s.append(f"| end {(r[31]-t0)/1e3:6.2f}")
    print(" ".join(s))
# averages over CTAs with 3 tiles
ep = []
for r in t:
    for j in range(6):
        es, ee = r[3 + 4 * j], r[4 + 4 * j]
        if es and ee:
            ep.append((ee - es) / 1e3)
print("epilogue per tile us: mean %.2f min %.2f max %.2f" % (np.mean(ep), np.min(ep), np.max(ep)))
