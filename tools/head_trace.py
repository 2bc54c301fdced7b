"""Timeline of the head sampler v5 per word (chain warp 0 of a CTA: Z(m) received, chain done,
outputs done; owner tile warp: Z(m) published) from the trace build (make trace).
    python tools/head_trace.py [B]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_2106_13308_b200", "lib", "trace", "libvqmc_trace.so"))
sys.path.insert(0, ROOT)
from paper_2106_13308_b200 import api  # noqa: E402

n, B = 10000, int(sys.argv[1]) if len(sys.argv) > 1 else 1024
h = api.default_made_hidden(n)
m = api.made_init(n, h, 0)
hd = C.c_void_p()
e = np.zeros((0, 2), np.int32)
assert L.vqmc_gpu_create(0, n, h, m.degrees.ctypes.data_as(C.c_void_p), m.parameters().ctypes.data_as(C.c_void_p),
                         e.ctypes.data_as(C.c_void_p), C.c_int64(0), B, C.byref(hd)) == 0
out = np.zeros(128 * 64, np.uint64)
assert L.vqmc_test_head_trace(hd, B, out.ctypes.data_as(C.c_void_p)) == 0
t = out.reshape(128, 64).astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
print("span us", (t[:, 63].max() - t0) / 1e3)
for cta in (0, 64, 127):
    r = t[cta]
    print(f"cta {cta}: start {(r[0] - t0) / 1e3:.2f} end {(r[63] - t0) / 1e3:.2f}")
    for w in range(15):
        zr, cd, od, pub = r[1 + 4 * w: 5 + 4 * w]
        if not zr:
            continue
        f = lambda v: f"{(v - t0) / 1e3:7.2f}" if v else "    -  "
        print(f"  word {w:2d}: Z published {f(pub)} received {f(zr)} chain done {f(cd)} ({(cd - zr) / 1e3:.2f})"
              f" outputs done {f(od)}")
