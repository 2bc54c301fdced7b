"""Quick GPU sanity check: product vs oracle on small cases (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import ctypes as C
import numpy as np
from paper_2106_13308_b200 import _capi as K
import pyoracle as O

def handle(n, h, seed, edges, B):
    deg = np.empty(h, np.int32); th = np.empty(2*h*n+h+n)
    K.check(K.lib.vqmc_made_init(n, h, seed, K.ptr(deg), K.ptr(th)))
    hd = C.c_void_p()
    e = np.ascontiguousarray(edges, np.int32)
    K.check(K.lib.vqmc_gpu_create(0, n, h, K.ptr(deg), K.ptr(th), K.ptr(e), len(e), B, C.byref(hd)))
    return hd, deg, th

cases = [tuple(map(int, a.split(':'))) for a in sys.argv[1:]] or [(20, 256), (100, 256), (1000, 64)]
for (n, B) in cases:
    h = O.default_made_hidden(n)
    e = O.random_maxcut_graph(n, 0) if n <= 1000 else O.random_regular_graph(n, 3, 0)
    hd, deg, th = handle(n, h, 0, e, B)
    m = O.Made(n, h, deg, th)
    m.theta = m.theta + (O.uniforms(0, 98, m.d) * 3.0 - 1.5)
    K.check(K.lib.vqmc_gpu_set_params(hd, K.ptr(m.theta)))
    U = O.uniforms(0, 1, n * B).reshape(n, B)
    W = (n + 31) // 32
    bits = np.empty((B, W), np.uint32); lp = np.empty(B)
    t = time.time()
    K.check(K.lib.vqmc_gpu_sample(hd, B, K.ptr(U), 0, 1, 0, K.ptr(bits), K.ptr(lp)))
    xg = K.unpack_bits(bits, n)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1, want_p=True)
    mism = (xg != xo)
    first = [np.argmax(r) if r.any() else -1 for r in mism]
    bad = [(b, i, abs(U[i, b] - po[b, i])) for b, i in enumerate(first) if i >= 0]
    print(f"n={n} B={B}: rows with flips {len(bad)}, max|u-p| at flip {max([x[2] for x in bad], default=0):.2e}, "
          f"lp maxrel {np.max(np.abs(lp - lo) / np.abs(lo)):.2e}")
    # energies on oracle samples
    ob = K.pack_bits(xo)
    cut = np.empty(B, np.int32); le = np.empty(B)
    K.check(K.lib.vqmc_gpu_maxcut_energy(hd, K.ptr(ob), B, K.ptr(cut), K.ptr(le)))
    leo, cuto = O.local_energy(n, e, xo)
    print("  energy exact:", np.array_equal(le, leo), np.array_equal(cut.astype(float), cuto))
    lpsi = np.empty(B)
    K.check(K.lib.vqmc_gpu_log_psi(hd, K.ptr(ob), B, K.ptr(lpsi), None))
    lpo = O.log_psi(m, xo)
    print("  log_psi maxrel", np.max(np.abs(lpsi - lpo) / np.abs(lpo)))
    g = np.empty(m.d)
    K.check(K.lib.vqmc_gpu_gradient_from_locals(hd, K.ptr(ob), K.ptr(leo), B, K.ptr(g)))
    go = O.gradient_from_locals(m, xo, leo)
    print("  grad norm-rel", np.linalg.norm(g - go) / np.linalg.norm(go), "max abs", np.abs(g-go).max(), "gmax", np.abs(go).max())
    K.check(K.lib.vqmc_gpu_destroy(hd))
print("OK")
