"""SGD + SR step rate at the headline configuration (N = 10k random 3-regular Max-Cut, MADE h = 424,
1024 samples): ms per SR step and CG iterations (the reference's CG, optimizer.cpp:46-71)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2106_13308_b200 import _capi as K  # noqa: E402
from paper_2106_13308_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = api.random_regular_graph(n, 3, 0)
h = api.default_made_hidden(n)
model = api.made_init(n, h, 0)
dev = model.device()
dev.set_problem(api.maxcut_spec(g))
st = K.StepStats()
it, res = C.c_int(0), C.c_double(0.0)
for s in range(steps + 1):
    if s == 1:
        K.check(K.lib.vqmc_gpu_synchronize(dev.h))
        t0 = time.perf_counter()
    K.check(K.lib.vqmc_gpu_train_step_sr(dev.h, 1024, 1, None, 0, 1, s, 0.1, 1e-3, 1e-6, 200, 1, 1, C.byref(st),
                                         C.byref(it), C.byref(res)))
    print(f"step {s}: energy {st.energy_mean:.2f} grad_norm {st.grad_norm:.3e} cg_iters {it.value} resid {res.value:.2e}")
K.check(K.lib.vqmc_gpu_synchronize(dev.h))
dt = (time.perf_counter() - t0) / steps
print(f"SR step: {dt * 1e3:.2f} ms ({1024 / dt:.0f} samples/s)")
