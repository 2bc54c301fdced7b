"""Kernel timing modes of the fused step (include/vqmc_b200.h vqmc_gpu_set_kernel_timing): the
timeline mode (2) keeps the production schedule -- gW2 and the [W2 | b2] Adam on the side stream
beside dg1 -> dz1 -> gW1 -- and reports every kernel's start / end after the step-start event; the
serial mode (1) and the timeline give the same parameters as an untimed step (timing events do not
change the arithmetic)."""
import ctypes as C

import numpy as np
import pytest

from paper_2106_13308_b200 import _capi as K
from paper_2106_13308_b200 import api

pytestmark = pytest.mark.gpu


def _step(dev, t):
    st = K.StepStats()
    K.check(K.lib.vqmc_gpu_train_step(dev.h, 256, 1, None, 3, 1, t, 0.01, 0.9, 0.999, 1e-8, t, C.byref(st)))
    return st


def _run(mode, steps=3):
    n = 1000
    g = api.random_regular_graph(n, 3, 0)
    m = api.made_init(n, api.default_made_hidden(n), 0)
    dev = api.DeviceReplica(m, 0, 256)
    dev.set_problem(api.maxcut_spec(g))
    K.check(K.lib.vqmc_gpu_set_phase_timing(dev.h, 1 if mode else 0))
    K.check(K.lib.vqmc_gpu_set_kernel_timing(dev.h, mode))
    for t in range(1, steps + 1):
        _step(dev, t)
    p = np.empty(len(m.parameters()))
    K.check(K.lib.vqmc_gpu_get_params(dev.h, K.ptr(p)))
    return dev, p


def test_timeline_reports_the_concurrent_schedule():
    dev, _ = _run(2)
    names = C.create_string_buffer(32 * 128)
    s, e = (C.c_float * 128)(), (C.c_float * 128)()
    cnt = C.c_int()
    K.check(K.lib.vqmc_gpu_kernel_timeline(dev.h, names, s, e, 128, C.byref(cnt)))
    got = [names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode() for i in range(cnt.value)]
    for k in ("head_sample", "z2_tail_umma", "maxcut_energy", "bw_gw2_umma", "bw_dg1_umma", "adam_w2", "adam_w1"):
        assert k in got, (k, got)
    span = {k: (s[i], e[i]) for i, k in enumerate(got)}
    assert all(0.0 <= a <= b for a, b in span.values())
    # the side stream's gW2 overlaps the main stream's dg1 (concurrent schedule, not the serial one)
    g0, g1 = span["bw_gw2_umma"]
    d0, d1 = span["bw_dg1_umma"]
    assert g0 < d1 and d0 < g1
    assert span["head_sample"][1] <= span["z2_tail_umma"][1] <= span["maxcut_energy"][1]


def test_timing_modes_do_not_change_the_step():
    _, p0 = _run(0)
    _, p1 = _run(1)
    _, p2 = _run(2)
    assert np.array_equal(p0, p2)  # same schedule, events only
    assert np.array_equal(p0, p1)  # serial backward: the same partial sums in the same order


def test_timeline_needs_the_step_start_event():
    n = 100
    g = api.random_regular_graph(n, 3, 0)
    m = api.made_init(n, api.default_made_hidden(n), 0)
    dev = api.DeviceReplica(m, 0, 64)
    dev.set_problem(api.maxcut_spec(g))
    K.check(K.lib.vqmc_gpu_set_kernel_timing(dev.h, 2))
    names = C.create_string_buffer(32 * 4)
    s, e = (C.c_float * 4)(), (C.c_float * 4)()
    cnt = C.c_int()
    with pytest.raises(ValueError, match="phase timing"):
        K.check(K.lib.vqmc_gpu_kernel_timeline(dev.h, names, s, e, 4, C.byref(cnt)))
