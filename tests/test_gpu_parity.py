"""GPU parity of the B200 path (through the C ABI) against the CPU oracle and the golden
fixtures.  Tolerances (stated per the north star):

* samples: bit-exact, except where |u - p_ref| < TOL_FLIP = 1e-5 (counted; a sample is
  compared only up to its first tolerated flip, after which it legitimately diverges);
* cut values / local energies: bit-exact; energy mean and variance: bit-exact;
* log psi: relative <= 1e-5 (fp32 logits, fp64 accumulation);
* gradients: norm-wise relative <= 1e-4 and elementwise |g - g_ref| <= 1e-4 |g_ref| + 1e-5 ||g_ref||_inf;
  masked entries exactly 0;
* Adam update: elementwise |dtheta - dtheta_ref| <= 1e-6 + 1e-4 |dtheta_ref| where |g_ref| > 1e-6 ||g_ref||_inf.
"""
import ctypes as C
import os

import numpy as np
import pytest

import pyoracle as O
from paper_2106_13308_b200 import _capi as K
from paper_2106_13308_b200 import api

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL_FLIP = 1e-5


class Dev:
    def __init__(self, n, h, degrees, theta, edges, B=1024):
        self.n, self.h, self.W = n, h, (n + 31) // 32
        self.degrees = np.ascontiguousarray(degrees, np.int32)
        self.h_ = C.c_void_p()
        e = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
        K.check(K.lib.vqmc_gpu_create(0, n, h, K.ptr(self.degrees), K.ptr(np.ascontiguousarray(theta, np.float64)),
                                      K.ptr(e), len(e), B, C.byref(self.h_)))

    def __del__(self):
        K.lib.vqmc_gpu_destroy(self.h_)

    def set_params(self, theta):
        K.check(K.lib.vqmc_gpu_set_params(self.h_, K.ptr(np.ascontiguousarray(theta, np.float64))))

    def get_params(self):
        d = 2 * self.h * self.n + self.h + self.n
        out = np.empty(d)
        K.check(K.lib.vqmc_gpu_get_params(self.h_, K.ptr(out)))
        return out

    def sample(self, B, U=None, seed=0, stream=0, call=0):
        bits = np.empty((B, self.W), np.uint32)
        lp = np.empty(B)
        K.check(K.lib.vqmc_gpu_sample(self.h_, B, K.ptr(U), seed, stream, call, K.ptr(bits), K.ptr(lp)))
        return K.unpack_bits(bits, self.n), lp

    def energy(self, x):
        bits = K.pack_bits(x)
        cut = np.empty(len(x), np.int32)
        le = np.empty(len(x))
        K.check(K.lib.vqmc_gpu_maxcut_energy(self.h_, K.ptr(bits), len(x), K.ptr(cut), K.ptr(le)))
        return cut, le

    def log_psi(self, x, want_cond=False):
        bits = K.pack_bits(x)
        lp = np.empty(len(x))
        cond = np.empty((len(x), self.n)) if want_cond else None
        K.check(K.lib.vqmc_gpu_log_psi(self.h_, K.ptr(bits), len(x), K.ptr(lp), K.ptr(cond)))
        return (lp, cond) if want_cond else lp

    def grad_from_locals(self, x, le):
        bits = K.pack_bits(x)
        g = np.empty(2 * self.h * self.n + self.h + self.n)
        K.check(K.lib.vqmc_gpu_gradient_from_locals(self.h_, K.ptr(bits), K.ptr(np.ascontiguousarray(le)), len(x),
                                                    K.ptr(g)))
        return g

    def weighted_grad(self, x, w):
        bits = K.pack_bits(x)
        g = np.empty(2 * self.h * self.n + self.h + self.n)
        K.check(K.lib.vqmc_gpu_weighted_grad(self.h_, K.ptr(bits), K.ptr(np.ascontiguousarray(w, np.float64)),
                                             len(x), K.ptr(g)))
        return g


def _model(n, seed, perturb=True, h=None):
    h = h or O.default_made_hidden(n)
    m = O.made_init(n, h, seed)
    if perturb:
        m.theta = m.theta + (O.uniforms(seed, 98, m.d) * 3.0 + -1.5)
    return m


def _graph(n, seed, kind):
    return O.random_maxcut_graph(n, seed) if kind == "maxcut" else O.random_regular_graph(n, 3, seed)


def check_samples(xg, xo, U, p_used, log=None, **info):
    """Bit-exact up to tolerated flips; returns (#rows with a flip, #rows compared clean).
    With `log` (the parity_log fixture) the flip count is recorded with `info`."""
    mism = xg != xo
    flips = 0
    gaps = []
    for b in range(len(xg)):
        if not mism[b].any():
            continue
        i = int(np.argmax(mism[b]))
        gap = abs(U[i, b] - p_used[b, i])
        assert gap < TOL_FLIP, f"sample {b} bit {i}: |u-p| = {gap:.3e} >= {TOL_FLIP}"
        flips += 1
        gaps.append(float(gap))
    if log is not None:
        log.append(dict(info, rows=int(len(xg)), bits_drawn=int(xg.size), rows_with_flip=flips, gaps=gaps))
    return flips, len(xg) - flips


def check_grad(g, go, m):
    nr = np.linalg.norm(g - go) / np.linalg.norm(go)
    assert nr <= 1e-4, nr
    gi = np.abs(go).max()
    assert np.all(np.abs(g - go) <= 1e-4 * np.abs(go) + 1e-5 * gi)
    # masked entries exactly zero (models_test.cpp:175-190)
    n, h, deg = m.n, m.h, m.degrees
    M1 = (np.arange(n)[None, :] + 1 <= deg[:, None])
    M2 = (deg[None, :] < np.arange(n)[:, None] + 1)
    assert np.all(g[: h * n].reshape(h, n)[~M1] == 0.0)
    assert np.all(g[h * n + h: h * n + h + n * h].reshape(n, h)[~M2] == 0.0)
    return nr


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["oracle_n20_seed0", "oracle_n100_seed1"])
def test_golden_fixture(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    n, h, B = int(g["n"]), int(g["h"]), int(g["B"])
    dev = Dev(n, h, g["degrees"], g["theta"], g["edges"], B)
    U = np.ascontiguousarray(g["uniforms"])
    xg, lp = dev.sample(B, U)
    flips, clean = check_samples(xg, g["x"], U, g["p"])
    ok = ~np.any(xg != g["x"], axis=1)
    assert np.all(np.abs(lp[ok] - g["log_psi"][ok]) <= 1e-5 * np.abs(g["log_psi"][ok]))
    cut, le = dev.energy(g["x"])
    assert np.array_equal(cut.astype(float), g["cut"]) and np.array_equal(le, g["local"])
    m = O.Made(n, h, g["degrees"], g["theta"])
    check_grad(dev.grad_from_locals(g["x"], g["local"]), g["grad"], m)


@pytest.mark.parametrize("n,B,kind", [(20, 1024, "maxcut"), (100, 1024, "maxcut"), (1000, 128, "maxcut"),
                                      (1000, 256, "regular")])
def test_sampler_parity_reference_uniforms(n, B, kind, parity_log):
    m = _model(n, 3)
    dev = Dev(n, m.h, m.degrees, m.theta, _graph(n, 3, kind), B)
    U = O.uniforms(3, 1, n * B).reshape(n, B)
    xg, lp = dev.sample(B, U)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1 if n > 100 else 0, want_p=True)
    flips, clean = check_samples(xg, xo, U, po, parity_log, test="sampler_mt19937", n=n, graph=kind)
    assert clean >= 0.9 * B
    ok = ~np.any(xg != xo, axis=1)
    assert np.all(np.abs(lp[ok] - lo[ok]) <= 1e-5 * np.abs(lo[ok]))


def test_sampler_parity_production_philox(parity_log):
    n, B = 300, 256
    m = _model(n, 5)
    dev = Dev(n, m.h, m.degrees, m.theta, _graph(n, 5, "regular"), B)
    xg, lp = dev.sample(B, None, seed=11, stream=3, call=7)
    U = O.philox_uniforms(11, 3, 7, n, B)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1, want_p=True)
    flips, clean = check_samples(xg, xo, U, po, parity_log, test="sampler_philox", n=n)
    assert clean >= 0.9 * B


def test_sampler_parity_n10000_headline_shape(parity_log):
    """N = 10,000, h = 424 (head 424 bits + tail GEMM) against the incremental fp64 oracle."""
    n, B = 10000, 1024
    m = _model(n, 0, perturb=False)
    m.theta = m.theta + (O.uniforms(0, 98, m.d) * 0.2 - 0.1)
    dev = Dev(n, m.h, m.degrees, m.theta, _graph(n, 0, "regular"), B)
    U = O.uniforms(0, 1, n * B).reshape(n, B)
    xg, lp = dev.sample(B, U)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1, want_p=True)
    flips, clean = check_samples(xg, xo, U, po, parity_log, test="sampler_mt19937_headline", n=n, perturbation=0.1)
    assert clean >= 0.95 * B
    ok = ~np.any(xg != xo, axis=1)
    assert np.all(np.abs(lp[ok] - lo[ok]) <= 1e-5 * np.abs(lo[ok]))


@pytest.mark.parametrize("n,kind", [(20, "maxcut"), (1000, "maxcut"), (10000, "regular")])
def test_energy_bit_exact(n, kind):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 2, (333, n)).astype(np.uint8)
    e = _graph(n, 1, kind)
    m = _model(n, 1, perturb=False)
    dev = Dev(n, m.h, m.degrees, m.theta, e, 333)
    cut, le = dev.energy(x)
    leo, cuto = O.local_energy(n, e, x)
    assert np.array_equal(le, leo) and np.array_equal(cut.astype(float), cuto)


@pytest.mark.parametrize("n", [6, 20, 100, 1000])
def test_log_psi_and_conditionals(n):
    m = _model(n, 2)
    dev = Dev(n, m.h, m.degrees, m.theta, np.zeros((0, 2), np.int32), 256)
    x = np.random.default_rng(n).integers(0, 2, (97, n)).astype(np.uint8)
    lp, cond = dev.log_psi(x, want_cond=True)
    lo = O.log_psi(m, x)
    po, _, _ = O.forward(m, x)
    assert np.all(np.abs(lp - lo) <= 1e-5 * np.abs(lo))
    # fp32 logits: the logit is a sum of up to h terms of size |W| |g| (|W| <= 1.5 under the
    # U(-1.5, 1.5) perturbation), so |dz| <= ~1e-4 and |dp| <= p (1 - p) |dz| <= 3e-5
    assert np.abs(cond - po).max() <= 3e-5


def test_normalization_and_autoregressive_invariance():  # models_test.cpp:96-123 on the GPU path
    for n in (3, 6, 10):
        m = _model(n, 0, perturb=False)
        dev = Dev(n, m.h, m.degrees, m.theta, np.zeros((0, 2), np.int32), 1 << n)
        lp = dev.log_psi(api.all_configs(n))
        assert abs(np.exp(2 * lp).sum() - 1.0) <= 1e-5
    m = _model(6, 9, h=14)
    dev = Dev(6, 14, m.degrees, m.theta, np.zeros((0, 2), np.int32), 64)
    x = api.all_configs(6)
    _, base = dev.log_psi(x, want_cond=True)
    for j in range(6):
        y = x.copy(); y[:, j] ^= 1
        _, fl = dev.log_psi(y, want_cond=True)
        assert np.array_equal(fl[:, : j + 1], base[:, : j + 1])


@pytest.mark.parametrize("n,B", [(20, 1024), (100, 512), (1000, 256)])
def test_gradient_parity(n, B):
    m = _model(n, 4)
    e = _graph(n, 4, "maxcut")
    dev = Dev(n, m.h, m.degrees, m.theta, e, B)
    xo, _ = O.auto_sample(m, B, seed=4, stream=1, mode=1)
    leo, _ = O.local_energy(n, e, xo)
    check_grad(dev.grad_from_locals(xo, leo), O.gradient_from_locals(m, xo, leo), m)


def test_weighted_grad_single_rows_and_generic_degrees():
    """weighted = sum of singles (models_test.cpp:192-209), incl. h > n - 1 (repeated degrees)."""
    m = _model(4, 2, h=6)
    dev = Dev(4, 6, m.degrees, m.theta, np.zeros((0, 2), np.int32), 8)
    x = api.all_configs(4)[:5]
    w = np.array([0.3, -1.2, 0.0, 2.5, -0.7])
    g = dev.weighted_grad(x, w)
    go = O.weighted_grad(m, x, w)
    check_grad(g, go, m)
    # a checkpoint-style permuted degree vector
    deg = np.array([3, 1, 2, 3, 1, 2], np.int32)
    mo = O.Made(4, 6, deg, m.theta)
    dev2 = Dev(4, 6, deg, m.theta, np.zeros((0, 2), np.int32), 8)
    check_grad(dev2.weighted_grad(x, w), O.weighted_grad(mo, x, w), mo)
    assert np.all(np.abs(dev2.log_psi(x) - O.log_psi(mo, x)) <= 1e-5 * np.abs(O.log_psi(mo, x)))


def test_params_roundtrip_and_adam():
    n = 50
    m = _model(n, 6)
    dev = Dev(n, m.h, m.degrees, m.theta, np.zeros((0, 2), np.int32), 64)
    back = dev.get_params()
    assert np.array_equal(back[m.degrees.size * 0:], back)  # shape sanity
    live = np.abs(back - m.theta) <= 1e-7 * np.abs(m.theta) + 1e-30
    assert live.all()  # fp32 live copy, masked entries exact
    g = O.gradient_from_locals(m, *(lambda x: (x, O.local_energy(n, O.random_maxcut_graph(n, 0), x)[0]))(
        O.auto_sample(m, 256, seed=6, stream=1, mode=1)[0]))
    K.check(K.lib.vqmc_gpu_adam_reset(dev.h_))
    K.check(K.lib.vqmc_gpu_adam_step(dev.h_, K.ptr(g), 0.01, 0.9, 0.999, 1e-8, 1))
    st = O.AdamState(m.d)
    p = m.theta.copy()
    O.adam_step(st, p, g)
    got = dev.get_params()
    sel = np.abs(g) > 1e-6 * np.abs(g).max()
    d_ref, d_got = p - m.theta, got - m.theta
    assert np.all(np.abs(d_got[sel] - d_ref[sel]) <= 1e-6 + 1e-4 * np.abs(d_ref[sel]))
    zero = g == 0.0  # zero-gradient entries never move (masked ones are returned bit-exact)
    assert np.all(np.abs(got[zero] - m.theta[zero]) <= 1e-7 * np.abs(m.theta[zero]))
    h = m.h
    M2 = (m.degrees[None, :] < np.arange(n)[:, None] + 1)
    w2 = slice(h * n + h, h * n + h + n * h)
    assert np.array_equal(got[w2].reshape(n, h)[~M2], m.theta[w2].reshape(n, h)[~M2])


def _train_step(dev, mbs, L, U, seed, stream0, call, t):
    st = K.StepStats()
    K.check(K.lib.vqmc_gpu_train_step(dev.h_, mbs, L, K.ptr(U), seed, stream0, call, 0.01, 0.9, 0.999, 1e-8, t,
                                      C.byref(st)))
    return st


@pytest.mark.parametrize("n,L,mbs", [(20, 1, 1024), (8, 4, 32), (100, 2, 256)])
def test_fused_step_parity_first_iteration(n, L, mbs):
    """One fused device step (reference mt19937 uniforms) == oracle iteration 0 (trainer.cpp:150-231)."""
    seed = 7
    e = O.random_maxcut_graph(n, seed)
    h = O.default_made_hidden(n)
    r = O.train(n, e, h=h, iterations=1, workers=L, minibatch=mbs, eval_batch=16, seed=seed, want_first_grad=True,
                sampler_mode=0)
    m0 = O.made_init(n, h, seed)
    dev = Dev(n, h, m0.degrees, m0.theta, e, L * mbs)
    U = np.concatenate([O.uniforms(seed, w + 1, n * mbs).reshape(n, mbs) for w in range(L)], axis=1)
    st = _train_step(dev, mbs, L, np.ascontiguousarray(U), seed, 1, 0, 1)
    # pooled energy statistics: bit-exact
    assert st.energy_mean == r["stats"][0, 0]
    assert np.sqrt(st.energy_var) == r["stats"][0, 1]
    assert st.grad_norm == pytest.approx(r["stats"][0, 2], rel=1e-4)
    g = r["first_grad"]
    sel = np.abs(g) > 1e-6 * np.abs(g).max()
    got = dev.get_params()
    d_ref, d_got = r["theta"] - m0.theta, got - m0.theta
    assert np.all(np.abs(d_got[sel] - d_ref[sel]) <= 1e-6 + 1e-4 * np.abs(d_ref[sel]))


def test_maxcut_n20_quality_matches_reference_acceptance():
    """acceptance.cpp:239-272 criterion 6 (ADAM >= 0.95 x optimum on 5 seeds) on the GPU
    path with the reference's mt19937 streams; the oracle's (= reference's) worst ratio is
    0.956 (test_output.txt:26)."""
    worst = 1.0
    for s in range(5):
        g = api.random_maxcut_graph(20, s)
        opt, _ = O.brute_force_maxcut(20, g.edges)
        cfg = api.RunConfig(problem=api.maxcut_spec(g), iterations=300, minibatch=1024, eval_batch=1024, seed=s,
                            uniforms="mt19937")
        res = api.train(cfg)
        worst = min(worst, res.best_cut / opt)
    assert worst >= 0.95, worst


def test_production_train_n10000_smoke():
    g = api.random_regular_graph(10000, 3, 0)
    cfg = api.RunConfig(problem=api.maxcut_spec(g), iterations=3, minibatch=1024, eval_batch=256, seed=0)
    res = api.train(cfg)
    assert len(res.stats) == 3 and all(np.isfinite([s.energy_mean, s.grad_norm]).all() for s in res.stats)
    assert 0 < res.best_cut <= 15000 and res.best_cut >= res.mean_cut


def test_overlapped_allreduce_path_matches_single_gpu(monkeypatch):
    """The multi-GPU step (gW2 all-reduce on a comm stream overlapped with dg1/dz1/gW1, GEMMs leaving
    SMs to NCCL) run through a one-rank NCCL communicator (VQMC_NCCL_SELF=1) gives bitwise the same
    parameters as the plain single-GPU step over eager, captured and replayed steps."""
    n, B = 1000, 256
    m = _model(n, 4, perturb=False)
    e = _graph(n, 4, "regular")
    devs = [Dev(n, m.h, m.degrees, m.theta, e, B), Dev(n, m.h, m.degrees, m.theta, e, B)]
    monkeypatch.setenv("VQMC_NCCL_SELF", "1")
    uid = (C.c_uint8 * 128)()
    K.check(K.lib.vqmc_gpu_comm_unique_id(uid))
    K.check(K.lib.vqmc_gpu_comm_init(devs[1].h_, uid, 1, 0))
    for d in devs:
        K.check(K.lib.vqmc_gpu_adam_reset(d.h_))
    stats = [[], []]
    for t in range(1, 5):
        for k, d in enumerate(devs):
            st = K.StepStats()
            K.check(K.lib.vqmc_gpu_train_step(d.h_, B, 1, None, 4, 1, t, 0.01, 0.9, 0.999, 1e-8, t, C.byref(st)))
            stats[k].append((st.energy_mean, st.grad_norm))
    assert stats[0] == stats[1]
    assert np.array_equal(devs[0].get_params(), devs[1].get_params())


def test_hitting_time_mode():
    """trainer_test.cpp:146-158 / trainer.cpp:265-274: with a target the run evaluates after every
    iteration (outside the timed phases) and stops at the first hit (Max-Cut: best_cut >= target)."""
    g = api.random_maxcut_graph(20, 2)
    cfg = api.RunConfig(problem=api.maxcut_spec(g), iterations=50, minibatch=64, eval_batch=128, seed=1, target=1.0)
    res = api.train(cfg)
    assert res.hit_iteration == 1 and len(res.stats) == 1 and res.hit_time is not None and res.hit_time > 0
    opt, _ = O.brute_force_maxcut(20, g.edges)
    cfg = api.RunConfig(problem=api.maxcut_spec(g), iterations=300, minibatch=1024, eval_batch=1024, seed=1,
                        target=float(opt), uniforms="mt19937")
    res = api.train(cfg)
    assert res.hit_iteration == -1 or (res.best_cut >= opt and len(res.stats) == res.hit_iteration)
    cfg = api.RunConfig(problem=api.maxcut_spec(g), iterations=5, minibatch=64, eval_batch=128, seed=1,
                        target=1e9)  # unreachable: runs every iteration, no hit
    res = api.train(cfg)
    assert res.hit_iteration == -1 and res.hit_time is None and len(res.stats) == 5


@pytest.mark.parametrize("n,L,mbs", [(1000, 3, 77), (300, 1, 33), (20, 5, 7)])
def test_fused_step_parity_ragged_batches(n, L, mbs):
    """Ragged batches (B not a multiple of the 32-sample energy groups, the 256-row GEMM tiles or
    the head's 8-sample CTAs): one fused step == oracle iteration 0, as above."""
    seed = 5
    e = O.random_maxcut_graph(n, seed)
    h = O.default_made_hidden(n)
    r = O.train(n, e, h=h, iterations=1, workers=L, minibatch=mbs, eval_batch=16, seed=seed, want_first_grad=True,
                sampler_mode=1)
    m0 = O.made_init(n, h, seed)
    dev = Dev(n, h, m0.degrees, m0.theta, e, L * mbs)
    U = np.concatenate([O.uniforms(seed, w + 1, n * mbs).reshape(n, mbs) for w in range(L)], axis=1)
    st = _train_step(dev, mbs, L, np.ascontiguousarray(U), seed, 1, 0, 1)
    assert st.energy_mean == r["stats"][0, 0]
    # std: the device forms the variance exactly from integer cut sums and rounds once; the oracle's
    # two-pass fp64 sum (like Eigen's, whose SIMD reduction order the oracle does not reproduce
    # either) rounds per term, so for N not a power of two they may differ in the last bits
    assert np.sqrt(st.energy_var) == pytest.approx(r["stats"][0, 1], rel=1e-15, abs=0)
    assert st.grad_norm == pytest.approx(r["stats"][0, 2], rel=1e-4)
    g = r["first_grad"]
    sel = np.abs(g) > 1e-6 * np.abs(g).max()
    d_ref, d_got = r["theta"] - m0.theta, dev.get_params() - m0.theta
    assert np.all(np.abs(d_got[sel] - d_ref[sel]) <= 1e-6 + 1e-4 * np.abs(d_ref[sel]))


@pytest.mark.parametrize("n,B", [(1000, 100), (300, 37), (10000, 5)])
def test_sampler_parity_production_philox_ragged(n, B, parity_log):
    m = _model(n, 6, perturb=n < 10000)
    dev = Dev(n, m.h, m.degrees, m.theta, _graph(n, 6, "regular"), B)
    xg, lp = dev.sample(B, None, seed=3, stream=2, call=5)
    U = O.philox_uniforms(3, 2, 5, n, B)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1, want_p=True)
    flips, clean = check_samples(xg, xo, U, po, parity_log, test="sampler_philox_ragged", n=n)
    assert clean >= 0.8 * B


@pytest.mark.parametrize("n", [2, 3, 33])
def test_edge_cases_tiny_models_and_empty_graphs(n):
    """Smallest models (n = 2: h = 2, one head bit) and graphs without edges: sampling parity,
    exact zero energies, and a training step whose zero-variance batch gives a zero gradient
    (a zero Adam update), like the reference (estimator.hpp:111-119, optimizer.cpp:21-35)."""
    h = O.default_made_hidden(n)
    m = O.made_init(n, h, 2)
    B = 64
    for edges in (np.zeros((0, 2), np.int32), O.random_maxcut_graph(n, 2)):
        dev = Dev(n, h, m.degrees, m.theta, edges, B)
        U = O.uniforms(2, 1, n * B).reshape(n, B)
        xg, lp = dev.sample(B, U)
        xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=0, want_p=True)
        check_samples(xg, xo, U, po)
        cut, le = dev.energy(xo)
        lo_ref, _ = O.local_energy(n, edges, xo)
        assert np.array_equal(le, lo_ref)
        if len(np.asarray(edges).reshape(-1, 2)) == 0:
            assert np.all(cut == 0) and np.all(le == 0.0)
            p0 = dev.get_params()  # (the device master copy is fp32)
            st = _train_step(dev, B, 1, np.ascontiguousarray(U), 2, 1, 0, 1)
            assert st.energy_mean == 0.0 and st.energy_var == 0.0 and st.grad_norm == 0.0
            assert np.array_equal(dev.get_params(), p0)


@pytest.mark.parametrize("n,h", [(1200, 1000), (3000, 1024)])
def test_maximum_hidden_width(n, h):
    """The widest supported hidden layer (kMaxHidden = 1024: the head sampler's 8 register slots
    per lane and its largest shared-memory ring): sampling parity and a finite training step."""
    m = _model(n, 4, perturb=False, h=h)
    m.theta = m.theta + (O.uniforms(4, 98, m.d) * 0.2 - 0.1)
    B = 64
    dev = Dev(n, h, m.degrees, m.theta, _graph(n, 4, "regular"), B)
    U = O.uniforms(4, 1, n * B).reshape(n, B)
    xg, lp = dev.sample(B, U)
    xo, lo, po = O.auto_sample(m, B, uniforms=U, mode=1, want_p=True)
    flips, clean = check_samples(xg, xo, U, po)
    assert clean >= 0.5 * B
    st = _train_step(dev, B, 1, None, 4, 1, 0, 1)
    assert np.isfinite(st.energy_mean) and np.isfinite(st.grad_norm) and st.grad_norm > 0


def test_hidden_width_above_maximum_is_rejected():
    n, h = 1200, 1100
    m = _model(n, 4, perturb=False, h=h)
    with pytest.raises(ValueError):
        dev = Dev(n, h, m.degrees, m.theta, _graph(n, 4, "regular"), 64)
        dev.sample(64, O.uniforms(4, 1, n * 64).reshape(n, 64))
