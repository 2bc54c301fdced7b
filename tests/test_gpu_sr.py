"""SR (stochastic reconfiguration) on the GPU against the oracle's restatement of
score_matrix (models.cpp:221-244), FisherEstimate (estimator.hpp:146-168) and sr_direction
(optimizer.cpp:36-92), plus the reference's SR tests (optimizer_test.cpp:64-150) and acceptance
criterion 6's SR half (acceptance.cpp:246-262; recorded "sr optimal 5/5", test_output.txt:26).

Tolerance: the GPU applies F through fp32-grade GEMMs (fp16 pairs) and runs the reference's CG in
fp64 to the same relative-residual contract (tol 1e-6), so the direction matches the oracle's
exact (LDLT, d <= 2000) or fp64-CG solution to within the CG tolerance amplified by the
conditioning: relative norm error <= 2e-3 (observed ~1e-4); masked entries exactly 0.
"""
import ctypes as C

import numpy as np
import pytest

import pyoracle as O
from paper_2106_13308_b200 import _capi as K
from paper_2106_13308_b200 import api

pytestmark = pytest.mark.gpu


def _setup(n, B, seed):
    h = O.default_made_hidden(n)
    m = O.made_init(n, h, seed)
    r = O.auto_sample(m, B, seed=seed, stream=1, mode=1)
    x = np.ascontiguousarray(r[0] if isinstance(r, tuple) else r, np.uint8)
    e = O.random_maxcut_graph(n, seed)
    g = O.gradient_from_locals(m, x, O.local_energy(n, e, x)[0])
    return m, e, x, g


def _gpu_direction(m, e, x, g, lam=1e-3, tol=1e-6, max_it=200, centered=True):
    model = api.MadeModel(m.n, m.h, m.degrees, m.theta)
    fisher = api.fisher_estimate(model, x, centered)
    info = {}
    d = api.sr_direction(api.SrConfig(lam=lam, tol=tol, max_iterations=max_it, centered=centered), g, fisher, info)
    return d, info


def _masks(m):
    n, h, deg = m.n, m.h, m.degrees
    M1 = (np.arange(n)[None, :] + 1 <= deg[:, None])
    M2 = (deg[None, :] < np.arange(n)[:, None] + 1)
    return M1, M2


@pytest.mark.parametrize("n,B,seed", [(20, 256, 0), (100, 256, 3), (100, 1024, 1)])
def test_sr_direction_matches_oracle(n, B, seed):
    m, e, x, g = _setup(n, B, seed)
    S = O.score_matrix(m, x)
    d_ref, it_ref, _ = O.sr_direction(S, g, lam=1e-3, tol=1e-6, max_iterations=200)
    d_gpu, info = _gpu_direction(m, e, x, g)
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    assert rel <= 2e-3, (rel, info, it_ref)
    assert info["residual"] <= 1e-6
    if m.d <= 2000:  # optimizer.cpp:66-73: exact dense solve, no CG iterations
        assert info["iterations"] == 0 and rel <= 1e-4, rel  # (fp32-grade score entries)
    else:
        assert 0 < info["iterations"] <= 200
    # the accepted solution satisfies the reference's residual contract in fp64 (oracle operator)
    Sc = S - S.mean(0)
    resid = Sc.T @ (Sc @ d_gpu) / B + 1e-3 * d_gpu - g
    assert np.linalg.norm(resid) <= 5e-3 * np.linalg.norm(g)
    M1, M2 = _masks(m)
    h = m.h
    assert np.all(d_gpu[: h * n].reshape(h, n)[~M1] == 0.0)
    assert np.all(d_gpu[h * n + h: h * n + h + n * h].reshape(n, h)[~M2] == 0.0)


def test_sr_uncentered_matches_oracle():
    m, e, x, g = _setup(100, 256, 5)
    S = O.score_matrix(m, x)
    d_ref, _, _ = O.sr_direction(S, g, lam=1e-3, centered=False)
    d_gpu, _ = _gpu_direction(m, e, x, g, centered=False)
    assert np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref) <= 2e-3


def test_sr_large_lambda_is_scaled_gradient():
    """optimizer_test.cpp:85-106: as lambda grows the direction turns into grad / lambda."""
    m, e, x, g = _setup(100, 256, 2)
    prev = 1e9
    for lam in (0.01, 1.0, 100.0, 10000.0):
        d, _ = _gpu_direction(m, e, x, g, lam=lam)
        ang = np.arccos(np.clip(d @ g / (np.linalg.norm(d) * np.linalg.norm(g)), -1.0, 1.0))
        assert ang <= prev + 1e-6
        prev = ang
    assert np.linalg.norm(d * 10000.0 - g) <= 1e-2 * np.linalg.norm(g)


def test_sr_cg_failure_raises():
    """optimizer_test.cpp:129-142: zero iterations cannot converge -> SrSolveError."""
    m, e, x, g = _setup(100, 256, 4)
    with pytest.raises(api.SrSolveError):
        _gpu_direction(m, e, x, g, max_it=0)
    model = api.MadeModel(m.n, m.h, m.degrees, m.theta)
    fisher = api.fisher_estimate(model, x)
    cfg = api.SrConfig(max_iterations=0, fallback=True)
    out = api.sr_step(cfg, np.zeros(m.d), g, fisher)  # fallback: the raw gradient step
    assert np.array_equal(out, -cfg.lr * g)


def test_sr_zero_gradient_is_zero_direction():
    m, e, x, g = _setup(20, 64, 0)
    d, info = _gpu_direction(m, e, x, np.zeros_like(g))
    assert np.all(d == 0.0) and info["iterations"] == 0


def test_sr_train_step_first_iteration_matches_oracle():
    """One SGD + SR iteration with the reference's streams (trainer.cpp:150-282): pooled energy
    statistics bit-exact, the parameter update lr * delta within the SR tolerance."""
    n, mbs, L, seed = 20, 128, 2, 3
    g = api.random_maxcut_graph(n, seed)
    r = O.train(n, g.edges, optimizer="sgd_sr", iterations=1, workers=L, minibatch=mbs, eval_batch=64, seed=seed,
                sampler_mode=1)
    cfg = api.RunConfig(problem=api.maxcut_spec(g), optimizer="sgd_sr", iterations=1, workers=L, minibatch=mbs,
                        eval_batch=64, seed=seed, uniforms="mt19937")
    res = api.train(cfg)
    assert res.stats[0].energy_mean == r["stats"][0, 0]
    assert res.stats[0].energy_std == r["stats"][0, 1]
    assert abs(res.stats[0].grad_norm - r["stats"][0, 2]) <= 1e-4 * r["stats"][0, 2]
    m0 = O.made_init(n, O.default_made_hidden(n), seed)
    d_ref, d_got = r["theta"] - m0.theta, res.final_params - m0.theta
    assert np.linalg.norm(d_got - d_ref) <= 2e-3 * np.linalg.norm(d_ref)


def test_maxcut_n20_sr_quality_matches_reference_acceptance():
    """acceptance.cpp:246-262 criterion 6, SR half: SGD + SR (150 iterations, minibatch 256)
    reaches the brute-force optimum; the reference's recorded run: 5/5 optimal, worst ratio 1.000
    (test_output.txt:26).  Criterion: >= 3/5 optimal and all >= 0.97 of the optimum."""
    optimal, worst = 0, 1.0
    for s in range(5):
        g = api.random_maxcut_graph(20, s)
        opt, _ = O.brute_force_maxcut(20, g.edges)
        cfg = api.RunConfig(problem=api.maxcut_spec(g), optimizer="sgd_sr", iterations=150, minibatch=256,
                            eval_batch=1024, seed=s, uniforms="mt19937")
        res = api.train(cfg)
        optimal += res.best_cut >= opt
        worst = min(worst, res.best_cut / opt)
    assert optimal >= 3 and worst >= 0.97, (optimal, worst)


def test_sr_dense_scores_match_oracle_score_matrix():
    """The small-model path's explicit score rows (fp32-grade D, G1, dz1 widened to fp64) against
    score_matrix (models.cpp:221-244) in the reference flatten order."""
    m, e, x, g = _setup(20, 128, 2)
    model = api.MadeModel(m.n, m.h, m.degrees, m.theta)
    out = np.empty((len(x), m.d))
    K.lib.vqmc_test_sr_scores.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    K.check(K.lib.vqmc_test_sr_scores(model.device().h, K.ptr(K.pack_bits(x)), len(x), K.ptr(out)))
    S = O.score_matrix(m, x)
    assert np.abs(out - S).max() <= 1e-5 * max(1.0, np.abs(S).max())
    assert np.all(out[S == 0.0] == 0.0)


@pytest.mark.parametrize("mdim", [1, 37, 300])
def test_sr_dense_cholesky(mdim):
    f = K.lib.vqmc_test_sr_chol
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(mdim)
    M = rng.standard_normal((mdim, mdim + 3))
    A = np.ascontiguousarray(M @ M.T + 0.1 * np.eye(mdim))
    b = rng.standard_normal(mdim)
    x = np.empty(mdim)
    assert f(mdim, K.ptr(A), K.ptr(b), K.ptr(x)) == 0
    assert np.abs(x - np.linalg.solve(A, b)).max() <= 1e-9 * np.abs(np.linalg.solve(A, b)).max()
    A[0, 0] = -1.0  # not positive definite -> flagged
    assert f(mdim, K.ptr(A), K.ptr(b), K.ptr(x)) == 1


def test_sr_step_through_nccl_matches_single_gpu(monkeypatch):
    """The multi-GPU SR step (gradient, q-sum and F p all-reduced over the ranks' NCCL communicator
    inside every CG iteration) run through a one-rank communicator (VQMC_NCCL_SELF=1) gives bitwise
    the single-GPU result over three SGD + SR steps (CG path, d > 2000)."""
    n, B = 100, 256
    h = O.default_made_hidden(n)
    m = O.made_init(n, h, 7)
    e = np.ascontiguousarray(O.random_maxcut_graph(n, 7), np.int32).reshape(-1, 2)
    monkeypatch.setenv("VQMC_NCCL_SELF", "1")
    hs = []
    for _ in range(2):
        hd = C.c_void_p()
        K.check(K.lib.vqmc_gpu_create(0, n, h, K.ptr(m.degrees), K.ptr(m.theta), K.ptr(e), len(e), B, C.byref(hd)))
        hs.append(hd)
    uid = (C.c_uint8 * 128)()
    K.check(K.lib.vqmc_gpu_comm_unique_id(uid))
    K.check(K.lib.vqmc_gpu_comm_init(hs[1], uid, 1, 0))
    out = [[], []]
    try:
        for t in range(3):
            for k, hd in enumerate(hs):
                st, it, res = K.StepStats(), C.c_int(0), C.c_double(0.0)
                K.check(K.lib.vqmc_gpu_train_step_sr(hd, B, 1, None, 7, 1, t, 0.1, 1e-3, 1e-6, 200, 0, 1, C.byref(st),
                                                     C.byref(it), C.byref(res)))
                out[k].append((st.energy_mean, st.grad_norm, it.value, res.value))
        assert out[0] == out[1]
        d = 2 * h * n + h + n
        th = [np.empty(d), np.empty(d)]
        for k, hd in enumerate(hs):
            K.check(K.lib.vqmc_gpu_get_params(hd, K.ptr(th[k])))
        assert np.array_equal(th[0], th[1])
    finally:
        for hd in hs:
            K.lib.vqmc_gpu_destroy(hd)


_CG_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/oracle")
import pyoracle as O
from paper_2106_13308_b200 import api
n, B, seed = 100, 512, 4
h = O.default_made_hidden(n)
m = O.made_init(n, h, seed)
x = np.ascontiguousarray(O.auto_sample(m, B, seed=seed, stream=1, mode=1)[0], np.uint8)
e = O.random_maxcut_graph(n, seed)
g = O.gradient_from_locals(m, x, O.local_energy(n, e, x)[0])
model = api.MadeModel(n, h, m.degrees, m.theta)
info = {}
d = api.sr_direction(api.SrConfig(lam=1e-3, tol=1e-6, max_iterations=200), g, api.fisher_estimate(model, x), info)
np.save(sys.argv[2], np.concatenate([d, [info["iterations"], info["residual"]]]))
"""


def test_sr_device_cg_loop_equals_host_loop(tmp_path):
    """The device-resident CG loop (one captured iteration under a conditional WHILE node, the
    convergence test on the device) takes the host loop's decisions: identical direction, iteration
    count and residual (VQMC_SR_HOST_LOOP=1 runs the host-driven loop)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "cg.py"
    script.write_text(_CG_SCRIPT)
    outs = []
    for host in ("0", "1"):
        out = tmp_path / f"cg_{host}.npy"
        env = dict(os.environ, VQMC_SR_HOST_LOOP=host)
        subprocess.run([sys.executable, str(script), root, str(out)], check=True, env=env, timeout=300)
        outs.append(np.load(out))
    dev, host = outs
    assert dev[-2] == host[-2] and dev[-2] > 0  # iterations
    assert np.array_equal(dev, host)
