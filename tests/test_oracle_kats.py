"""Pins the CPU oracle (oracle/vqmc_oracle.cpp) to the reference's own known-answer
tests and properties (proj/tests/*.cpp).  CPU only."""
import numpy as np
import pytest

import pyoracle as O


def test_default_hidden_width():  # models_test.cpp:59-63
    assert [O.default_made_hidden(n) for n in (4, 12, 20)] == [10, 31, 45]
    # Appendix B of SURVEY.md
    assert [O.default_made_hidden(n) for n in (100, 1000, 5000, 10000)] == [106, 239, 363, 424]


def test_degrees_masks_and_counts():  # models_test.cpp:65-84
    m = O.made_init(4, 5, 0)
    assert list(m.degrees) == [1, 2, 3, 1, 2]
    assert m.d == 49
    assert O.made_init(8, 22, 0).d == 382


def test_init_deterministic_and_bounded():  # models_test.cpp:86-94
    a, b = O.made_init(6, 10, 3), O.made_init(6, 10, 3)
    assert np.array_equal(a.theta, b.theta)
    W1, b1, W2, b2 = a.split()
    assert np.all(b1 == 0) and np.all(b2 == 0)
    assert np.abs(W1).max() <= 1 / np.sqrt(6) and np.abs(W2).max() <= 1 / np.sqrt(10)


def _all_configs(n):
    idx = np.arange(1 << n)
    return ((idx[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1).astype(np.uint8)


@pytest.mark.parametrize("n", [3, 6, 10])
@pytest.mark.parametrize("seed", [0, 1])
def test_normalized(n, seed):  # models_test.cpp:96-104
    m = O.made_init(n, O.default_made_hidden(n), seed)
    lp = 2 * O.log_psi(m, _all_configs(n))
    assert abs(np.exp(lp).sum() - 1.0) <= 1e-10


def test_autoregressive_invariance():  # models_test.cpp:106-123
    m = O.made_init(6, 14, 9)
    rng = np.random.default_rng(4)
    for _ in range(20):
        x = rng.integers(0, 2, size=(1, 6)).astype(np.uint8)
        base, _, _ = O.forward(m, x)
        for j in range(6):
            y = x.copy(); y[0, j] ^= 1
            fl, _, _ = O.forward(m, y)
            assert np.array_equal(fl[0, : j + 1], base[0, : j + 1])


def _perturb(m, seed, lo=0.05, hi=0.35, stream=99):
    sh = O.uniforms(seed, stream, m.d)
    m.theta = m.theta + (sh * (hi - lo) + lo)


def test_fd_gradient():  # models_test.cpp:151-173
    m = O.made_init(5, 7, 1)
    _perturb(m, 1)
    for idx in (0, 13, 31):
        x = _all_configs(5)[idx: idx + 1]
        g = O.weighted_grad(m, x, np.ones(1))
        fd = np.empty(m.d)
        for p in range(m.d):
            mm = m.copy(); mm.theta[p] += 1e-5; up = O.log_psi(mm, x)[0]
            mm.theta[p] -= 2e-5; dn = O.log_psi(mm, x)[0]
            fd[p] = (up - dn) / 2e-5
        assert np.linalg.norm(g - fd) / np.linalg.norm(fd) <= 1e-6


def test_masked_grads_zero_and_layout():  # models_test.cpp:175-190
    m = O.made_init(6, 9, 8)
    n, h = 6, 9
    x = _all_configs(6)[45:46]
    g = O.weighted_grad(m, x, np.ones(1))
    deg = m.degrees
    for k in range(h):
        for j in range(n):
            if not (j + 1 <= deg[k]):
                assert g[k * n + j] == 0.0
    for i in range(n):
        for k in range(h):
            if not (deg[k] < i + 1):
                assert g[h * n + h + i * h + k] == 0.0


def test_weighted_is_sum_of_singles():  # models_test.cpp:192-209
    m = O.made_init(4, 6, 2)
    x = _all_configs(4)[:5]
    w = np.array([0.3, -1.2, 0.0, 2.5, -0.7])
    exp = sum(w[b] * O.weighted_grad(m, x[b: b + 1], np.ones(1)) for b in range(5))
    assert np.abs(O.weighted_grad(m, x, w) - exp).max() <= 1e-12


def test_sampler_determinism_and_cache():  # sampler_test.cpp:70-84
    m = O.made_init(8, 15, 7)
    xa, la = O.auto_sample(m, 512, seed=3, stream=2)
    xb, lb = O.auto_sample(m, 512, seed=3, stream=2)
    assert np.array_equal(xa, xb) and np.array_equal(la, lb)
    m2 = O.made_init(7, 12, 4)
    x, lp = O.auto_sample(m2, 256, seed=9, stream=0)
    assert np.abs(lp - O.log_psi(m2, x)).max() <= 1e-12


def test_zero_params_sample_uniform():  # sampler_test.cpp:51-57
    m = O.made_init(6, 10, 0)
    m.theta[:] = 0
    x, _ = O.auto_sample(m, 50000, seed=1, stream=0)
    g = O.goodness_of_fit(6, np.full(64, 1 / 64), x)
    assert g["tv"] <= 0.03


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ancestral_matches_enumeration(seed):  # sampler_test.cpp:59-68
    m = O.made_init(6, 12, seed)
    probs = O.enumerate_distribution(m)
    x, _ = O.auto_sample(m, 50000, seed=seed, stream=5)
    assert O.goodness_of_fit(6, probs, x)["tv"] <= 0.03


def test_incremental_sampler_equals_reference_sampler():
    """The incremental restatement is bit-identical to the n-forward one on these cases."""
    for n, seed in ((5, 0), (20, 3), (37, 1)):
        m = O.made_init(n, O.default_made_hidden(n), seed)
        _perturb(m, seed, -1.5, 1.5, 98)
        x0, l0, p0 = O.auto_sample(m, 300, seed=seed, stream=1, want_p=True)
        x1, l1, p1 = O.auto_sample(m, 300, seed=seed, stream=1, mode=1, want_p=True)
        assert np.array_equal(x0, x1)
        assert np.allclose(l0, l1, rtol=1e-12, atol=1e-12)
        assert np.allclose(p0, p1, rtol=1e-12, atol=1e-15)


def test_uniform_injection_equals_stream():
    m = O.made_init(10, 20, 5)
    u = O.uniforms(5, 7, 10 * 64).reshape(10, 64)
    xa, la = O.auto_sample(m, 64, seed=5, stream=7)
    xb, lb = O.auto_sample(m, 64, uniforms=u)
    assert np.array_equal(xa, xb) and np.array_equal(la, lb)


def test_diagonal_local_energy_and_cut_identity():  # estimator_test.cpp:45-55; hamiltonian_test.cpp:99-111
    k3 = np.array([[0, 1], [0, 2], [1, 2]], np.int32)
    x = np.array([[0, 0, 1], [0, 0, 0], [1, 0, 1]], np.uint8)
    le, cut = O.local_energy(3, k3, x)
    assert list(cut) == [2.0, 0.0, 2.0]
    assert np.array_equal(cut, 0.5 * 3 - 2 * le)


@pytest.mark.parametrize("seed", [0, 3])
def test_argmin_diagonal_is_brute_force(seed):  # hamiltonian_test.cpp:113-129
    e = O.random_maxcut_graph(10, seed)
    x = _all_configs(10)
    le, cut = O.local_energy(10, e, x)
    assert cut[np.argmin(le)] == O.brute_force_maxcut(10, e)[0]


def test_graph_generation():  # hamiltonian_test.cpp:131-143 and SURVEY §8 a14 probed counts
    a, b = O.random_maxcut_graph(12, 5), O.random_maxcut_graph(12, 5)
    assert np.array_equal(a, b) and np.all(a[:, 0] < a[:, 1]) and len(a) > 33
    assert len(O.random_maxcut_graph(20, 0)) == 150
    assert len(O.random_maxcut_graph(100, 0)) == 3698
    assert len(O.random_maxcut_graph(1000, 0)) == 374632
    r = O.random_regular_graph(100, 3, 0)
    assert len(r) == 150 and np.all(np.bincount(r.reshape(-1), minlength=100) == 3)
    assert len({tuple(t) for t in r.tolist()}) == 150 and np.all(r[:, 0] < r[:, 1])


def test_brute_force_known_graphs():  # oracle_test.cpp:93-117
    assert O.brute_force_maxcut(3, np.array([[0, 1], [0, 2], [1, 2]]))[0] == 2
    assert O.brute_force_maxcut(2, np.array([[0, 1]]))[0] == 1
    k4 = np.array([[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]])
    assert O.brute_force_maxcut(4, k4)[0] == 4


def test_adam_contract():  # optimizer_test.cpp:39-62
    st = O.AdamState(4)
    p = np.full(4, 1.5)
    O.adam_step(st, p, np.zeros(4))
    assert st.t == 1 and np.all(p == 1.5)
    O.adam_step(st, p, np.zeros(4))
    assert st.t == 2
    st = O.AdamState(3, lr=0.01)
    p = np.zeros(3)
    O.adam_step(st, p, np.array([4.0, -0.5, 1e-3]))
    assert p[0] == pytest.approx(-0.01, rel=1e-6)
    assert p[1] == pytest.approx(0.01, rel=1e-6)
    assert p[2] == pytest.approx(-0.01, rel=1e-3)


def test_allreduce_tree_order():  # trainer_test.cpp:21-35
    a, b, c = np.array([1.0, 2.0]), np.array([3.0, 4.0]), np.array([5.0, 6.0])
    assert list(O.allreduce_mean([a, b])) == [2.0, 3.0]
    assert np.array_equal(O.allreduce_mean([a]), a)
    assert O.allreduce_mean([a, b, c])[0] == ((a[0] + b[0]) + c[0]) / 3.0


def test_data_parallel_equals_serial_replay():  # trainer_test.cpp:37-68 (Max-Cut instance)
    n, mbs, L, seed = 6, 64, 4, 11
    e = O.random_maxcut_graph(n, 3)
    r = O.train(n, e, h=8, optimizer="sgd", iterations=1, workers=L, minibatch=mbs, eval_batch=256,
                seed=seed, want_first_grad=True)
    m = O.made_init(n, 8, seed)
    grads = []
    for w in range(L):
        x, lp = O.auto_sample(m, mbs, seed=seed, stream=w + 1)
        le, _ = O.local_energy(n, e, x)
        grads.append(O.gradient_from_locals(m, x, le))
    assert np.abs(r["first_grad"] - O.allreduce_mean(grads)).max() <= 1e-12


def test_rerun_reproduces_bitwise():  # trainer_test.cpp:70-92
    e = O.random_maxcut_graph(8, 3)
    a = O.train(8, e, iterations=10, workers=4, minibatch=32, eval_batch=128, seed=5)
    b = O.train(8, e, iterations=10, workers=4, minibatch=32, eval_batch=128, seed=5)
    assert np.array_equal(a["theta"], b["theta"]) and a["final_energy"] == b["final_energy"]


def test_maxcut_run_reports_cuts():  # trainer_test.cpp:156-172
    e = O.random_maxcut_graph(8, 3)
    r = O.train(8, e, iterations=40, minibatch=128, eval_batch=512, seed=4)
    assert r["best_cut"] >= r["mean_cut"] and r["best_cut"] <= len(e)


def test_invalid_configs_rejected():  # trainer_test.cpp:191-201
    e = O.random_maxcut_graph(4, 0)
    for kw in (dict(workers=0), dict(iterations=0), dict(minibatch=1)):
        with pytest.raises(RuntimeError):
            O.train(4, e, **kw)


# --- SR: optimizer_test.cpp:64-150, models_test.cpp:211-218 ---------------
def test_score_rows_are_twice_single_sample_gradients():  # models_test.cpp:211-218
    m = O.made_init(6, 10, 1)
    x, _ = O.auto_sample(m, 5, seed=1, stream=1)
    S = O.score_matrix(m, x)
    for b in range(5):
        w = np.zeros(5)
        w[b] = 1.0
        assert np.abs(S[b] - 2.0 * O.weighted_grad(m, x, w)).max() <= 1e-12


def test_sr_zero_fisher_is_grad_over_lambda():  # optimizer_test.cpp:64-71
    g = np.linspace(1.0, 6.0, 6)
    d, _, _ = O.sr_direction(np.zeros((4, 6)), g, lam=0.001)
    assert np.abs(d - g / 0.001).max() <= 1e-6 * np.linalg.norm(g)


def test_sr_identity_fisher_rescales():  # optimizer_test.cpp:73-82 (centred=False: S^T S / B = I)
    S = np.eye(5) * np.sqrt(5.0)
    g = np.linspace(-2.0, 2.0, 5)
    d, _, _ = O.sr_direction(S, g, lam=0.5, centered=False)
    assert np.abs(d - g / 1.5).max() <= 1e-10


def test_sr_large_lambda_monotone_angle():  # optimizer_test.cpp:84-106
    rng = np.random.default_rng(1)
    S, g = rng.standard_normal((16, 8)), rng.standard_normal(8)
    prev = 1e9
    for lam in (0.01, 1.0, 100.0, 10000.0):
        d, _, _ = O.sr_direction(S, g, lam=lam)
        ang = np.arccos(d @ g / (np.linalg.norm(d) * np.linalg.norm(g)))
        assert ang <= prev + 1e-12
        prev = ang


def test_sr_cg_path_residual_contract():  # optimizer_test.cpp:108-126 (d > 2000: CG)
    rng = np.random.default_rng(2)
    S, g = rng.standard_normal((6, 2100)), rng.standard_normal(2100)
    d, it, res = O.sr_direction(S, g, lam=0.001, tol=1e-6)
    Sc = S - S.mean(0)
    r = Sc.T @ (Sc @ d) / 6 + 0.001 * d - g
    assert np.linalg.norm(r) <= 1e-6 * np.linalg.norm(g) and it > 0 and res <= 1e-6


def test_sr_cg_failure_raises():  # optimizer_test.cpp:128-142
    S = np.zeros((4, 2100))
    S[0, 0] = 1.0
    with pytest.raises(O.SrSolveError):
        O.sr_direction(S, np.ones(2100), max_iterations=0)
