"""Pins the CPU oracle to numbers recorded by the REFERENCE ITSELF
(`/root/reference/proj/test_output.txt`), i.e. outputs of the real Eigen build:

* acceptance criterion 1 (test_output.txt:21): "worst TV 0.0140 <= 0.02, worst z 1.72"
  — 5 perturbed MADE models at n=8, 1e5 samples each (acceptance.cpp:61-97).
  Reproducing both printed figures exercises mix_seed/make_stream, made_init's
  fill order, the uniform(-1.5,1.5) perturbation, the n-forward sampler and its
  uniform consumption order, log_prob and the GoF statistic.
* acceptance criterion 6 (test_output.txt:26): "adam worst ratio 0.956" — Max-Cut
  n=20, 5 seeds, MADE+AUTO+ADAM, 300 iterations, batch 1024 (acceptance.cpp:239-272).
  This is a 300-step trajectory of the whole north-star path (sampler, Max-Cut
  local energy, REINFORCE gradient, tree all-reduce, Adam, final evaluation).
  Its SR half, "sr optimal 5/5 (worst ratio 1.000)" — SGD + SR, 150 iterations, batch 256
  (acceptance.cpp:246-257) — pins the SR restatement (score_matrix, FisherEstimate, the dense
  sr_direction at d = 1865).

The CPU-generated golden fixtures (tests/golden/) are checked here too.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import pyoracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_pin_criterion1_sampler_exactness():
    worst_tv, worst_z = 0.0, -1e9
    for seed in range(5):
        m = O.made_init(8, O.default_made_hidden(8), seed)
        m.theta = m.theta + (O.uniforms(seed, 98, m.d) * 3.0 + -1.5)  # U(-1.5, 1.5)
        probs = O.enumerate_distribution(m)
        x, _ = O.auto_sample(m, 100000, seed=seed, stream=100)
        g = O.goodness_of_fit(8, probs, x)
        worst_tv, worst_z = max(worst_tv, g["tv"]), max(worst_z, g["z"])
    assert "%.4f" % worst_tv == "0.0140"
    assert "%.2f" % worst_z == "1.72"


def test_pin_criterion6_maxcut_adam_ratio():
    worst = 1.0
    for s in range(5):
        e = O.random_maxcut_graph(20, s)
        opt, _ = O.brute_force_maxcut(20, e)
        r = O.train(20, e, optimizer="adam", iterations=300, minibatch=1024, eval_batch=1024, seed=s,
                    sampler_mode=0)
        worst = min(worst, r["best_cut"] / opt)
    assert "%.3f" % worst == "0.956"


def test_pin_criterion6_maxcut_sr_optimal():
    def run(s):  # (ctypes releases the GIL: the five seeds run on five host threads)
        e = O.random_maxcut_graph(20, s)
        opt, _ = O.brute_force_maxcut(20, e)
        r = O.train(20, e, optimizer="sgd_sr", iterations=150, minibatch=256, eval_batch=1024, seed=s,
                    sampler_mode=1)
        return r["best_cut"], opt

    with ThreadPoolExecutor(5) as ex:
        res = list(ex.map(run, range(5)))
    optimal = sum(c >= o for c, o in res)
    worst = min(c / o for c, o in res)
    assert optimal == 5 and "%.3f" % worst == "1.000"


def test_golden_fixtures_reproduce():
    path = os.path.join(GOLDEN, "oracle_n20_seed0.npz")
    if not os.path.exists(path):
        import pytest
        pytest.skip("golden fixture not generated")
    g = np.load(path)
    m = O.Made(int(g["n"]), int(g["h"]), g["degrees"], g["theta"])
    x, lp, p = O.auto_sample(m, int(g["B"]), uniforms=g["uniforms"], want_p=True)
    assert np.array_equal(x, g["x"]) and np.array_equal(lp, g["log_psi"])
    le, cut = O.local_energy(m.n, g["edges"], x)
    assert np.array_equal(cut, g["cut"])
    grad = O.gradient_from_locals(m, x, le)
    assert np.allclose(grad, g["grad"], rtol=1e-12, atol=1e-15)
