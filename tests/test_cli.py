"""The `vqmc` command-line drop-in (tools/vqmc_cli.cpp) against the reference CLI contract
(proj/tools/vqmc.cpp, proj/tests/cli_test.sh): subcommands, flag precedence with --config,
output files, pairing rejection and exit codes.  The solve / sample-test runs need a GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2106_13308_b200", "bin", "vqmc")


def run(*args, env=None, cwd=None):
    e = dict(os.environ)
    if env:
        e.update(env)
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, env=e, cwd=cwd)


def test_gen_instance_matches_reference_generator(tmp_path):
    p = tmp_path / "g6.txt"
    r = run("gen-instance", "--problem", "maxcut", "--n", 6, "--seed", 1, "--out", p)
    assert r.returncode == 0 and "wrote" in r.stdout
    lines = p.read_text().split("\n")
    assert lines[0] == "graph 6"
    edges = [tuple(int(t) - 1 for t in ln.split()[1:]) for ln in lines[1:] if ln]
    assert np.array_equal(np.array(edges), O.random_maxcut_graph(6, 1))


def test_oracle_subcommand(tmp_path):  # cli_test.sh:27-29
    p = tmp_path / "g10.txt"
    run("gen-instance", "--problem", "maxcut", "--n", 10, "--seed", 3, "--out", p)
    r = run("oracle", "--instance", p)
    assert r.returncode == 0
    assert int(r.stdout.split("\n")[0].split()[-1]) == O.brute_force_maxcut(10, O.random_maxcut_graph(10, 3))[0]


def test_config_precedence_and_parsing(tmp_path):  # cli_test.sh:49-63
    g = tmp_path / "g.txt"
    run("gen-instance", "--problem", "maxcut", "--n", 8, "--seed", 0, "--out", g)
    cfg = tmp_path / "cfg.ini"
    cfg.write_text("iterations=3\nminibatch=16\neval-batch=32\nseed=7  # comment\n\n")
    dry = {"VQMC_CLI_DRYRUN": "1"}
    r = run("solve", "--instance", g, "--config", cfg, env=dry)
    assert r.returncode == 0 and "iterations 3 " in r.stdout and "seed 7 " in r.stdout and "minibatch 16 " in r.stdout
    r = run("solve", "--instance", g, "--config", cfg, "--iterations", 2, "--seed=5", env=dry)
    assert "iterations 2 " in r.stdout and "seed 5 " in r.stdout
    r = run("solve", "--instance", g, "--iterations", 2, "--iterations", 9, env=dry)  # TakeLast
    assert "iterations 9 " in r.stdout


@pytest.mark.parametrize("args", [
    ["solve", "--no-such-flag"],                                     # unknown flag
    ["solve"],                                                       # missing instance
    ["solve", "--problem", "maxcut", "--n", 6, "--model", "made", "--sampler", "mcmc"],  # pairing
    ["solve", "--problem", "maxcut", "--n", 6, "--model", "rbm", "--sampler", "auto"],
    ["solve", "--problem", "maxcut", "--n", 6, "--iterations", "abc"],
    ["gen-instance", "--problem", "ising", "--n", 4, "--out", "/tmp/x.txt"],  # not in {tim, maxcut}
    ["solve", "--problem", "tim", "--n", 6, "--optimizer", "sgd"],  # plain SGD is outside the path
    ["bogus"],
])
def test_usage_errors_exit_1(args):  # cli_test.sh:65-78
    assert run(*args).returncode == 1


def test_gen_instance_tim_matches_reference_generator(tmp_path):  # vqmc.cpp:533-537, hamiltonian.cpp:126-177
    p = tmp_path / "t7.txt"
    r = run("gen-instance", "--problem", "tim", "--n", 7, "--seed", 2, "--out", p)
    assert r.returncode == 0
    lines = [ln.split() for ln in p.read_text().strip().split("\n")]
    assert lines[0] == ["tim", "7"]
    ref = O.random_tim(7, 2)
    alpha = np.zeros(7); beta = np.zeros(7); pairs = []
    for t in lines[1:]:
        if t[0] == "alpha":
            alpha[int(t[1]) - 1] = float(t[2])
        elif t[0] == "beta":
            beta[int(t[1]) - 1] = float(t[2])
        else:
            pairs.append((int(t[1]) - 1, int(t[2]) - 1, float(t[3])))
    assert np.array_equal(alpha, ref.alpha) and np.array_equal(beta, ref.beta)  # %.17g round-trips
    assert np.array_equal(np.array([q[2] for q in pairs]), ref.pv)
    assert np.array_equal(np.array([q[0] for q in pairs]), ref.pi)


def test_tim_instance_resolution_and_validation(tmp_path):
    dry = {"VQMC_CLI_DRYRUN": "1"}
    p = tmp_path / "t.txt"
    p.write_text("tim 3\nalpha 1 0.5\npair 1 3 -0.25  # comment\n")
    r = run("solve", "--instance", p, "--iterations", 2, env=dry)
    assert r.returncode == 0 and "problem tim" in r.stdout and "n 3 " in r.stdout
    r = run("solve", "--n", 9, "--workers", 4, "--gpus", 2, env=dry)  # --problem defaults to tim
    assert r.returncode == 0 and "problem tim gpus 2" in r.stdout
    p.write_text("tim 3\nalpha 1 -0.5\n")  # HamiltonianSpec::validate
    r = run("solve", "--instance", p, "--iterations", 2, env=dry)
    assert r.returncode == 1 and "alpha must be non-negative" in r.stderr
    p.write_text("tim 3\npair 2 1 0.5\n")  # load_spec: i < j
    r = run("solve", "--instance", p, env=dry)
    assert r.returncode == 1 and "i < j" in r.stderr


@pytest.mark.gpu
def test_solve_outputs_and_checkpoint_roundtrip(tmp_path):  # cli_test.sh:31-47, 96-99
    g = tmp_path / "g.txt"
    run("gen-instance", "--problem", "maxcut", "--n", 5, "--seed", 1, "--out", g)  # small: TV needs few bins
    out = tmp_path / "run"
    r = run("solve", "--instance", g, "--iterations", 5, "--minibatch", 32, "--eval-batch", 64, "--seed", 1,
            "--out", out, "--save-model", tmp_path / "model.txt")
    assert r.returncode == 0, r.stderr
    rows = (out / "curve.csv").read_text().strip().split("\n")
    assert rows[0] == "iter,energy_mean,energy_std,grad_norm,time_s" and len(rows) == 6
    s = json.loads((out / "summary.json").read_text())
    assert s["config"]["seed"] == 1 and s["iterations_run"] == 5 and s["best_cut"] >= s["mean_cut"]
    assert '"seed": 1' in (out / "summary.json").read_text()
    r = run("sample-test", "--checkpoint", tmp_path / "model.txt", "--samples", 20000)
    assert r.returncode == 0 and "tv_distance" in r.stdout and "PASS" in r.stdout
    r = run("sample-test", "--model", "made", "--n", 5, "--seed", 3, "--samples", 20000)
    assert r.returncode == 0


@pytest.mark.gpu
def test_solve_reference_streams_reaches_near_optimum(tmp_path):
    """MADE + AUTO + ADAM on n=20 through the CLI with the reference's streams
    (acceptance.cpp:239-272: ADAM >= 0.95 x the brute-force optimum)."""
    g = tmp_path / "g20.txt"
    run("gen-instance", "--problem", "maxcut", "--n", 20, "--seed", 0, "--out", g)
    out = tmp_path / "run"
    r = run("solve", "--instance", g, "--iterations", 300, "--minibatch", 1024, "--seed", 0, "--reference-streams",
            "--out", out)
    assert r.returncode == 0, r.stderr
    best = json.loads((out / "summary.json").read_text())["best_cut"]
    opt, _ = O.brute_force_maxcut(20, O.random_maxcut_graph(20, 0))
    assert best >= 0.95 * opt


@pytest.mark.gpu
def test_solve_sgd_sr(tmp_path):
    """--optimizer sgd_sr (vqmc.cpp:416-425): SGD + SR on n=20 with the reference's streams
    reaches the optimum (acceptance.cpp:246-257); the summary echoes the SR settings
    (vqmc.cpp:170-176); a CG budget of 0 without --sr-fallback is a numerical failure (exit 2)."""
    g = tmp_path / "g20.txt"
    run("gen-instance", "--problem", "maxcut", "--n", 20, "--seed", 1, "--out", g)
    out = tmp_path / "run"
    r = run("solve", "--instance", g, "--optimizer", "sgd_sr", "--iterations", 150, "--minibatch", 256, "--seed", 1,
            "--reference-streams", "--out", out)
    assert r.returncode == 0, r.stderr
    s = json.loads((out / "summary.json").read_text())
    assert s["config"]["optimizer"] == "sgd_sr" and s["config"]["lr"] == 0.1
    assert s["config"]["sr_lambda"] == 0.001 and s["config"]["sr_centered"] is True
    opt, _ = O.brute_force_maxcut(20, O.random_maxcut_graph(20, 1))
    assert s["best_cut"] >= 0.97 * opt
    r = run("solve", "--problem", "maxcut", "--n", 30, "--optimizer", "sgd_sr", "--iterations", 1, "--minibatch",
            64, "--sr-maxiter", 0, "--out", tmp_path / "fail")
    assert r.returncode == 2 and "did not converge" in r.stderr
    r = run("solve", "--problem", "maxcut", "--n", 30, "--optimizer", "sgd_sr", "--iterations", 1, "--minibatch",
            64, "--sr-maxiter", 0, "--sr-fallback", "--out", tmp_path / "fb")
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_solve_target_reports_hit(tmp_path):  # vqmc.cpp:240-243 (hitting-time mode)
    out = tmp_path / "run"
    r = run("solve", "--problem", "maxcut", "--n", 12, "--iterations", 20, "--minibatch", 64, "--eval-batch", 64,
            "--target", 1, "--out", out)
    assert r.returncode == 0, r.stderr
    s = json.loads((out / "summary.json").read_text())
    assert s["hit_iteration"] == 1 and s["hit_time_s"] > 0 and s["iterations_run"] == 1


@pytest.mark.gpu
def test_solve_tim_instance(tmp_path):
    """solve on a TIM instance file (vqmc.cpp:119-140, 194-263): ADAM on random_tim(12, 100) with the
    reference's streams lands near the reference's converged energy; no cut in the summary."""
    p = tmp_path / "t12.txt"
    run("gen-instance", "--problem", "tim", "--n", 12, "--seed", 100, "--out", p)
    out = tmp_path / "run"
    r = run("solve", "--instance", p, "--iterations", 300, "--minibatch", 1024, "--seed", 0, "--reference-streams",
            "--out", out)
    assert r.returncode == 0, r.stderr
    s = json.loads((out / "summary.json").read_text())
    assert s["config"]["problem"] == "tim" and "best_cut" not in s and s["iterations_run"] == 300
    ref = O.train_spec(O.random_tim(12, 100), iterations=300, minibatch=1024, seed=0)["final_energy"]
    assert abs(s["final_energy"] - ref) <= 0.03 * abs(ref)
    rows = (out / "curve.csv").read_text().strip().split("\n")
    assert len(rows) == 301
    r = run("solve", "--problem", "tim", "--n", 10, "--iterations", 3, "--minibatch", 64, "--gpus", 64,
            "--workers", 64, "--out", tmp_path / "x")
    assert r.returncode == 1 and "visible" in r.stderr
