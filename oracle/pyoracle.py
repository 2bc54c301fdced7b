"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the CPU oracle (vqmc_oracle.cpp).

The oracle restates the reference VQMC path (arxiv/paper_2106_13308,
/root/reference/proj) in fp64 C++.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libvqmc_oracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    L.oracle_last_error.restype = C.c_char_p
    L.oracle_blas_path.restype = C.c_char_p
    L.oracle_mix_seed.restype = C.c_uint64
    L.oracle_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.oracle_default_made_hidden.argtypes = [C.c_int]
    L.oracle_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, _dp]
    L.oracle_philox_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _dp]
    L.oracle_made_init.argtypes = [C.c_int, C.c_int, C.c_uint64, _ip, _dp]
    L.oracle_forward.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, _u8, C.c_void_p, C.c_void_p, C.c_void_p]
    L.oracle_log_psi.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, _u8, _dp]
    L.oracle_auto_sample.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_uint64, C.c_uint64,
                                     C.c_void_p, C.c_int, _u8, _dp, C.c_void_p]
    L.oracle_local_energy.argtypes = [C.c_int, _ip, C.c_int64, C.c_int, _u8, _dp, C.c_void_p]
    L.oracle_energy_and_variance.argtypes = [_dp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.oracle_weighted_grad.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, _u8, _dp, _dp]
    L.oracle_gradient_from_locals.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, _u8, _dp, _dp]
    L.oracle_adam_step.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, C.POINTER(C.c_int64),
                                   C.c_double, C.c_double, C.c_double, C.c_double]
    L.oracle_allreduce_mean.argtypes = [C.c_int, C.c_int64, _dp, _dp]
    for fn in ("oracle_random_maxcut_graph",):
        getattr(L, fn).argtypes = [C.c_int, C.c_uint64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    L.oracle_random_regular_graph.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int64,
                                              C.POINTER(C.c_int64)]
    L.oracle_erdos_renyi_graph.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_void_p, C.c_int64,
                                           C.POINTER(C.c_int64)]
    L.oracle_brute_force_maxcut.restype = C.c_int64
    L.oracle_brute_force_maxcut.argtypes = [C.c_int, _ip, C.c_int64, C.POINTER(C.c_uint64)]
    L.oracle_train.argtypes = [C.c_int, C.c_int, _ip, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int,
                               C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]
    L.oracle_evaluate.argtypes = [C.c_int, C.c_int, _ip, _dp, _ip, C.c_int64, C.c_int, C.c_uint64, C.c_uint64,
                                  C.c_void_p, C.c_int, _dp]
    L.oracle_enumerate_distribution.argtypes = [C.c_int, C.c_int, _ip, _dp, _dp]
    L.oracle_time_reference_step.argtypes = [C.c_int, C.c_int, _ip, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                             C.c_int, _dp]
    L.oracle_goodness_of_fit.argtypes = [C.c_int, _dp, C.c_int64, _u8, _dp]
    L.oracle_set_train_sr.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, C.c_int]
    L.oracle_score_matrix.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, _u8, _dp]
    L.oracle_sr_direction.argtypes = [C.c_int64, C.c_int, _dp, C.c_int, _dp, C.c_double, C.c_double, C.c_int,
                                      _dp, C.POINTER(C.c_int), C.POINTER(C.c_double)]
    L.oracle_random_tim.argtypes = [C.c_int, C.c_uint64, _dp, _dp, _ip, _ip, _dp]
    L.oracle_diagonal_energy.argtypes = [C.c_int, _dp, _dp, _ip, _ip, _dp, C.c_int64, C.c_int, _u8, _dp]
    L.oracle_local_energy_spec.argtypes = [C.c_int, C.c_int, _ip, _dp, _dp, _dp, _ip, _ip, _dp, C.c_int64,
                                           C.c_int, _u8, _dp, _dp]
    L.oracle_train_spec.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, _ip, _dp, C.c_int64, C.c_int, C.c_double,
                                    C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().oracle_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def mix_seed(seed, stream):
    return lib().oracle_mix_seed(seed, stream)


def default_made_hidden(n):
    return lib().oracle_default_made_hidden(n)


def uniforms(seed, stream, count, skip=0):
    out = np.empty(count, np.float64)
    _check(lib().oracle_uniforms(seed, stream, skip, count, out))
    return out


def philox_uniforms(seed, stream, call, n, B):
    out = np.empty((n, B), np.float64)
    _check(lib().oracle_philox_uniforms(seed, stream, call, n, B, out))
    return out


class Made:
    """Reference MADE parameters: theta in reference flatten order (models.cpp:264-275)."""

    def __init__(self, n, h, degrees, theta):
        self.n, self.h = int(n), int(h)
        self.degrees = np.ascontiguousarray(degrees, np.int32)
        self.theta = np.ascontiguousarray(theta, np.float64)

    @property
    def d(self):
        return 2 * self.h * self.n + self.h + self.n

    def copy(self):
        return Made(self.n, self.h, self.degrees.copy(), self.theta.copy())

    def split(self):
        n, h, t = self.n, self.h, self.theta
        W1 = t[: h * n].reshape(h, n)
        b1 = t[h * n: h * n + h]
        W2 = t[h * n + h: h * n + h + n * h].reshape(n, h)
        b2 = t[h * n + h + n * h:]
        return W1, b1, W2, b2


def made_init(n, h, seed):
    deg = np.empty(h, np.int32)
    theta = np.empty(2 * h * n + h + n, np.float64)
    _check(lib().oracle_made_init(n, h, seed, deg, theta))
    return Made(n, h, deg, theta)


def forward(m: Made, x):
    x = np.ascontiguousarray(x, np.uint8)
    B = x.shape[0]
    p = np.empty((B, m.n)); pr = np.empty((B, m.n)); z1 = np.empty((B, m.h))
    _check(lib().oracle_forward(m.n, m.h, m.degrees, m.theta, B, x, _ptr(p), _ptr(pr), _ptr(z1)))
    return p, pr, z1


def log_psi(m: Made, x):
    x = np.ascontiguousarray(x, np.uint8)
    out = np.empty(x.shape[0])
    _check(lib().oracle_log_psi(m.n, m.h, m.degrees, m.theta, x.shape[0], x, out))
    return out


def auto_sample(m: Made, B, seed=0, stream=0, uniforms=None, mode=0, want_p=False):
    """mode 0 = reference n-forward sampler, mode 1 = incremental restatement."""
    x = np.empty((B, m.n), np.uint8)
    lp = np.empty(B)
    p = np.empty((B, m.n)) if want_p else None
    u = None if uniforms is None else np.ascontiguousarray(uniforms, np.float64)
    _check(lib().oracle_auto_sample(m.n, m.h, m.degrees, m.theta, B, seed, stream, _ptr(u), mode, x, lp,
                                    _ptr(p)))
    return (x, lp, p) if want_p else (x, lp)


def local_energy(n, edges, x):
    x = np.ascontiguousarray(x, np.uint8)
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    B = x.shape[0]
    le = np.empty(B); cut = np.empty(B)
    _check(lib().oracle_local_energy(n, e, e.size // 2, B, x, le, _ptr(cut)))
    return le, cut


def energy_and_variance(l):
    l = np.ascontiguousarray(l, np.float64)
    m = C.c_double(); v = C.c_double()
    _check(lib().oracle_energy_and_variance(l, l.size, C.byref(m), C.byref(v)))
    return m.value, v.value


def weighted_grad(m: Made, x, w):
    x = np.ascontiguousarray(x, np.uint8)
    g = np.empty(m.d)
    _check(lib().oracle_weighted_grad(m.n, m.h, m.degrees, m.theta, x.shape[0], x,
                                      np.ascontiguousarray(w, np.float64), g))
    return g


def gradient_from_locals(m: Made, x, local):
    x = np.ascontiguousarray(x, np.uint8)
    g = np.empty(m.d)
    _check(lib().oracle_gradient_from_locals(m.n, m.h, m.degrees, m.theta, x.shape[0], x,
                                             np.ascontiguousarray(local, np.float64), g))
    return g


class AdamState:
    def __init__(self, d, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        self.m = np.zeros(d); self.v = np.zeros(d); self.t = 0
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps


def adam_step(st: AdamState, params, grad):
    t = C.c_int64(st.t)
    _check(lib().oracle_adam_step(params.size, params, np.ascontiguousarray(grad, np.float64), st.m, st.v,
                                  C.byref(t), st.lr, st.b1, st.b2, st.eps))
    st.t = t.value


def allreduce_mean(vs):
    vs = np.ascontiguousarray(np.stack(vs), np.float64)
    out = np.empty(vs.shape[1])
    _check(lib().oracle_allreduce_mean(vs.shape[0], vs.shape[1], vs, out))
    return out


def _graph(fn, *args):
    ne = C.c_int64()
    _check(fn(*args, None, 0, C.byref(ne)))
    e = np.empty((ne.value, 2), np.int32)
    _check(fn(*args, _ptr(e), ne.value, C.byref(ne)))
    return e


def random_maxcut_graph(n, seed):
    return _graph(lib().oracle_random_maxcut_graph, n, seed)


def random_regular_graph(n, d, seed):
    return _graph(lib().oracle_random_regular_graph, n, d, seed)


def erdos_renyi_graph(n, p, seed):
    return _graph(lib().oracle_erdos_renyi_graph, n, p, seed)


def brute_force_maxcut(n, edges):
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    am = C.c_uint64()
    v = lib().oracle_brute_force_maxcut(n, e, e.size // 2, C.byref(am))
    if v < 0:
        raise RuntimeError(lib().oracle_last_error().decode())
    return int(v), int(am.value)


class SrSolveError(RuntimeError):
    """SR conjugate gradient did not converge (optimizer.hpp:46-55)."""

    def __init__(self, msg, residual, iterations):
        super().__init__(msg)
        self.residual, self.iterations = residual, iterations


def score_matrix(m: Made, x):
    """score_matrix (models.cpp:221-244): B x d rows 2 grad log psi, reference flatten order."""
    x = np.ascontiguousarray(x, np.uint8)
    out = np.empty((x.shape[0], m.d))
    _check(lib().oracle_score_matrix(m.n, m.h, m.degrees, m.theta, x.shape[0], x, out))
    return out


def sr_direction(scores, grad, lam=1e-3, tol=1e-6, max_iterations=200, centered=True):
    """sr_direction (optimizer.cpp:64-82) over explicit score rows; returns (delta, iters, resid)."""
    S = np.ascontiguousarray(scores, np.float64)
    g = np.ascontiguousarray(grad, np.float64)
    out = np.empty(S.shape[1]); it = C.c_int(0); res = C.c_double(0.0)
    rc = lib().oracle_sr_direction(S.shape[1], S.shape[0], S, 1 if centered else 0, g, lam, tol, max_iterations,
                                   out, C.byref(it), C.byref(res))
    if rc == -3:
        raise SrSolveError(lib().oracle_last_error().decode(), res.value, it.value)
    _check(rc)
    return out, it.value, res.value


_OPT = {"sgd": 0, "adam": 1, "sgd_sr": 2}


def train(n, edges, h=0, optimizer="adam", lr=0.0, iterations=300, workers=1, minibatch=1024,
          eval_batch=1024, seed=0, sampler_mode=0, threads=True, want_first_grad=False,
          sr_lambda=1e-3, sr_tol=1e-6, sr_max_iterations=200, sr_fallback=False, sr_centered=True):
    """Restated vqmc::train for MADE+AUTO on a Max-Cut instance (trainer.cpp:111-322)."""
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    hh = h if h > 0 else default_made_hidden(n)
    d = 2 * hh * n + hh + n
    stats = np.empty((iterations, 4)); ev = np.empty(4); theta = np.empty(d)
    g0 = np.empty(d) if want_first_grad else None
    _check(lib().oracle_set_train_sr(sr_lambda, sr_tol, sr_max_iterations, 1 if sr_fallback else 0,
                                     1 if sr_centered else 0))
    _check(lib().oracle_train(n, hh, e, e.size // 2, _OPT[optimizer], lr, iterations,
                              workers, minibatch, eval_batch, seed, sampler_mode, 1 if threads else 0,
                              _ptr(stats), _ptr(ev), _ptr(theta), _ptr(g0)))
    out = dict(stats=stats, final_energy=ev[0], final_energy_std=ev[1], best_cut=ev[2], mean_cut=ev[3],
               theta=theta, h=hh)
    if want_first_grad:
        out["first_grad"] = g0
    return out


def evaluate(m: Made, edges, B, seed=0, stream=1_000_000_007, uniforms=None, mode=0):
    """evaluate (trainer.cpp:91-108): {energy, energy_std, best_cut, mean_cut} of B samples."""
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    u = None if uniforms is None else np.ascontiguousarray(uniforms, np.float64)
    out = np.empty(4)
    _check(lib().oracle_evaluate(m.n, m.h, m.degrees, m.theta, e, e.size // 2, B, seed, stream, _ptr(u), mode, out))
    return out


def enumerate_distribution(m: Made):
    p = np.empty(1 << m.n)
    _check(lib().oracle_enumerate_distribution(m.n, m.h, m.degrees, m.theta, p))
    return p


def goodness_of_fit(n, probs, x):
    x = np.ascontiguousarray(x, np.uint8)
    out = np.empty(5)
    _check(lib().oracle_goodness_of_fit(n, np.ascontiguousarray(probs, np.float64), x.shape[0], x, out))
    return dict(tv=out[0], chi2=out[1], dof=int(out[2]), z=out[3], reject=bool(out[4]))


def time_reference_step(n, edges, workers, minibatch, seed=0, bits_limit=None, h=0):
    """One reference iteration on `workers` host threads, sampler extrapolated from
    `bits_limit` bits; returns dict of seconds (see oracle_time_reference_step)."""
    e = np.ascontiguousarray(edges, np.int32).reshape(-1)
    out = np.empty(5)
    _check(lib().oracle_time_reference_step(n, h, e, e.size // 2, workers, minibatch, seed,
                                            bits_limit or n, out))
    return dict(sample_s=out[0], estimate_s=out[1], update_s=out[2], step_s=out[3], bits_timed=int(out[4]))


# ---------------------------------------------------------------------------
# General Ising spec (TIM): hamiltonian.hpp:26-44, hamiltonian.cpp:36-69,126-142,
# estimator.hpp:43-90
# ---------------------------------------------------------------------------
class Spec:
    """H = -sum_i (alpha_i X_i + beta_i Z_i) - sum_{i<j} beta_ij Z_i Z_j (pairs: i, j, value)."""

    def __init__(self, n, alpha, beta, pi, pj, pv):
        self.n = n
        self.alpha = np.ascontiguousarray(alpha, np.float64)
        self.beta = np.ascontiguousarray(beta, np.float64)
        self.pi = np.ascontiguousarray(pi, np.int32)
        self.pj = np.ascontiguousarray(pj, np.int32)
        self.pv = np.ascontiguousarray(pv, np.float64)

    @property
    def npairs(self):
        return self.pi.size

    def args(self):
        return (self.alpha, self.beta, self.pi, self.pj, self.pv, self.npairs)


def random_tim(n, seed):
    np_ = n * (n - 1) // 2
    a = np.empty(n); b = np.empty(n)
    pi = np.empty(np_, np.int32); pj = np.empty(np_, np.int32); pv = np.empty(np_)
    _check(lib().oracle_random_tim(n, seed, a, b, pi, pj, pv))
    return Spec(n, a, b, pi, pj, pv)


def maxcut_spec(n, edges):
    """maxcut_spec (hamiltonian.cpp:109-119): alpha = beta = 0, beta_ij = -1/4 per edge."""
    e = np.asarray(edges, np.int32).reshape(-1, 2)
    return Spec(n, np.zeros(n), np.zeros(n), e[:, 0], e[:, 1], np.full(e.shape[0], -0.25))


def diagonal_energy(spec: Spec, x):
    x = np.ascontiguousarray(x, np.uint8)
    out = np.empty(x.shape[0])
    _check(lib().oracle_diagonal_energy(spec.n, *spec.args(), x.shape[0], x, out))
    return out


def local_energy_spec(spec: Spec, m: Made, x, cached_log_psi):
    """local_energy_batch (estimator.hpp:43-90) with the off-diagonal (flipped-neighbour) branch."""
    x = np.ascontiguousarray(x, np.uint8)
    out = np.empty(x.shape[0])
    _check(lib().oracle_local_energy_spec(m.n, m.h, m.degrees, m.theta, *spec.args(), x.shape[0], x,
                                          np.ascontiguousarray(cached_log_psi, np.float64), out))
    return out


def train_spec(spec: Spec, h=0, optimizer="adam", lr=0.0, iterations=300, workers=1, minibatch=1024,
               eval_batch=1024, seed=0, sampler_mode=0, threads=True, want_first_grad=False,
               sr_lambda=1e-3, sr_tol=1e-6, sr_max_iterations=200, sr_fallback=False, sr_centered=True):
    """Restated vqmc::train for MADE+AUTO on a general spec (TIM) (trainer.cpp:111-322)."""
    n = spec.n
    hh = h if h > 0 else default_made_hidden(n)
    d = 2 * hh * n + hh + n
    stats = np.empty((iterations, 4)); ev = np.empty(4); theta = np.empty(d)
    g0 = np.empty(d) if want_first_grad else None
    _check(lib().oracle_set_train_sr(sr_lambda, sr_tol, sr_max_iterations, 1 if sr_fallback else 0,
                                     1 if sr_centered else 0))
    _check(lib().oracle_train_spec(n, hh, *spec.args(), _OPT[optimizer], lr, iterations, workers, minibatch,
                                   eval_batch, seed, sampler_mode, 1 if threads else 0, _ptr(stats), _ptr(ev),
                                   _ptr(theta), _ptr(g0)))
    out = dict(stats=stats, final_energy=ev[0], final_energy_std=ev[1], theta=theta, h=hh)
    if want_first_grad:
        out["first_grad"] = g0
    return out


def dense_hamiltonian(spec: Spec):
    """dense_matrix (oracle.cpp) in numpy for small n: H[x, y], bit 1 = MSB of the index."""
    n = spec.n
    N = 1 << n
    idx = np.arange(N)
    X = ((idx[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1).astype(np.float64)
    S = 1.0 - 2.0 * X
    diag = -(S @ spec.beta) - np.sum(spec.pv[None, :] * S[:, spec.pi] * S[:, spec.pj], axis=1)
    H = np.diag(diag)
    for i in range(n):
        if spec.alpha[i] != 0.0:
            H[idx, idx ^ (1 << (n - 1 - i))] -= spec.alpha[i]
    return H
