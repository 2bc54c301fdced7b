"""Python mirror of the reference's C++ API (arxiv/paper_2106_13308, proj/include/vqmc/*.hpp)
on top of the B200 C ABI (include/vqmc_b200.h).  Names, argument meaning and error
behaviour follow the reference: ValueError where it throws std::invalid_argument,
RuntimeError (VqmcError) where it throws std::runtime_error.

Configurations are numpy uint8 arrays (B x n, entries 0/1) instead of Eigen MatrixXd;
parameters are fp64 vectors in the reference flatten order.  Every compute call runs
on the GPU through libvqmc_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import time
from typing import Callable, List, Optional

import numpy as np

from . import _capi as K
from ._capi import check, ptr

kProbEps = 1e-7  # models.hpp:26
kEvalStream = 1_000_000_007  # trainer.cpp:48


# ---------------------------------------------------------------------------
# L0 common (common.hpp)
# ---------------------------------------------------------------------------
def mix_seed(seed: int, stream: int) -> int:
    return int(K.lib.vqmc_mix_seed(seed, stream))


class Stream:
    """make_stream(seed, stream) (common.hpp:64-66): a std::mt19937_64 stream consumed
    through uniform_real_distribution<double>(0, 1), tracked by its draw position so the
    GPU sampler can be fed the reference's exact uniforms (parity mode)."""

    def __init__(self, seed: int, stream: int = 0):
        self.seed, self.stream, self.position = int(seed), int(stream), 0

    def uniforms(self, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        check(K.lib.vqmc_stream_uniforms(self.seed, self.stream, self.position, count, ptr(out)))
        self.position += count
        return out


def make_stream(seed: int, stream: int = 0) -> Stream:
    return Stream(seed, stream)


class PhiloxStream:
    """Production-mode generator: counter-based Philox4x32-10 keyed by (seed, stream);
    each sampling call consumes one counter value."""

    def __init__(self, seed: int, stream: int = 0, call: int = 0):
        self.seed, self.stream, self.call = int(seed), int(stream), int(call)


def config_index(x) -> int:  # common.hpp:35-39
    idx = 0
    for v in np.asarray(x).reshape(-1):
        idx = (idx << 1) | (1 if v > 0.5 else 0)
    return idx


def index_to_config(n: int, idx: int) -> np.ndarray:
    return np.array([(idx >> (n - 1 - i)) & 1 for i in range(n)], np.uint8)


def all_configs(n: int) -> np.ndarray:
    idx = np.arange(1 << n, dtype=np.int64)
    return ((idx[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1).astype(np.uint8)


# ---------------------------------------------------------------------------
# L1 problem (hamiltonian.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Graph:
    n: int
    edges: np.ndarray  # E x 2 int32, i < j, 0-based


@dataclasses.dataclass
class MaxCutProblem:
    graph: Graph
    num_edges: int


def _edges_call(fn, *args) -> np.ndarray:
    ne = C.c_int64()
    check(fn(*args, None, 0, C.byref(ne)))
    e = np.empty((ne.value, 2), np.int32)
    check(fn(*args, ptr(e), ne.value, C.byref(ne)))
    return e


def random_maxcut_graph(n: int, seed: int) -> Graph:  # hamiltonian.cpp:144-160
    return Graph(n, _edges_call(K.lib.vqmc_random_maxcut_graph, n, seed))


def random_regular_graph(n: int, d: int, seed: int) -> Graph:
    return Graph(n, _edges_call(K.lib.vqmc_random_regular_graph, n, d, seed))


def erdos_renyi_graph(n: int, p: float, seed: int) -> Graph:
    return Graph(n, _edges_call(K.lib.vqmc_erdos_renyi_graph, n, p, seed))


def load_graph(path: str) -> Graph:  # hamiltonian.cpp:243-266
    n = C.c_int()
    ne = C.c_int64()
    check(K.lib.vqmc_load_graph(path.encode(), C.byref(n), None, 0, C.byref(ne)))
    e = np.empty((ne.value, 2), np.int32)
    check(K.lib.vqmc_load_graph(path.encode(), C.byref(n), ptr(e), ne.value, C.byref(ne)))
    return Graph(n.value, e)


def save_graph(g: Graph, path: str) -> None:  # hamiltonian.cpp:236-241
    e = np.ascontiguousarray(g.edges, np.int32)
    check(K.lib.vqmc_save_graph(path.encode(), g.n, ptr(e), len(e)))


def maxcut_spec(g: Graph) -> MaxCutProblem:  # hamiltonian.cpp:109-119 (validate :36-54)
    e = np.ascontiguousarray(g.edges, np.int32).reshape(-1, 2)
    if len(e):
        if np.any(e[:, 0] < 0) or np.any(e[:, 1] >= g.n) or np.any(e[:, 0] >= e[:, 1]):
            raise ValueError("pair indices must satisfy 0 <= i < j < n")
        if len(np.unique(e[:, 0].astype(np.int64) * g.n + e[:, 1])) != len(e):
            raise ValueError("duplicate pair")
    return MaxCutProblem(Graph(g.n, e), len(e))


@dataclasses.dataclass
class HamiltonianSpec:
    """HamiltonianSpec (hamiltonian.hpp:34-44): H = -sum_i (alpha_i X_i + beta_i Z_i)
    - sum_{i<j} beta_ij Z_i Z_j; pairs as three arrays (pair_i < pair_j, 0-based, value)."""
    n: int
    alpha: np.ndarray
    beta: np.ndarray
    pair_i: np.ndarray
    pair_j: np.ndarray
    pair_value: np.ndarray

    def __post_init__(self):
        self.alpha = np.ascontiguousarray(self.alpha, np.float64)
        self.beta = np.ascontiguousarray(self.beta, np.float64)
        self.pair_i = np.ascontiguousarray(self.pair_i, np.int32)
        self.pair_j = np.ascontiguousarray(self.pair_j, np.int32)
        self.pair_value = np.ascontiguousarray(self.pair_value, np.float64)

    def validate(self) -> None:  # hamiltonian.cpp:36-54
        if self.n < 1:
            raise ValueError("spec requires n >= 1")
        if self.alpha.shape != (self.n,) or self.beta.shape != (self.n,):
            raise ValueError("alpha/beta length does not match n")
        if np.any(self.alpha < 0.0):
            raise ValueError("alpha must be non-negative")
        if len(self.pair_i):
            if (np.any(self.pair_i < 0) or np.any(self.pair_j >= self.n) or np.any(self.pair_i >= self.pair_j)):
                raise ValueError("pair indices must satisfy 0 <= i < j < n")
            if len(np.unique(self.pair_i.astype(np.int64) * self.n + self.pair_j)) != len(self.pair_i):
                raise ValueError("duplicate pair")


def random_tim(n: int, seed: int) -> HamiltonianSpec:  # hamiltonian.cpp:126-142
    if n < 1:
        raise ValueError("random_tim requires n >= 1")
    npairs = n * (n - 1) // 2
    a, b = np.empty(n), np.empty(n)
    pi, pj, pv = np.empty(npairs, np.int32), np.empty(npairs, np.int32), np.empty(npairs)
    check(K.lib.vqmc_random_tim(n, seed, ptr(a), ptr(b), ptr(pi), ptr(pj), ptr(pv)))
    return HamiltonianSpec(n, a, b, pi, pj, pv)


def load_spec(path: str) -> HamiltonianSpec:  # hamiltonian.cpp:204-234
    n, npairs = C.c_int(), C.c_int64()
    check(K.lib.vqmc_load_spec(path.encode(), C.byref(n), None, None, None, None, None, 0, C.byref(npairs)))
    a, b = np.empty(n.value), np.empty(n.value)
    pi, pj, pv = (np.empty(npairs.value, np.int32), np.empty(npairs.value, np.int32), np.empty(npairs.value))
    check(K.lib.vqmc_load_spec(path.encode(), C.byref(n), ptr(a), ptr(b), ptr(pi), ptr(pj), ptr(pv), npairs.value,
                               C.byref(npairs)))
    spec = HamiltonianSpec(n.value, a, b, pi, pj, pv)
    spec.validate()
    return spec


def save_spec(spec: HamiltonianSpec, path: str) -> None:  # hamiltonian.cpp:162-177
    check(K.lib.vqmc_save_spec(path.encode(), spec.n, ptr(spec.alpha), ptr(spec.beta), ptr(spec.pair_i),
                               ptr(spec.pair_j), ptr(spec.pair_value), len(spec.pair_i)))


def diagonal_energy(spec: HamiltonianSpec, x) -> float:
    """H_xx (hamiltonian.cpp:61-69) of one configuration (host, fp64, the reference's order)."""
    x = np.asarray(x, np.float64).reshape(-1)
    if x.shape != (spec.n,):
        raise ValueError(f"configuration length {x.size} does not match spec n = {spec.n}")
    s = 1.0 - 2.0 * x
    e = 0.0
    for i in range(spec.n):
        e -= spec.beta[i] * s[i]
    for i, j, v in zip(spec.pair_i, spec.pair_j, spec.pair_value):
        e -= v * s[i] * s[j]
    return e


# ---------------------------------------------------------------------------
# L2 model (models.hpp)
# ---------------------------------------------------------------------------
class MadeModel:
    """Value type like the reference's MadeModel (models.hpp:34-46): n, h, degrees and the
    flattened fp64 parameters.  A device replica is created lazily and kept in sync."""

    def __init__(self, n: int, h: int, degrees, theta):
        self.n, self.h = int(n), int(h)
        self.degrees = np.ascontiguousarray(degrees, np.int32)
        self._theta = np.ascontiguousarray(theta, np.float64)
        self._version = 0
        self._dev: Optional["DeviceReplica"] = None

    def param_count(self) -> int:
        return 2 * self.h * self.n + self.h + self.n

    def clone(self) -> "MadeModel":
        return MadeModel(self.n, self.h, self.degrees.copy(), self.parameters().copy())

    def parameters(self) -> np.ndarray:
        if self._dev is not None and self._dev.device_newer:
            self._theta = self._dev.get_params()
            self._dev.device_newer = False
        return self._theta

    def _set(self, theta) -> None:
        theta = np.ascontiguousarray(theta, np.float64)
        if theta.shape != (self.param_count(),):
            raise ValueError("parameter vector length mismatch")
        self._theta = theta.copy()
        self._version += 1
        if self._dev is not None:  # the host copy is now the newer one: the next sync uploads it
            self._dev.device_newer = False

    def device(self, device: int = 0) -> "DeviceReplica":
        if self._dev is None:
            self._dev = DeviceReplica(self, device)
        self._dev.sync()
        return self._dev


class DeviceReplica:
    """One vqmc_gpu handle holding a model replica (and optionally a Max-Cut instance)."""

    def __init__(self, model: MadeModel, device: int = 0, max_batch: int = 1024):
        self.model = model
        self.h = C.c_void_p()
        empty = np.zeros((0, 2), np.int32)
        check(K.lib.vqmc_gpu_create(device, model.n, model.h, ptr(model.degrees), ptr(model._theta),
                                    ptr(empty), 0, max_batch, C.byref(self.h)))
        self.version = model._version
        self.problem_id = None
        self.device_newer = False

    def __del__(self):
        try:
            if self.h:
                K.lib.vqmc_gpu_destroy(self.h)
        except Exception:
            pass

    def sync(self) -> None:
        if self.version != self.model._version:
            check(K.lib.vqmc_gpu_set_params(self.h, ptr(self.model._theta)))
            self.version = self.model._version
            self.device_newer = False

    def set_problem(self, problem) -> None:
        """A MaxCutProblem (edges; the exact integer-cut path) or a HamiltonianSpec (TIM)."""
        if self.problem_id is not problem:
            if isinstance(problem, HamiltonianSpec):
                if problem.n != self.model.n:
                    raise ValueError("spec n does not match the model")
                check(K.lib.vqmc_gpu_set_spec(self.h, ptr(problem.alpha), ptr(problem.beta), ptr(problem.pair_i),
                                              ptr(problem.pair_j), ptr(problem.pair_value), len(problem.pair_i)))
            else:
                check(K.lib.vqmc_gpu_clear_spec(self.h))
                e = np.ascontiguousarray(problem.graph.edges, np.int32)
                check(K.lib.vqmc_gpu_set_edges(self.h, ptr(e), len(e)))
            self.problem_id = problem

    def get_params(self) -> np.ndarray:
        out = np.empty(self.model.param_count())
        check(K.lib.vqmc_gpu_get_params(self.h, ptr(out)))
        return out


def default_made_hidden(n: int) -> int:  # models.cpp:79-82
    return int(K.lib.vqmc_default_made_hidden(n))


def made_init(n: int, h: int, seed: int) -> MadeModel:  # models.cpp:84-104
    deg = np.empty(max(h, 0), np.int32)
    theta = np.empty(max(2 * h * n + h + n, 0), np.float64)
    check(K.lib.vqmc_made_init(n, h, seed, ptr(deg), ptr(theta)))
    return MadeModel(n, h, deg, theta)


def parameter_vector(model: MadeModel) -> np.ndarray:  # models.cpp:264-275
    return model.parameters().copy()


def set_parameters(model: MadeModel, params) -> None:  # models.cpp:287-300
    model._set(params)


def _bits(model: MadeModel, configs) -> tuple:
    x = np.asarray(configs)
    if x.ndim == 1:
        x = x[None, :]
    if x.shape[1] != model.n:
        raise ValueError(f"configuration width {x.shape[1]} does not match model n = {model.n}")
    return K.pack_bits(x), x.shape[0]


def log_psi_batch(model: MadeModel, configs) -> np.ndarray:  # models.cpp:122-124
    bits, B = _bits(model, configs)
    out = np.empty(B)
    check(K.lib.vqmc_gpu_log_psi(model.device().h, ptr(bits), B, ptr(out), None))
    return out


def log_prob(model: MadeModel, configs) -> np.ndarray:  # models.cpp:118-120
    return 2.0 * log_psi_batch(model, configs)


def conditionals(model: MadeModel, configs) -> np.ndarray:  # models.cpp:114-116
    bits, B = _bits(model, configs)
    lp = np.empty(B)
    cond = np.empty((B, model.n))
    check(K.lib.vqmc_gpu_log_psi(model.device().h, ptr(bits), B, ptr(lp), ptr(cond)))
    return cond


def log_psi(model: MadeModel, x) -> float:
    return float(log_psi_batch(model, np.asarray(x)[None, :])[0])


def weighted_grad_log_psi(model: MadeModel, configs, weights) -> np.ndarray:  # models.cpp:175-198
    bits, B = _bits(model, configs)
    w = np.ascontiguousarray(weights, np.float64)
    if w.shape != (B,):
        raise ValueError("weights length does not match the batch")
    g = np.empty(model.param_count())
    check(K.lib.vqmc_gpu_weighted_grad(model.device().h, ptr(bits), ptr(w), B, ptr(g)))
    return g


def grad_log_psi(model: MadeModel, x) -> np.ndarray:
    return weighted_grad_log_psi(model, np.asarray(x)[None, :], np.ones(1))


# ---------------------------------------------------------------------------
# L3 sampler (sampler.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class SampleBatch:
    configs: np.ndarray  # B x n uint8
    log_psi: np.ndarray
    kind: str = "auto"
    acceptance_rate: float = 1.0
    wall_time: float = 0.0
    bits: Optional[np.ndarray] = None  # packed words, as produced on the device


def auto_sample(model: MadeModel, batch_size: int, rng) -> SampleBatch:  # sampler.cpp:35-59
    """rng: Stream (the reference's mt19937_64 uniforms, consumed [bit][sample] like the
    reference) or PhiloxStream (production mode; advances its call counter)."""
    if batch_size < 1:
        raise ValueError("auto_sample requires batch_size >= 1")
    t0 = time.perf_counter()
    W = (model.n + 31) // 32
    bits = np.empty((batch_size, W), np.uint32)
    lp = np.empty(batch_size)
    dev = model.device()
    if isinstance(rng, PhiloxStream):
        check(K.lib.vqmc_gpu_sample(dev.h, batch_size, None, rng.seed, rng.stream, rng.call, ptr(bits), ptr(lp)))
        rng.call += 1
    else:
        u = rng.uniforms(model.n * batch_size)
        check(K.lib.vqmc_gpu_sample(dev.h, batch_size, ptr(u), 0, 0, 0, ptr(bits), ptr(lp)))
    return SampleBatch(K.unpack_bits(bits, model.n), lp, wall_time=time.perf_counter() - t0, bits=bits)


def forward_pass_count(kind: str, n: int, batch_size: int) -> int:  # sampler.cpp:124-128 (AUTO)
    if kind != "auto":
        raise ValueError("only the AUTO sampler is on this path")
    return n


# ---------------------------------------------------------------------------
# L4 estimator (estimator.hpp)
# ---------------------------------------------------------------------------
def local_energy_batch(problem, model: MadeModel, configs, cached_log_psi=None) -> np.ndarray:
    """local_energy_batch (estimator.hpp:43-90).  MaxCutProblem: the diagonal branch (exact
    integer cuts).  HamiltonianSpec: the diagonal plus the flipped-neighbour terms
    -alpha_k exp(log psi(x ^ e_k) - cached_log_psi) (cached_log_psi: SampleBatch::log_psi; None =
    the model's own log psi of the configurations)."""
    bits, B = _bits(model, configs)
    dev = model.device()
    dev.set_problem(problem)
    out = np.empty(B)
    if isinstance(problem, HamiltonianSpec):
        c = None if cached_log_psi is None else np.ascontiguousarray(cached_log_psi, np.float64)
        if c is not None and c.shape != (B,):
            raise ValueError("cached log psi length does not match the batch")
        check(K.lib.vqmc_gpu_local_energy(dev.h, ptr(bits), B, ptr(c), ptr(out)))
        return out
    check(K.lib.vqmc_gpu_maxcut_energy(dev.h, ptr(bits), B, None, ptr(out)))
    if not np.all(np.isfinite(out)):
        raise RuntimeError("non-finite local energy (amplitude underflow?)")
    return out


def cut_values(problem: MaxCutProblem, model: MadeModel, configs) -> np.ndarray:
    """cut_value (hamiltonian.cpp:121-124) for every row."""
    bits, B = _bits(model, configs)
    dev = model.device()
    dev.set_problem(problem)
    out = np.empty(B, np.int32)
    check(K.lib.vqmc_gpu_maxcut_energy(dev.h, ptr(bits), B, ptr(out), None))
    return out.astype(np.float64)


def energy_and_variance(local_energies) -> tuple:  # estimator.hpp:94-100
    l = np.asarray(local_energies, np.float64)
    if l.size < 2:
        raise ValueError("variance needs at least two samples")
    s = 0.0
    for v in l:  # sequential fp64 sum, like the reference's reduction on exact data
        s += v
    mean = s / l.size
    ss = float(np.sum((l - mean) ** 2))
    return mean, ss / (l.size - 1)


def gradient_from_locals(model: MadeModel, configs, local_energies) -> np.ndarray:  # estimator.hpp:111-119
    bits, B = _bits(model, configs)
    if B < 2:
        raise ValueError("gradient estimate needs at least two samples")
    l = np.ascontiguousarray(local_energies, np.float64)
    g = np.empty(model.param_count())
    check(K.lib.vqmc_gpu_gradient_from_locals(model.device().h, ptr(bits), ptr(l), B, ptr(g)))
    return g


# ---------------------------------------------------------------------------
# L5 optimizer (optimizer.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class AdamState:
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    t: int = 0


def adam_step(state: AdamState, model: MadeModel, grad) -> None:
    """adam_step (optimizer.cpp:21-35) applied to the model's device replica (moments live on
    the device; a fresh AdamState resets them)."""
    dev = model.device()
    if state.t == 0:
        check(K.lib.vqmc_gpu_adam_reset(dev.h))
    state.t += 1
    g = np.ascontiguousarray(grad, np.float64)
    if g.shape != (model.param_count(),):
        raise ValueError("gradient length mismatch")
    check(K.lib.vqmc_gpu_adam_step(dev.h, ptr(g), state.lr, state.beta1, state.beta2, state.eps, state.t))
    dev.device_newer = True


def sgd_step(params, grad, lr):  # optimizer.hpp:57-59
    return np.asarray(params) - lr * np.asarray(grad)


@dataclasses.dataclass
class SrConfig:  # optimizer.hpp:38-45
    lr: float = 0.1
    lam: float = 1e-3           # diagonal regularization (SrConfig::lambda)
    tol: float = 1e-6           # relative residual
    max_iterations: int = 200   # CG budget
    fallback: bool = False      # on CG failure, continue with the raw gradient
    centered: bool = True       # subtract the mean score before forming F


SrSolveError = K.SrSolveError


class FisherEstimate:
    """fisher_estimate(model, configs, centered) (estimator.hpp:146-174).  The B x d score matrix
    is never formed: the device applies F v = S^T (S v) / B through the model's structure."""

    def __init__(self, model: "MadeModel", configs, centered: bool = True):
        self.model = model
        self.bits, self.B = _bits(model, configs)
        if self.B < 2:
            raise ValueError("Fisher needs at least two samples")
        self.centered = centered

    def samples(self) -> int:
        return self.B

    def dim(self) -> int:
        return self.model.param_count()


def fisher_estimate(model: "MadeModel", configs, centered: bool = True) -> FisherEstimate:
    return FisherEstimate(model, configs, centered)


def sr_direction(cfg: SrConfig, grad, fisher: FisherEstimate, info: Optional[dict] = None) -> np.ndarray:
    """sr_direction (optimizer.cpp:64-82): solves (F + lambda I) delta = grad (CG on the GPU);
    raises SrSolveError unless ||(F + lambda I) delta - grad|| <= tol ||grad||."""
    g = np.ascontiguousarray(grad, np.float64)
    if g.shape != (fisher.dim(),):
        raise ValueError("gradient length mismatch")
    out = np.empty_like(g)
    it, res = C.c_int(0), C.c_double(0.0)
    rc = K.lib.vqmc_gpu_sr_direction(fisher.model.device().h, ptr(fisher.bits), fisher.B, ptr(g), cfg.lam, cfg.tol,
                                     cfg.max_iterations, 1 if fisher.centered else 0, ptr(out), C.byref(it),
                                     C.byref(res))
    if info is not None:
        info.update(iterations=it.value, residual=res.value)
    check(rc)
    return out


def sr_step(cfg: SrConfig, params, grad, fisher: FisherEstimate) -> np.ndarray:  # optimizer.cpp:84-92
    try:
        return np.asarray(params) - cfg.lr * sr_direction(cfg, grad, fisher)
    except SrSolveError:
        if not cfg.fallback:
            raise
        return np.asarray(params) - cfg.lr * np.asarray(grad)


# ---------------------------------------------------------------------------
# L6 trainer (trainer.hpp)
# ---------------------------------------------------------------------------
def allreduce_mean(vectors: List[np.ndarray]) -> np.ndarray:  # trainer.cpp:324-335 (fixed tree)
    if not vectors:
        raise ValueError("allreduce_mean needs at least one vector")
    level = [np.asarray(v, np.float64) for v in vectors]
    while len(level) > 1:
        nxt = [level[i] + level[i + 1] for i in range(0, len(level) - 1, 2)]
        if len(level) % 2 == 1:
            nxt.append(level[-1])
        level = nxt
    return level[0] / float(len(vectors))


@dataclasses.dataclass
class StepStats:
    energy_mean: float = 0.0
    energy_std: float = 0.0
    grad_norm: float = 0.0
    wall_time: float = 0.0


@dataclasses.dataclass
class RunConfig:
    """The MADE / AUTO / {ADAM, SGD + SR} slice of RunConfig (trainer.hpp:31-58).  `problem` is the
    reference's `maxcut` (a MaxCutProblem: exact cut path, best/mean cut reported) or its `spec`
    (a HamiltonianSpec, e.g. random_tim: local energies with the off-diagonal branch)."""
    problem: Optional[object] = None
    hidden: int = 0
    optimizer: str = "adam"
    lr: float = 0.0
    iterations: int = 300
    workers: int = 1            # data-parallel workers per rank (segments of one GPU batch)
    minibatch: int = 1024       # per worker
    eval_batch: int = 1024
    seed: int = 0
    target: Optional[float] = None
    uniforms: str = "philox"    # "philox" (production) or "mt19937" (reference streams, parity)
    sr: SrConfig = dataclasses.field(default_factory=SrConfig)
    gradient_observer: Optional[Callable[[int, np.ndarray], None]] = None
    device: int = 0


@dataclasses.dataclass
class RunResult:
    stats: List[StepStats]
    final_energy: float = 0.0
    final_energy_std: float = 0.0
    best_cut: Optional[float] = None
    mean_cut: Optional[float] = None
    total_time: float = 0.0
    replicas_identical: bool = True
    final_params: Optional[np.ndarray] = None
    hit_time: Optional[float] = None
    hit_iteration: int = -1
    made: Optional[MadeModel] = None


def resolve_lr(cfg: RunConfig) -> float:  # trainer.cpp:35-46
    if cfg.lr > 0.0:
        return cfg.lr
    return 0.01 if cfg.optimizer == "adam" else 0.1


def _mt_uniforms(streams: List[Stream], n: int, mbs: int) -> np.ndarray:
    """[n][L*mbs] uniforms: worker w's block is its stream's next n*mbs draws ([bit][sample])."""
    u = np.empty((n, len(streams) * mbs))
    for w, s in enumerate(streams):
        u[:, w * mbs:(w + 1) * mbs] = s.uniforms(n * mbs).reshape(n, mbs)
    return np.ascontiguousarray(u)


def train(cfg: RunConfig, comm=None) -> RunResult:
    """vqmc::train for MADE + AUTO + ADAM or SGD + SR on a Max-Cut instance (trainer.cpp:111-322),
    one fused device step per iteration.

    `comm` (optional, one process per GPU): a ``dp.Communicator`` or a tuple (rank, world,
    nccl_unique_id) with rank 0's ``vqmc_gpu_comm_unique_id`` shared by every rank (see
    ``dp.make_communicator``).  This rank then plays reference workers rank*L .. rank*L + L - 1,
    its handle joins the NCCL communicator (one all-reduce per step: the gradient and the exact
    cut statistics), and the returned StepStats are pooled over all world*L*minibatch samples,
    like the reference's (trainer.cpp:246-256)."""
    if cfg.problem is None:
        raise ValueError("a problem (MaxCutProblem or HamiltonianSpec) is required")
    if isinstance(cfg.problem, HamiltonianSpec):
        cfg.problem.validate()
        if cfg.optimizer != "adam":
            raise ValueError("general (TIM) specs train with ADAM on the B200 path")
    if cfg.workers < 1:
        raise ValueError("workers must be >= 1")
    if cfg.iterations < 1:
        raise ValueError("iterations must be >= 1")
    if cfg.minibatch < 2:
        raise ValueError("minibatch must be >= 2")
    if cfg.optimizer not in ("adam", "sgd_sr"):
        raise ValueError("the B200 path implements the ADAM and SGD + SR optimizers")
    n = cfg.problem.n if isinstance(cfg.problem, HamiltonianSpec) else cfg.problem.graph.n
    h = cfg.hidden if cfg.hidden > 0 else default_made_hidden(n)
    model = made_init(n, h, cfg.seed)
    lr = resolve_lr(cfg)
    rank, world, uid = _comm_parts(comm)
    dev = model.device(cfg.device)
    dev.set_problem(cfg.problem)
    if uid is not None:
        ub = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        check(K.lib.vqmc_gpu_comm_init(dev.h, ub, world, rank))
    check(K.lib.vqmc_gpu_adam_reset(dev.h))
    L, mbs = cfg.workers, cfg.minibatch
    stream0 = 1 + rank * L
    streams = [Stream(cfg.seed, stream0 + w) for w in range(L)]
    eval_stream = Stream(cfg.seed, kEvalStream)
    st = K.StepStats()
    result = RunResult(stats=[])
    t_run = time.perf_counter()
    acc_time = 0.0
    for it in range(cfg.iterations):
        t0 = time.perf_counter()
        u = _mt_uniforms(streams, n, mbs) if cfg.uniforms == "mt19937" else None
        if cfg.optimizer == "sgd_sr":  # trainer.cpp:165-168, 189-199, 223-225
            cg_it, cg_res = C.c_int(0), C.c_double(0.0)
            check(K.lib.vqmc_gpu_train_step_sr(dev.h, mbs, L, ptr(u), cfg.seed, stream0, it, lr, cfg.sr.lam,
                                               cfg.sr.tol, cfg.sr.max_iterations, 1 if cfg.sr.fallback else 0,
                                               1 if cfg.sr.centered else 0, C.byref(st), C.byref(cg_it),
                                               C.byref(cg_res)))
        else:
            check(K.lib.vqmc_gpu_train_step(dev.h, mbs, L, ptr(u), cfg.seed, stream0, it, lr, 0.9, 0.999, 1e-8,
                                            it + 1, C.byref(st)))
        dev.device_newer = True
        wall = time.perf_counter() - t0
        if cfg.gradient_observer is not None:  # trainer.cpp:187-188 (worker 0, outside the timing)
            g = np.empty(model.param_count())
            check(K.lib.vqmc_gpu_last_gradient(dev.h, ptr(g)))
            cfg.gradient_observer(it, g)
        result.stats.append(StepStats(st.energy_mean, math.sqrt(st.energy_var), st.grad_norm, wall))
        acc_time += wall
        if cfg.target is not None:
            ev = evaluate(cfg, model, eval_stream)
            hit = ev[0] <= cfg.target if isinstance(cfg.problem, HamiltonianSpec) else ev[2] >= cfg.target
            if hit:  # trainer.cpp:265-273
                result.hit_time, result.hit_iteration = acc_time, it + 1
                break
    ev = evaluate(cfg, model, eval_stream)
    result.final_energy, result.final_energy_std, result.best_cut, result.mean_cut = ev
    if isinstance(cfg.problem, HamiltonianSpec):  # no cut (trainer.cpp:296-299 only for maxcut)
        result.best_cut = result.mean_cut = None
    result.final_params = model.parameters().copy()
    result.total_time = time.perf_counter() - t_run
    result.made = model
    return result


def _comm_parts(comm):
    """(rank, world, unique_id or None) of train()'s `comm` argument."""
    if comm is None:
        return 0, 1, None
    if hasattr(comm, "rank"):
        rank, world, uid = comm.rank, comm.world, getattr(comm, "unique_id", None)
    else:
        if len(comm) != 3:
            raise ValueError("comm must be (rank, world, nccl_unique_id)")
        rank, world, uid = comm
    rank, world = int(rank), int(world)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad (rank, world)")
    if world > 1 and uid is None:
        raise ValueError("a multi-rank run needs the NCCL unique id of rank 0 (dp.make_communicator)")
    if uid is not None and len(bytes(uid)) != 128:
        raise ValueError("the NCCL unique id has 128 bytes")
    return rank, world, uid


def evaluate(cfg: RunConfig, model: MadeModel, eval_stream) -> tuple:  # trainer.cpp:91-108
    dev = model.device()
    dev.set_problem(cfg.problem)
    out = np.empty(4)
    B = cfg.eval_batch
    if isinstance(eval_stream, PhiloxStream):
        check(K.lib.vqmc_gpu_evaluate(dev.h, B, None, eval_stream.seed, eval_stream.stream, eval_stream.call,
                                      ptr(out)))
        eval_stream.call += 1
    elif cfg.uniforms == "mt19937":
        u = eval_stream.uniforms(model.n * B)
        check(K.lib.vqmc_gpu_evaluate(dev.h, B, ptr(u), 0, 0, 0, ptr(out)))
    else:
        # production: Philox on the eval stream, counter = number of eval calls so far
        call = getattr(eval_stream, "_calls", 0)
        check(K.lib.vqmc_gpu_evaluate(dev.h, B, None, eval_stream.seed, eval_stream.stream, call, ptr(out)))
        eval_stream._calls = call + 1
    return tuple(float(v) for v in out)
