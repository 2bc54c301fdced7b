// vqmc_b200/vqmc.hpp — header-only C++ facade with the reference's API names
// (namespace vqmc, proj/include/vqmc/*.hpp) over the C ABI of libvqmc_b200.so.
//
// Scope: the north-star path (Max-Cut, MADE, AUTO sampler, ADAM / SGD + SR), general Ising (TIM)
// specs, and one host thread per GPU for multi-GPU training.  Eigen is not available,
// so Vector is std::vector<double> and ConfigBatch a small row-major 0/1 matrix; names,
// argument meaning, default values and exception types follow the reference:
// std::invalid_argument for usage errors, std::runtime_error for numerical / device errors.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iomanip>
#include <memory>
#include <optional>
#include <random>
#include <thread>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vqmc_b200.h"

namespace vqmc {

using Vector = std::vector<double>;

/// SR conjugate gradient did not converge (optimizer.hpp:46-55).
struct SrSolveError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == VQMC_OK) return;
  if (rc == VQMC_ERR_INVALID) throw std::invalid_argument(vqmc_last_error());
  if (rc == VQMC_ERR_SR) throw SrSolveError(vqmc_last_error());
  throw std::runtime_error(vqmc_last_error());
}

// ---- L0 common (common.hpp) -------------------------------------------------------
/// B x n configurations, entries 0/1, row-major (the reference's ConfigBatch is a B x n
/// Eigen matrix of 0.0/1.0 doubles).
struct ConfigBatch {
  int rows_ = 0, cols_ = 0;
  std::vector<uint8_t> x;
  ConfigBatch() = default;
  ConfigBatch(int r, int c) : rows_(r), cols_(c), x((size_t)r * c, 0) {}
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  uint8_t& operator()(int r, int c) { return x[(size_t)r * cols_ + c]; }
  uint8_t operator()(int r, int c) const { return x[(size_t)r * cols_ + c]; }
  std::vector<uint32_t> packed() const {
    const int W = (cols_ + 31) / 32;
    std::vector<uint32_t> w((size_t)rows_ * W, 0u);
    for (int r = 0; r < rows_; ++r)
      for (int c = 0; c < cols_; ++c)
        if ((*this)(r, c)) w[(size_t)r * W + (c >> 5)] |= 1u << (c & 31);
    return w;
  }
  static ConfigBatch from_packed(const std::vector<uint32_t>& w, int rows, int cols) {
    ConfigBatch b(rows, cols);
    const int W = (cols + 31) / 32;
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) b(r, c) = (w[(size_t)r * W + (c >> 5)] >> (c & 31)) & 1u;
    return b;
  }
};

inline uint64_t mix_seed(uint64_t seed, uint64_t stream) { return vqmc_mix_seed(seed, stream); }
inline std::mt19937_64 make_stream(uint64_t seed, uint64_t stream = 0) {
  return std::mt19937_64(mix_seed(seed, stream));
}

// ---- L1 problem (hamiltonian.hpp) -------------------------------------------------
struct Graph {
  int n = 0;
  std::vector<std::pair<int, int>> edges;
};
struct MaxCutProblem {
  Graph graph;
  std::size_t num_edges = 0;
};

namespace detail {
inline std::vector<int32_t> flat(const Graph& g) {
  std::vector<int32_t> e;
  e.reserve(2 * g.edges.size());
  for (const auto& [i, j] : g.edges) {
    e.push_back(i);
    e.push_back(j);
  }
  return e;
}
inline Graph unflat(int n, const std::vector<int32_t>& e) {
  Graph g;
  g.n = n;
  for (size_t t = 0; t + 1 < e.size(); t += 2) g.edges.emplace_back(e[t], e[t + 1]);
  return g;
}
template <class F>
Graph generate(int n, F&& fn) {
  int64_t ne = 0;
  check(fn(nullptr, 0, &ne));
  std::vector<int32_t> e((size_t)(2 * ne));
  check(fn(e.data(), ne, &ne));
  return unflat(n, e);
}
}  // namespace detail

inline Graph random_maxcut_graph(int n, uint64_t seed) {  // hamiltonian.cpp:144-160
  return detail::generate(n, [&](int32_t* e, int64_t cap, int64_t* ne) {
    return vqmc_random_maxcut_graph(n, seed, e, cap, ne);
  });
}
inline Graph random_regular_graph(int n, int d, uint64_t seed) {
  return detail::generate(n, [&](int32_t* e, int64_t cap, int64_t* ne) {
    return vqmc_random_regular_graph(n, d, seed, e, cap, ne);
  });
}
inline Graph load_graph(const std::string& path) {  // hamiltonian.cpp:243-266
  int n = 0;
  int64_t ne = 0;
  check(vqmc_load_graph(path.c_str(), &n, nullptr, 0, &ne));
  std::vector<int32_t> e((size_t)(2 * ne));
  check(vqmc_load_graph(path.c_str(), &n, e.data(), ne, &ne));
  return detail::unflat(n, e);
}
inline void save_graph(const Graph& g, const std::string& path) {
  const auto e = detail::flat(g);
  check(vqmc_save_graph(path.c_str(), g.n, e.data(), (int64_t)g.edges.size()));
}
inline MaxCutProblem maxcut_spec(const Graph& g) {  // hamiltonian.cpp:109-119 (validate :36-54)
  std::vector<std::pair<int, int>> s = g.edges;
  for (const auto& [i, j] : s)
    if (i < 0 || j >= g.n || i >= j) throw std::invalid_argument("pair indices must satisfy 0 <= i < j < n");
  std::sort(s.begin(), s.end());
  if (std::adjacent_find(s.begin(), s.end()) != s.end()) throw std::invalid_argument("duplicate pair");
  return MaxCutProblem{g, g.edges.size()};
}

/// One ZZ coupling term, 0-based, i < j (hamiltonian.hpp:26-31).
struct PairCoupling {
  int i;
  int j;
  double value;
};
/// H = -sum_i (alpha_i X_i + beta_i Z_i) - sum_{i<j} beta_ij Z_i Z_j (hamiltonian.hpp:34-44).
struct HamiltonianSpec {
  int n = 0;
  Vector alpha, beta;
  std::vector<PairCoupling> pairs;
  void validate() const {  // hamiltonian.cpp:36-54
    if (n < 1) throw std::invalid_argument("spec requires n >= 1");
    if ((int)alpha.size() != n || (int)beta.size() != n)
      throw std::invalid_argument("alpha/beta length does not match n");
    for (double a : alpha)
      if (a < 0.0) throw std::invalid_argument("alpha must be non-negative");
    std::vector<std::pair<int, int>> s;
    for (const auto& p : pairs) {
      if (p.i < 0 || p.j >= n || p.i >= p.j) throw std::invalid_argument("pair indices must satisfy 0 <= i < j < n");
      s.emplace_back(p.i, p.j);
    }
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) throw std::invalid_argument("duplicate pair");
  }
};

namespace detail {
struct SpecArrays {
  std::vector<int32_t> pi, pj;
  Vector pv;
};
inline SpecArrays arrays(const HamiltonianSpec& s) {
  SpecArrays a;
  for (const auto& p : s.pairs) {
    a.pi.push_back(p.i);
    a.pj.push_back(p.j);
    a.pv.push_back(p.value);
  }
  return a;
}
inline HamiltonianSpec from_arrays(int n, Vector alpha, Vector beta, const std::vector<int32_t>& pi,
                                   const std::vector<int32_t>& pj, const Vector& pv) {
  HamiltonianSpec s;
  s.n = n;
  s.alpha = std::move(alpha);
  s.beta = std::move(beta);
  s.pairs.reserve(pi.size());
  for (size_t t = 0; t < pi.size(); ++t) s.pairs.push_back({pi[t], pj[t], pv[t]});
  return s;
}
}  // namespace detail

inline HamiltonianSpec random_tim(int n, uint64_t seed) {  // hamiltonian.cpp:126-142
  if (n < 1) throw std::invalid_argument("random_tim requires n >= 1");
  const size_t np = (size_t)n * (n - 1) / 2;
  Vector a((size_t)n), b((size_t)n), pv(np);
  std::vector<int32_t> pi(np), pj(np);
  check(vqmc_random_tim(n, seed, a.data(), b.data(), pi.data(), pj.data(), pv.data()));
  return detail::from_arrays(n, std::move(a), std::move(b), pi, pj, pv);
}
inline HamiltonianSpec load_spec(const std::string& path) {  // hamiltonian.cpp:204-234
  int n = 0;
  int64_t np = 0;
  check(vqmc_load_spec(path.c_str(), &n, nullptr, nullptr, nullptr, nullptr, nullptr, 0, &np));
  Vector a((size_t)n), b((size_t)n), pv((size_t)np);
  std::vector<int32_t> pi((size_t)np), pj((size_t)np);
  check(vqmc_load_spec(path.c_str(), &n, a.data(), b.data(), pi.data(), pj.data(), pv.data(), np, &np));
  HamiltonianSpec s = detail::from_arrays(n, std::move(a), std::move(b), pi, pj, pv);
  s.validate();
  return s;
}
inline void save_spec(const HamiltonianSpec& s, const std::string& path) {  // hamiltonian.cpp:162-177
  const auto a = detail::arrays(s);
  check(vqmc_save_spec(path.c_str(), s.n, s.alpha.data(), s.beta.data(), a.pi.data(), a.pj.data(), a.pv.data(),
                       (int64_t)s.pairs.size()));
}

// ---- L2 model (models.hpp) --------------------------------------------------------
class GpuReplica;

struct MadeModel {
  int n = 0;
  int h = 0;
  std::vector<int> degrees;
  Vector theta;  // flattened parameters (models.cpp:264-275)
  int param_count() const { return 2 * h * n + h + n; }
  mutable std::shared_ptr<GpuReplica> replica;  // device copy, re-synchronised on demand
};

inline int default_made_hidden(int n) { return vqmc_default_made_hidden(n); }

inline MadeModel made_init(int n, int h, uint64_t seed) {  // models.cpp:84-104
  MadeModel m;
  m.n = n;
  m.h = h;
  if (n < 2) throw std::invalid_argument("made_init requires n >= 2");
  if (h < 1) throw std::invalid_argument("made_init requires h >= 1");
  std::vector<int32_t> deg(h);
  m.theta.resize((size_t)m.param_count());
  check(vqmc_made_init(n, h, seed, deg.data(), m.theta.data()));
  m.degrees.assign(deg.begin(), deg.end());
  return m;
}
inline Vector parameter_vector(const MadeModel& m) { return m.theta; }
inline void set_parameters(MadeModel& m, const Vector& p) {
  if ((int)p.size() != m.param_count()) throw std::invalid_argument("parameter vector length mismatch");
  m.theta = p;
}

/// One device handle holding a replica of a model (and optionally a Max-Cut instance).
class GpuReplica {
 public:
  explicit GpuReplica(const MadeModel& m, int device = 0, int max_batch = 1024) : n_(m.n) {
    std::vector<int32_t> deg(m.degrees.begin(), m.degrees.end());
    check(vqmc_gpu_create(device, m.n, m.h, deg.data(), m.theta.data(), nullptr, 0, max_batch, &h_));
    theta_ = m.theta;
  }
  ~GpuReplica() { vqmc_gpu_destroy(h_); }
  GpuReplica(const GpuReplica&) = delete;
  GpuReplica& operator=(const GpuReplica&) = delete;
  vqmc_gpu_t* get() const { return h_; }
  void sync(const MadeModel& m) {
    if (m.theta != theta_) {
      check(vqmc_gpu_set_params(h_, m.theta.data()));
      theta_ = m.theta;
    }
  }
  void set_problem(const MaxCutProblem& p) {
    if (spec_set_) {
      check(vqmc_gpu_clear_spec(h_));
      spec_set_ = false;
    }
    const auto e = detail::flat(p.graph);
    if (e != edges_) {
      check(vqmc_gpu_set_edges(h_, e.data(), (int64_t)p.graph.edges.size()));
      edges_ = e;
    }
  }
  void set_problem(const HamiltonianSpec& s) {
    if (s.n != n_) throw std::invalid_argument("spec n does not match the model");
    const auto a = detail::arrays(s);
    check(vqmc_gpu_set_spec(h_, s.alpha.data(), s.beta.data(), a.pi.data(), a.pj.data(), a.pv.data(),
                            (int64_t)s.pairs.size()));
    spec_set_ = true;
  }
  Vector params(int d) const {
    Vector t((size_t)d);
    check(vqmc_gpu_get_params(h_, t.data()));
    return t;
  }
  void mark_device_updated(const Vector& t) { theta_ = t; }

 private:
  vqmc_gpu_t* h_ = nullptr;
  int n_;
  Vector theta_;
  std::vector<int32_t> edges_;
  bool spec_set_ = false;
};

inline GpuReplica& replica(const MadeModel& m) {
  if (!m.replica) m.replica = std::make_shared<GpuReplica>(m);
  m.replica->sync(m);
  return *m.replica;
}

inline Vector log_psi_batch(const MadeModel& m, const ConfigBatch& c) {  // models.cpp:122-124
  if (c.cols() != m.n) throw std::invalid_argument("configuration width does not match model n");
  const auto w = c.packed();
  Vector out((size_t)c.rows());
  check(vqmc_gpu_log_psi(replica(m).get(), w.data(), c.rows(), out.data(), nullptr));
  return out;
}
inline Vector log_prob(const MadeModel& m, const ConfigBatch& c) {
  Vector v = log_psi_batch(m, c);
  for (double& x : v) x *= 2.0;
  return v;
}
inline Vector weighted_grad_log_psi(const MadeModel& m, const ConfigBatch& c, const Vector& w) {
  if ((int)w.size() != c.rows()) throw std::invalid_argument("weights length does not match the batch");
  const auto bits = c.packed();
  Vector g((size_t)m.param_count());
  check(vqmc_gpu_weighted_grad(replica(m).get(), bits.data(), w.data(), c.rows(), g.data()));
  return g;
}

// ---- L3 sampler (sampler.hpp) ------------------------------------------------------
struct SampleBatch {
  ConfigBatch configs;
  Vector log_psi;
  double acceptance_rate = 1.0;
  double wall_time = 0.0;
};

/// auto_sample (sampler.cpp:35-59): the caller's mt19937_64 is consumed exactly like the
/// reference's (one U[0,1) per bit and sample, bit-major), so samples match it.
inline SampleBatch auto_sample(const MadeModel& m, int B, std::mt19937_64& rng) {
  if (B < 1) throw std::invalid_argument("auto_sample requires batch_size >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<double> u((size_t)m.n * B);
  for (double& v : u) v = unit(rng);
  const int W = (m.n + 31) / 32;
  std::vector<uint32_t> bits((size_t)B * W);
  SampleBatch out;
  out.log_psi.resize((size_t)B);
  check(vqmc_gpu_sample(replica(m).get(), B, u.data(), 0, 0, 0, bits.data(), out.log_psi.data()));
  out.configs = ConfigBatch::from_packed(bits, B, m.n);
  out.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// ---- L4 estimator (estimator.hpp) --------------------------------------------------
struct StepStats {
  double energy_mean = 0.0, energy_std = 0.0, grad_norm = 0.0, wall_time = 0.0;
};

inline Vector local_energy_batch(const MaxCutProblem& p, const MadeModel& m, const ConfigBatch& c,
                                 const Vector& /*cached_log_psi*/ = {}) {  // estimator.hpp:43-57
  auto& r = replica(m);
  r.set_problem(p);
  const auto bits = c.packed();
  Vector out((size_t)c.rows());
  check(vqmc_gpu_maxcut_energy(r.get(), bits.data(), c.rows(), nullptr, out.data()));
  for (double v : out)
    if (!std::isfinite(v)) throw std::runtime_error("non-finite local energy (amplitude underflow?)");
  return out;
}
/// local_energy_batch (estimator.hpp:43-90) on a general spec: the diagonal plus the flipped-
/// neighbour terms, with the sampler's cached log psi (empty: the model's own).
inline Vector local_energy_batch(const HamiltonianSpec& s, const MadeModel& m, const ConfigBatch& c,
                                 const Vector& cached_log_psi = {}) {
  if (c.cols() != s.n) throw std::invalid_argument("configuration width does not match spec n");
  auto& r = replica(m);
  r.set_problem(s);
  const auto bits = c.packed();
  Vector out((size_t)c.rows());
  check(vqmc_gpu_local_energy(r.get(), bits.data(), c.rows(), cached_log_psi.empty() ? nullptr : cached_log_psi.data(),
                              out.data()));
  return out;
}
inline std::pair<double, double> energy_and_variance(const Vector& l) {  // estimator.hpp:94-100
  if (l.size() < 2) throw std::invalid_argument("variance needs at least two samples");
  double s = 0.0;
  for (double v : l) s += v;
  const double mean = s / (double)l.size();
  double ss = 0.0;
  for (double v : l) ss += (v - mean) * (v - mean);
  return {mean, ss / (double)(l.size() - 1)};
}
inline Vector gradient_from_locals(const MadeModel& m, const ConfigBatch& c, const Vector& l) {
  if (c.rows() < 2) throw std::invalid_argument("gradient estimate needs at least two samples");
  const auto bits = c.packed();
  Vector g((size_t)m.param_count());
  check(vqmc_gpu_gradient_from_locals(replica(m).get(), bits.data(), l.data(), c.rows(), g.data()));
  return g;
}

// ---- L5 optimizer (optimizer.hpp) ---------------------------------------------------
struct AdamState {
  double lr = 0.01, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  long t = 0;
  std::shared_ptr<GpuReplica> device;  // moments live on the device of this replica
};

/// adam_step on a (model-sized) parameter vector; the moments live with the device replica.
inline void adam_step(AdamState& st, MadeModel& m, const Vector& grad) {
  auto& r = replica(m);
  if (!st.device || st.device.get() != m.replica.get()) {
    st.device = m.replica;
    check(vqmc_gpu_adam_reset(r.get()));
  }
  st.t += 1;
  check(vqmc_gpu_adam_step(r.get(), grad.data(), st.lr, st.beta1, st.beta2, st.eps, st.t));
  m.theta = r.params(m.param_count());
  r.mark_device_updated(m.theta);
}

// ---- L6 trainer (trainer.hpp) -------------------------------------------------------
inline Vector allreduce_mean(const std::vector<Vector>& vs) {  // trainer.cpp:324-335
  if (vs.empty()) throw std::invalid_argument("allreduce_mean needs at least one vector");
  std::vector<Vector> level = vs;
  while (level.size() > 1) {
    std::vector<Vector> next;
    for (size_t i = 0; i + 1 < level.size(); i += 2) {
      Vector s(level[i].size());
      for (size_t t = 0; t < s.size(); ++t) s[t] = level[i][t] + level[i + 1][t];
      next.push_back(std::move(s));
    }
    if (level.size() % 2 == 1) next.push_back(level.back());
    level = std::move(next);
  }
  Vector out = level.front();
  for (double& v : out) v /= (double)vs.size();
  return out;
}

enum class OptimizerKind { kAdam, kSgdSr };  // (kSgd and RBM/MCMC are outside the B200 path)

struct SrConfig {  // optimizer.hpp:38-45
  double lr = 0.1;
  double lambda = 1e-3;
  double tol = 1e-6;
  int max_iterations = 200;
  bool fallback = false;
  bool centered = true;
};

struct RunConfig {  // the MADE / AUTO / {ADAM, SGD + SR} slice of trainer.hpp:31-58
  std::optional<MaxCutProblem> maxcut;  // Max-Cut instance (exact cut path; best / mean cut reported)
  std::optional<HamiltonianSpec> spec;  // otherwise a general spec (TIM), ADAM
  int hidden = 0;
  OptimizerKind optimizer = OptimizerKind::kAdam;
  SrConfig sr;
  double lr = 0.0;
  int iterations = 300;
  int workers = 1;
  int minibatch = 1024;
  int eval_batch = 1024;
  uint64_t seed = 0;
  std::optional<double> target;
  bool reference_streams = false;  // true: the reference's mt19937_64 uniforms (bit parity), else Philox
  int device = 0;                  // first GPU
  int gpus = 1;  // GPUs (devices device .. device + gpus - 1), one host thread and NCCL rank each;
                 // the `workers` reference workers are split evenly over them (trainer.cpp:284-287)
};

struct PhaseTimings {
  double sample = 0.0, estimate = 0.0, reduce = 0.0, update = 0.0;
};

struct RunResult {
  std::vector<StepStats> stats;
  double final_energy = 0.0, final_energy_std = 0.0;
  std::optional<double> best_cut, mean_cut;
  double total_time = 0.0;
  PhaseTimings phases;
  bool replicas_identical = true;  // one replica per device; NCCL gives every rank the same update
  Vector final_params;
  std::optional<double> hit_time;
  int hit_iteration = -1;
  std::optional<MadeModel> made;
};

constexpr uint64_t kEvalStream = 1'000'000'007ULL;  // trainer.cpp:48

inline double resolve_lr(const RunConfig& c) {  // trainer.cpp:35-46
  return c.lr > 0.0 ? c.lr : (c.optimizer == OptimizerKind::kAdam ? 0.01 : 0.1);
}

namespace detail {
/// Which reference workers a GPU rank plays (trainer.cpp:121-127): rank r of G runs workers
/// r * L / G .. (r + 1) * L / G - 1 as segments of its batch; worker w draws from
/// make_stream(seed, w + 1), so the rank's first stream is 1 + r * L / G.
struct RankPlan {
  int rank = 0, gpus = 1, workers = 1, device = 0;
  uint64_t stream0 = 1;
};
inline RankPlan rank_plan(const RunConfig& cfg, int rank) {
  if (cfg.gpus < 1) throw std::invalid_argument("gpus must be >= 1");
  if (cfg.workers % cfg.gpus != 0) throw std::invalid_argument("workers must be a multiple of gpus");
  RankPlan p;
  p.rank = rank;
  p.gpus = cfg.gpus;
  p.workers = cfg.workers / cfg.gpus;
  p.device = cfg.device + rank;
  p.stream0 = 1 + (uint64_t)rank * (uint64_t)p.workers;
  return p;
}

/// One rank's training loop (worker_body, trainer.cpp:150-282): with a communicator every step
/// all-reduces the gradient and the energy statistics, so each rank sees the pooled StepStats
/// and applies the same update (replicas stay identical).
inline RunResult train_rank(const RunConfig& cfg, const RankPlan& plan, const uint8_t* uid) {
  const auto run0 = std::chrono::steady_clock::now();
  const bool maxcut = cfg.maxcut.has_value();
  const int n = maxcut ? cfg.maxcut->graph.n : cfg.spec->n;
  const int h = cfg.hidden > 0 ? cfg.hidden : default_made_hidden(n);
  MadeModel model = made_init(n, h, cfg.seed);  // trainer.cpp:318
  model.replica = std::make_shared<GpuReplica>(model, plan.device);
  auto& r = replica(model);
  if (maxcut) r.set_problem(*cfg.maxcut);
  else r.set_problem(*cfg.spec);
  if (plan.gpus > 1) check(vqmc_gpu_comm_init(r.get(), uid, plan.gpus, plan.rank));
  check(vqmc_gpu_adam_reset(r.get()));
  const double lr = resolve_lr(cfg);
  const int L = plan.workers, mbs = cfg.minibatch;
  std::vector<std::mt19937_64> rngs;
  for (int w = 0; w < L; ++w) rngs.push_back(make_stream(cfg.seed, plan.stream0 + w));
  auto eval_rng = make_stream(cfg.seed, kEvalStream);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  RunResult res;
  double acc_time = 0.0;
  uint64_t eval_calls = 0;
  auto evaluate = [&](double out[4]) {  // trainer.cpp:91-108 (every rank: identical replicas and stream)
    if (cfg.reference_streams) {
      std::vector<double> u((size_t)n * cfg.eval_batch);
      for (double& v : u) v = unit(eval_rng);
      check(vqmc_gpu_evaluate(r.get(), cfg.eval_batch, u.data(), 0, 0, 0, out));
    } else {
      check(vqmc_gpu_evaluate(r.get(), cfg.eval_batch, nullptr, cfg.seed, kEvalStream, eval_calls++, out));
    }
  };
  std::vector<double> u;
  for (int it = 0; it < cfg.iterations; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    const double* up = nullptr;
    if (cfg.reference_streams) {  // worker w's block: its stream's next n * mbs draws, [bit][sample]
      u.assign((size_t)n * L * mbs, 0.0);
      for (int w = 0; w < L; ++w)
        for (int i = 0; i < n; ++i)
          for (int b = 0; b < mbs; ++b) u[(size_t)i * L * mbs + (size_t)w * mbs + b] = unit(rngs[w]);
      up = u.data();
    }
    vqmc_step_stats_t st{};
    if (cfg.optimizer == OptimizerKind::kSgdSr) {  // trainer.cpp:165-168, 189-199, 223-225
      int cg_it = 0;
      double cg_res = 0.0;
      check(vqmc_gpu_train_step_sr(r.get(), mbs, L, up, cfg.seed, plan.stream0, (uint64_t)it, lr, cfg.sr.lambda,
                                   cfg.sr.tol, cfg.sr.max_iterations, cfg.sr.fallback ? 1 : 0,
                                   cfg.sr.centered ? 1 : 0, &st, &cg_it, &cg_res));
    } else {
      check(vqmc_gpu_train_step(r.get(), mbs, L, up, cfg.seed, plan.stream0, (uint64_t)it, lr, 0.9, 0.999, 1e-8,
                                it + 1, &st));
    }
    StepStats s;
    s.energy_mean = st.energy_mean;
    s.energy_std = std::sqrt(st.energy_var);
    s.grad_norm = st.grad_norm;
    s.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    acc_time += s.wall_time;
    res.stats.push_back(s);
    if (cfg.target) {  // trainer.cpp:265-273
      double ev[4];
      evaluate(ev);
      if (maxcut ? ev[2] >= *cfg.target : ev[0] <= *cfg.target) {
        res.hit_time = acc_time;
        res.hit_iteration = it + 1;
        break;
      }
    }
  }
  double ev[4];
  evaluate(ev);
  res.final_energy = ev[0];
  res.final_energy_std = ev[1];
  if (maxcut) {
    res.best_cut = ev[2];
    res.mean_cut = ev[3];
  }
  model.theta = r.params(model.param_count());
  r.mark_device_updated(model.theta);
  res.final_params = model.theta;
  res.made = model;
  res.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - run0).count();
  return res;
}
}  // namespace detail

/// train (trainer.cpp:111-322) for MADE + AUTO + ADAM or SGD + SR on a Max-Cut instance, or ADAM on
/// a general spec: one fused device step per iteration.  gpus = G > 1 runs one host thread per GPU
/// (the reference's worker threads, trainer.cpp:284-287), each an NCCL rank playing workers / G of
/// the reference workers; replicas_identical compares the ranks' final parameters bitwise.
inline RunResult train(const RunConfig& cfg) {
  if (!cfg.maxcut && !cfg.spec) throw std::invalid_argument("a Max-Cut instance or a Hamiltonian spec is required");
  if (!cfg.maxcut) {
    cfg.spec->validate();
    if (cfg.optimizer != OptimizerKind::kAdam)
      throw std::invalid_argument("general (TIM) specs train with ADAM on the B200 path");
  }
  if (cfg.workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (cfg.iterations < 1) throw std::invalid_argument("iterations must be >= 1");
  if (cfg.minibatch < 2) throw std::invalid_argument("minibatch must be >= 2");
  if (cfg.gpus == 1) return detail::train_rank(cfg, detail::rank_plan(cfg, 0), nullptr);
  std::vector<detail::RankPlan> plans;
  for (int g = 0; g < cfg.gpus; ++g) plans.push_back(detail::rank_plan(cfg, g));
  int visible = 0;
  check(vqmc_gpu_device_count(&visible));
  if (cfg.device + cfg.gpus > visible)
    throw std::invalid_argument("gpus: " + std::to_string(cfg.gpus) + " devices from " + std::to_string(cfg.device) +
                                " requested, " + std::to_string(visible) + " visible");
  uint8_t uid[128];
  check(vqmc_gpu_comm_unique_id(uid));
  std::vector<RunResult> rs((size_t)cfg.gpus);
  std::vector<std::exception_ptr> errs((size_t)cfg.gpus);
  std::vector<std::thread> threads;
  for (int g = 0; g < cfg.gpus; ++g)
    threads.emplace_back([&, g] {
      try {
        rs[(size_t)g] = detail::train_rank(cfg, plans[(size_t)g], uid);
      } catch (...) {
        errs[(size_t)g] = std::current_exception();
      }
    });
  for (auto& t : threads) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  RunResult res = std::move(rs[0]);
  for (int g = 1; g < cfg.gpus; ++g)
    if (rs[(size_t)g].final_params != res.final_params) res.replicas_identical = false;
  return res;
}

// ---- checkpoints (models.cpp:348-387) ------------------------------------------------
inline void save_model(const MadeModel& m, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  out << "vqmc-model 1 made " << m.n << " " << m.h << "\n";
  out << "degrees";
  for (int d : m.degrees) out << " " << d;
  out << "\n";
  out << std::setprecision(17);
  for (double v : m.theta) out << v << "\n";
}

inline MadeModel load_made(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error(path + ": empty checkpoint");
  std::istringstream hs(line);
  std::vector<std::string> tok;
  std::string t;
  while (hs >> t) tok.push_back(t);
  if (tok.size() != 5 || tok[0] != "vqmc-model" || tok[1] != "1" || tok[2] != "made")
    throw std::runtime_error(path + ": bad checkpoint header");
  const int n = std::stoi(tok[3]), h = std::stoi(tok[4]);
  MadeModel m = made_init(n, h, 0);
  std::string label;
  if (!(in >> label) || label != "degrees") throw std::runtime_error(path + ": missing degrees line");
  for (int k = 0; k < h; ++k)
    if (!(in >> m.degrees[k]) || m.degrees[k] < 1 || m.degrees[k] > n - 1)
      throw std::runtime_error(path + ": invalid degrees");
  for (int p = 0; p < m.param_count(); ++p)
    if (!(in >> m.theta[p])) throw std::runtime_error(path + ": truncated parameter block");
  double extra;
  if (in >> extra) throw std::runtime_error(path + ": parameter count mismatch");
  return m;
}

}  // namespace vqmc
