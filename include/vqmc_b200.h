/*
 * vqmc_b200.h — C ABI of the B200-native VQMC training step (Max-Cut; general Ising / TIM specs).
 *
 * Drop-in boundary for the reference's C++ free-function API
 * (arxiv/paper_2106_13308, /root/reference/proj).  The reference has no FFI;
 * each entry point below replaces the reference function cited beside it, with
 * plain pointers and sizes (no Eigen / torch types).  Conventions:
 *
 *  - Every function returns an int status: VQMC_OK (0) or an error code; the
 *    message is in vqmc_last_error() (thread-local).  VQMC_ERR_INVALID mirrors
 *    the reference's std::invalid_argument, VQMC_ERR_NUMERIC its
 *    std::runtime_error (non-finite local energy), so a C++ facade can rethrow
 *    the same exception types and keep the CLI's exit codes
 *    (proj/tools/vqmc.cpp:35-37).
 *  - Host pointers are caller-owned.  Device state (parameters, Adam moments,
 *    batch buffers) is owned by the handle; steady-state calls do not allocate.
 *  - Parameters cross the boundary as fp64 in the reference flatten order
 *    theta = [W1 (h x n, row-major k*n+j), b1 (h), W2 (n x h, row-major i*h+k),
 *    b2 (n)], length d = 2hn + h + n (proj/src/models.cpp:264-300).
 *  - Configurations cross the boundary bit-packed: sample b, bit i is bit (i & 31)
 *    of word bits[b * W + (i >> 5)], W = ceil(n / 32).  (The reference's
 *    ConfigBatch is a B x n matrix of 0.0/1.0 doubles, proj/include/vqmc/common.hpp:29-32.)
 *  - Uniforms for injected-uniform ("parity") sampling are fp64 in the
 *    reference's consumption order [bit][sample] (proj/src/sampler.cpp:47-53).
 *    With uniforms == NULL the sampler draws counter-based Philox4x32-10
 *    uniforms keyed by (seed, stream) with counter (bit, sample, call).
 *  - Calls are thread-safe across handles, not within one handle.
 */
#ifndef VQMC_B200_H
#define VQMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQMC_OK 0
#define VQMC_ERR_INVALID 1 /* std::invalid_argument in the reference */
#define VQMC_ERR_NUMERIC 2 /* std::runtime_error (numerical) in the reference */
#define VQMC_ERR_CUDA 3
#define VQMC_ERR_NCCL 4
#define VQMC_ERR_SR 5 /* SrSolveError (optimizer.hpp:46-55): SR CG missed its residual contract */

typedef struct vqmc_gpu vqmc_gpu_t;

/* Per-step results of vqmc_gpu_train_step (this rank's minibatch). */
typedef struct {
  double energy_mean;     /* mean local energy of this rank's batch (estimator.hpp:94-100) */
  double energy_var;      /* unbiased variance of this rank's batch */
  double grad_norm;       /* ||reduced gradient||_2 after the all-reduce (trainer.cpp:253) */
  int64_t cut_sum;        /* sum of cut values (exact; pooled stats across ranks use these) */
  int64_t cut_sq_sum;     /* sum of squared cut values */
  int32_t best_cut;       /* max cut in the batch */
  int32_t batch;          /* B */
} vqmc_step_stats_t;

/* Thread-local message of the last failing call on this thread. */
const char* vqmc_last_error(void);

/* Number of visible CUDA devices. */
int vqmc_gpu_device_count(int* count);

/* Handle = one model replica + Max-Cut instance on one GPU.
 * Replaces: MadeModel value + HamiltonianSpec/MaxCutProblem (models.hpp:34-46,
 * hamiltonian.hpp:78-84; maxcut_spec hamiltonian.cpp:109-119 incl. validate :36-54).
 * degrees: h entries in [1, n-1] (models.cpp:91 for made_init, or a checkpoint's).
 * edges: num_edges pairs (i, j), 0-based, i < j, no duplicates.
 * max_batch: initial batch capacity (buffers grow on demand outside the step).  Every call takes
 * at most 49152 samples (B = minibatch * workers); larger batches return VQMC_ERR_INVALID. */
int vqmc_gpu_create(int device, int n, int h, const int32_t* degrees, const double* theta,
                    const int32_t* edges, int64_t num_edges, int max_batch, vqmc_gpu_t** out);
int vqmc_gpu_destroy(vqmc_gpu_t* g);
/* Replace the Max-Cut instance (same n); validates like vqmc_gpu_create. */
int vqmc_gpu_set_edges(vqmc_gpu_t* g, const int32_t* edges, int64_t num_edges);

/* parameter_vector / set_parameters (models.cpp:264-300).  Masked entries keep
 * the values last set on the host (their gradient is exactly zero). */
int vqmc_gpu_param_count(const vqmc_gpu_t* g, int64_t* d);
int vqmc_gpu_set_params(vqmc_gpu_t* g, const double* theta);
int vqmc_gpu_get_params(vqmc_gpu_t* g, double* theta);

/* auto_sample (sampler.cpp:35-59): B exact autoregressive samples.
 * bits_out: B x W words (may be NULL); log_psi_out: B (may be NULL). */
int vqmc_gpu_sample(vqmc_gpu_t* g, int B, const double* uniforms, uint64_t seed, uint64_t stream,
                    uint64_t call, uint32_t* bits_out, double* log_psi_out);

/* log_psi_batch / conditionals (models.cpp:114-120) for given configurations.
 * cond_out: B x n clamped conditionals p(x_i = 1 | x_<i) (may be NULL). */
int vqmc_gpu_log_psi(vqmc_gpu_t* g, const uint32_t* bits, int B, double* log_psi_out,
                     double* cond_out);

/* local_energy_batch, diagonal (Max-Cut) branch (estimator.hpp:43-57) and
 * cut_value (hamiltonian.cpp:121-124).  Either output may be NULL. */
int vqmc_gpu_maxcut_energy(vqmc_gpu_t* g, const uint32_t* bits, int B, int32_t* cut_out,
                           double* local_out);

/* HamiltonianSpec (hamiltonian.hpp:34-44; validate hamiltonian.cpp:36-54): a general Ising
 * problem H = -sum_i (alpha_i X_i + beta_i Z_i) - sum_{i<j} beta_ij Z_i Z_j on the handle's n
 * spins (the TIM instances of random_tim / load_spec).  alpha, beta: n entries (alpha >= 0);
 * pairs: num_pairs (i, j, value), 0-based, i < j, no duplicates.  While a spec is set,
 * vqmc_gpu_local_energy, vqmc_gpu_evaluate and vqmc_gpu_train_step use its local energy (with the
 * off-diagonal branch); vqmc_gpu_clear_spec returns to the handle's Max-Cut instance. */
int vqmc_gpu_set_spec(vqmc_gpu_t* g, const double* alpha, const double* beta, const int32_t* pair_i,
                      const int32_t* pair_j, const double* pair_value, int64_t num_pairs);
int vqmc_gpu_clear_spec(vqmc_gpu_t* g);

/* local_energy_batch (estimator.hpp:43-90): l_b = H_xx - sum_{k: alpha_k > 0} alpha_k
 * exp(log psi(x_b ^ e_k) - cached_log_psi_b) (exponents shifted by their maximum when it exceeds
 * 50).  cached_log_psi: B entries (SampleBatch::log_psi), or NULL for the model's own log psi of
 * the configurations.  Without a spec: the Max-Cut diagonal branch.  VQMC_ERR_NUMERIC on a
 * non-finite result. */
int vqmc_gpu_local_energy(vqmc_gpu_t* g, const uint32_t* bits, int B, const double* cached_log_psi,
                          double* local_out);

/* weighted_grad_log_psi (models.cpp:175-198): sum_b w_b grad log psi(x_b),
 * reference flatten order, d entries. */
int vqmc_gpu_weighted_grad(vqmc_gpu_t* g, const uint32_t* bits, const double* weights, int B,
                           double* grad_out);

/* gradient_from_locals (estimator.hpp:111-119): weights 2 (l_b - mean l) / B. */
int vqmc_gpu_gradient_from_locals(vqmc_gpu_t* g, const uint32_t* bits, const double* local, int B,
                                  double* grad_out);

/* adam_step (optimizer.cpp:21-35) on the handle's parameters and moments.
 * grad: d entries (reference order) or NULL to use the gradient of the last
 * vqmc_gpu_train_step.  t is the step count AFTER the increment (1 on the first step). */
int vqmc_gpu_adam_step(vqmc_gpu_t* g, const double* grad, double lr, double beta1, double beta2,
                       double eps, int64_t t);
/* Zero the Adam moments (fresh AdamState). */
int vqmc_gpu_adam_reset(vqmc_gpu_t* g);

/* Data-parallel plumbing (replaces allreduce_mean trainer.cpp:324-335 and the
 * std::barrier phases :174-279): one NCCL communicator per rank. */
int vqmc_gpu_comm_unique_id(uint8_t id_out[128]);
int vqmc_gpu_comm_init(vqmc_gpu_t* g, const uint8_t id[128], int nranks, int rank);

/* sr_direction (optimizer.cpp:64-82) with the Fisher estimate of the configurations `bits`
 * (FisherEstimate over score_matrix rows, estimator.hpp:146-168, models.cpp:221-244; centred
 * unless centered == 0): solves (F + lambda I) delta = grad by conjugate gradient on the GPU
 * (the scores are never materialised), accepting the solution only if
 * ||(F + lambda I) delta - grad|| <= tol ||grad|| (else VQMC_ERR_SR, with iterations_out /
 * residual_out set).  grad and delta_out: d entries, reference order. */
int vqmc_gpu_sr_direction(vqmc_gpu_t* g, const uint32_t* bits, int B, const double* grad, double lambda, double tol,
                          int max_iterations, int centered, double* delta_out, int* iterations_out,
                          double* residual_out);

/* One SGD + SR iteration (OptimizerKind::kSgdSr; trainer.cpp:150-282 with :165-168, :189-199,
 * :223-225) on this GPU: sampling, local energies, REINFORCE gradient, the mean over the
 * `workers` segments, the SR direction over the pooled scores of all workers*minibatch samples,
 * and params -= lr * direction.  fallback != 0: a CG failure applies the raw gradient instead
 * (SrConfig::fallback); otherwise VQMC_ERR_SR and the parameters are unchanged.  With a
 * communicator (vqmc_gpu_comm_init) the Fisher estimate pools every rank's samples: the gradient,
 * the centring sum and F p are all-reduced inside each CG iteration (CG path, d > 2000). */
int vqmc_gpu_train_step_sr(vqmc_gpu_t* g, int minibatch, int workers, const double* uniforms, uint64_t seed,
                           uint64_t stream0, uint64_t call, double lr, double lambda, double tol, int max_iterations,
                           int fallback, int centered, vqmc_step_stats_t* stats_out, int* iterations_out,
                           double* residual_out);

/* One fused VQMC iteration (worker_body, trainer.cpp:150-282) for `workers`
 * data-parallel workers of `minibatch` samples each on this GPU (worker s of
 * this rank draws from stream stream0 + s; the reference's worker w uses
 * make_stream(seed, w + 1), trainer.cpp:126): sampling, Max-Cut local energies,
 * REINFORCE weights with each worker's in-batch baseline, MADE backward, the
 * all-reduce mean over workers and ranks (NCCL if a communicator is set), and
 * Adam (lr, beta1, beta2, eps, step count t).  uniforms: NULL (Philox, counter
 * `call`) or [n][workers*minibatch] fp64 (parity mode).  stats_out == NULL:
 * asynchronous; else blocks until this rank's statistics are on the host. */
int vqmc_gpu_train_step(vqmc_gpu_t* g, int minibatch, int workers, const double* uniforms,
                        uint64_t seed, uint64_t stream0, uint64_t call, double lr, double beta1,
                        double beta2, double eps, int64_t t, vqmc_step_stats_t* stats_out);

/* Copy the last step's cut values (B int32) to the host. */
int vqmc_gpu_last_cuts(vqmc_gpu_t* g, int32_t* cuts_out, int B);
/* Copy the configurations of the handle's last batch (the last train step's samples, or the
 * last vqmc_gpu_evaluate / sample / log_psi batch) to the host: B x W packed words.  The
 * reference keeps them in SampleBatch::configs (sampler.hpp:24-30); the parity tests compare
 * them with the oracle's draws and feed them to the oracle's downstream functions. */
int vqmc_gpu_last_samples(vqmc_gpu_t* g, uint32_t* bits_out, int B);
/* The reduced gradient of the last vqmc_gpu_train_step (allreduce_mean over every worker and
 * rank, i.e. what Adam consumed), d entries in the reference order: the value the reference
 * hands to RunConfig::gradient_observer (trainer.hpp:57, trainer.cpp:187-188). */
int vqmc_gpu_last_gradient(vqmc_gpu_t* g, double* grad_out);

/* evaluate (trainer.cpp:91-108): fresh batch, out = {energy_mean, energy_std,
 * best_cut, mean_cut}.  uniforms as in vqmc_gpu_sample. */
int vqmc_gpu_evaluate(vqmc_gpu_t* g, int B, const double* uniforms, uint64_t seed,
                      uint64_t stream, uint64_t call, double out[4]);

/* Pooled mean / unbiased variance of N Max-Cut local energies from exact cut sums
 * (energy_and_variance, estimator.hpp:94-100, over the pooled batch trainer.cpp:246-248). */
int vqmc_pooled_stats(int64_t num_edges, int64_t N, int64_t cut_sum, int64_t cut_sq_sum,
                      double* mean, double* var);

/* Block until all work queued on the handle's stream is done. */
int vqmc_gpu_synchronize(vqmc_gpu_t* g);

/* Number of kernel launches the handle has issued (for the bench's gpu_launches). */
int64_t vqmc_gpu_launch_count(const vqmc_gpu_t* g);

/* Device-side timing of the last train step (ms): level 2 gives the phases sample,
 * energy+weights, backward, allreduce, update; level 1 gives the whole step in out_ms[0]. */
int vqmc_gpu_phase_times(vqmc_gpu_t* g, float out_ms[5]);
/* CUDA-event timing inside train_step: 0 off (default), 1 whole step, 2 per phase. */
int vqmc_gpu_set_phase_timing(vqmc_gpu_t* g, int level);

/* Replay the training step as a captured CUDA graph (default on; the first step of a
 * configuration runs eagerly, the second is captured). */
int vqmc_gpu_set_graph(vqmc_gpu_t* g, int enable);

/* Per-kernel CUDA-event timing of the last train step (roofline evidence):
 * names_out = count slots of 32 chars, ms_out = count durations.  enable = 1: the backward runs
 * serially (every kernel timed alone); enable = 2: timeline mode, the production (concurrent)
 * schedule with events on both streams. */
int vqmc_gpu_set_kernel_timing(vqmc_gpu_t* g, int enable);
int vqmc_gpu_kernel_times(vqmc_gpu_t* g, char* names_out, float* ms_out, int cap, int* count);
/* Timeline mode (kernel timing 2, phase timing >= 1): each kernel's start / end event of the last
 * step in ms after the step-start event (start = when its stream reached it). */
int vqmc_gpu_kernel_timeline(vqmc_gpu_t* g, char* names_out, float* start_ms, float* end_ms, int cap, int* count);

/* ---- Host utilities of the same library (C++; no GPU needed) ---- */

/* mix_seed (common.hpp:56-61). */
uint64_t vqmc_mix_seed(uint64_t seed, uint64_t stream);
/* default_made_hidden (models.cpp:79-82). */
int vqmc_default_made_hidden(int n);
/* made_init (models.cpp:84-104): degrees_out h, theta_out d. */
int vqmc_made_init(int n, int h, uint64_t seed, int32_t* degrees_out, double* theta_out);
/* `count` U[0,1) draws of make_stream(seed, stream) (std::mt19937_64 +
 * uniform_real_distribution, the reference's sampler stream), after `skip`. */
int vqmc_stream_uniforms(uint64_t seed, uint64_t stream, uint64_t skip, int64_t count,
                         double* out);
/* Graph generators; call with edges_out == NULL to get *num_edges first.
 * random_maxcut_graph (hamiltonian.cpp:144-160); random d-regular and G(n,p) are new. */
int vqmc_random_maxcut_graph(int n, uint64_t seed, int32_t* edges_out, int64_t cap,
                             int64_t* num_edges);
int vqmc_random_regular_graph(int n, int d, uint64_t seed, int32_t* edges_out, int64_t cap,
                              int64_t* num_edges);
int vqmc_erdos_renyi_graph(int n, double p, uint64_t seed, int32_t* edges_out, int64_t cap,
                           int64_t* num_edges);
/* random_tim (hamiltonian.cpp:126-142): alpha, beta n entries; pairs n(n-1)/2 (row-major i < j). */
int vqmc_random_tim(int n, uint64_t seed, double* alpha, double* beta, int32_t* pair_i, int32_t* pair_j,
                    double* pair_value);
/* load_spec / save_spec "tim" text format (hamiltonian.cpp:162-234); load with alpha == NULL first
 * to get *n_out and *num_pairs. */
int vqmc_load_spec(const char* path, int* n_out, double* alpha, double* beta, int32_t* pair_i,
                   int32_t* pair_j, double* pair_value, int64_t cap, int64_t* num_pairs);
int vqmc_save_spec(const char* path, int n, const double* alpha, const double* beta, const int32_t* pair_i,
                   const int32_t* pair_j, const double* pair_value, int64_t num_pairs);
/* load_graph / save_graph text format (hamiltonian.cpp:236-266). */
int vqmc_load_graph(const char* path, int* n_out, int32_t* edges_out, int64_t cap,
                    int64_t* num_edges);
int vqmc_save_graph(const char* path, int n, const int32_t* edges, int64_t num_edges);

#ifdef __cplusplus
}
#endif

#endif /* VQMC_B200_H */
