// Internal declarations of the B200 VQMC library (handle layout, kernels, helpers).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "head4.cuh"
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "vqmc_b200.h"

namespace vqmc_b200 {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, mapped to status codes at the ABI.
// ---------------------------------------------------------------------------
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// SR conjugate gradient did not meet its residual contract (optimizer.hpp:46-55)
struct SrSolveError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define VQMC_CUDA(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::vqmc_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                   " (" __FILE__ ":" + std::to_string(__LINE__) + ")");  \
  } while (0)

constexpr double kProbEps = 1e-7;  // proj/include/vqmc/models.hpp:26
// logit(1 - 1e-7) = ln((1 - 1e-7) / 1e-7): p_raw >= 1 - eps  <=>  z >= kLogitHi.
constexpr float kLogitHi = 16.118095650958319f;
constexpr int kMaxHidden = 1024;
constexpr int kMaxBatch = 49152;  // samples per call: stats_weights_kernel holds B fp32 weights in one CTA's smem
constexpr int kTailBN = 192;  // tail sampler / S p pair tile: 256 samples x 192 outputs
constexpr int kGw1MaxSplits = 16;  // split-K of the gW1 GEMM over the batch
// Exact per-rank cut statistics ride in the gradient all-reduce as fp32 16-bit limbs, stored right
// after the live gradient (G[L.total ...]): cut sum (3), cut^2 sum (4), best cut per rank (2 each).
constexpr int kMaxRanks = 256;  // limb sums stay < 2^24 (exact in fp32) for <= 256 ranks
__host__ __device__ constexpr int rstat_count(int nranks) { return 7 + 2 * nranks; }

// ---------------------------------------------------------------------------
// Device-resident parameter layout ("live" layout).  One contiguous fp32
// buffer so Adam is a single elementwise pass:
//   W1T [Hd][h]  : W1T[j][k] = M1(k,j) * W1[k][j]   (only inputs j < Hd = max degree
//                  can ever be live, so the dead columns j >= Hd are not stored)
//   b1  [h]
//   W2  [n][h]   : M2(i,k) * W2[i][k]
//   b2  [n]
// Masked entries are stored as exact zeros; their gradient is exactly zero, so
// Adam never moves them (proj/src/optimizer.cpp:21-35 with zero moments).  The
// reference values of masked / dead entries are kept in a host copy for export.
// ---------------------------------------------------------------------------
struct Layout {
  int n = 0, h = 0, Hd = 0, W = 0;
  int64_t off_w1t = 0, off_b1 = 0, off_w2 = 0, off_b2 = 0, total = 0;
  void init(int n_, int h_, int Hd_) {
    n = n_;
    h = h_;
    Hd = Hd_;
    W = (n + 31) / 32;
    off_w1t = 0;
    off_b1 = off_w1t + (int64_t)Hd * h;
    off_w2 = off_b1 + h;
    off_b2 = off_w2 + (int64_t)n * h;
    total = off_b2 + n;
  }
};

struct Handle;
struct RngSpec;
struct SpecState;  // general Ising spec (TIM) and its scratch (spec.cu)
// Timing event on the handle's stream; inside a graph capture it becomes an external event
// record node so replays still record (and can be timed).
void record_event(Handle* h, cudaEvent_t ev);
void record_event_on(Handle* h, cudaEvent_t ev, cudaStream_t stream);

// Per-step scalars kept in device memory so a captured CUDA graph of the step can be replayed:
// they describe the step about to run; the step's last kernel (Adam) advances call / t and the
// Adam bias corrections for the next one.
struct StepParams {
  uint64_t call;  // Philox counter of this step
  int64_t t;      // Adam step count of this step (1-based)
  float lr, b1, b2, eps;
  float bc1, bc2;    // 1 - beta^t
  float ibc1, ibc2;  // 1 / bc (fp32 division, once)
  float nbc1, nbc2, nibc1, nibc2;  // the same for t + 1 (Adam's first block, off the step's tail)
};

// RAII per-kernel event pair (active only when Handle::ktimer is set).
struct KScope {
  Handle* H;
  int slot;
  cudaStream_t s;
  KScope(Handle* h, const char* name, cudaStream_t stream = nullptr);  // (nullptr: the handle's stream)
  ~KScope();
};

// TMA descriptors (gemm.cu): K-major operand, element (mn, k) at ptr[mn * ld + k], box {128 bytes
// of K, box_mn}, SWIZZLE_128B; ek = umma_gemm.cuh element kind (kElemU8 for 8-bit operands).
CUtensorMap tmap_kmajor(const void* ptr, int64_t K, int64_t MN, int64_t ld, int box_mn, int ek);

// Kernel launchers (kernels.cu).  All enqueue on h->stream.
void launch_params_refresh(Handle* h);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `kern` on the current device, once per
// (kernel, device, size): function attributes are per device, and handles on different devices
// may share a process (thread-safe).
void ensure_smem_attr(const void* kern, size_t bytes);
void launch_head_pack(Handle* h);
void launch_head_v2(Handle* h, int B, const double* d_uniforms, RngSpec rng, bool given_bits,
                    double* d_cond);
void launch_z2(Handle* h, int B, int col0, const double* d_uniforms, RngSpec rng,
               bool given_bits, double* d_cond, bool want_lp = true);
void launch_finalize_logpsi(Handle* h, int B, int n_tiles);
void launch_energy(Handle* h, int B);
// dense-graph energy (energy_dense.cu)
bool dense_energy_preferred(int n, int64_t num_edges);
void setup_dense_energy(Handle* h);  // after the edge list is uploaded
void free_dense_energy(Handle* h);
void launch_energy_dense(Handle* h, int B);
// lin: fp64 local energies of a general spec (else the Max-Cut cuts of the energy kernel); lstat:
// [sum l, sum l^2, then per segment] (general spec only)
void launch_weights_from_locals(Handle* h, int B, int seg, bool with_wg1 = false, const double* lin = nullptr,
                                double* lstat = nullptr);
void launch_cuts_reduce(Handle* h, int B);
void launch_backward(Handle* h, int B, bool wg1_done = false);
void launch_backward_tail(Handle* h, int B);  // dg1, dz1, gW1 (+ finalize)
// dz1, gW1 (+ finalize); after_dz1 (optional) is recorded on the stream between dz1 and gW1
void launch_backward_after_dg1(Handle* h, int B, cudaEvent_t after_dz1 = nullptr);
void launch_dg1_umma(Handle* h, int B);
int gemm_sms(const Handle* h);  // SMs the persistent GEMMs may use
void launch_tail_umma(Handle* h, int B, const double* d_uniforms, RngSpec rng, bool want_lp);
void launch_dg1_umma(Handle* h, int B);
void launch_gw2_umma(Handle* h, int B, bool wg1_done = false, cudaStream_t stream = nullptr);
void launch_split_w2(Handle* h);
void launch_gw1_umma(Handle* h, int B, int& splits_out);
// SR (sr.cu, gemm.cu)
int launch_sp_umma(Handle* h, int B);
void ensure_sr(Handle* h, int B);
void comm_allreduce_sum(Handle* h, void* buf, size_t count, bool f64);  // capi.cu (NCCL; no-op alone)
void sr_build_scores(Handle* h, int B, bool centered);  // small models: explicit fp64 score rows
void free_sr(Handle* h);
void launch_sr_grad_from_G(Handle* h, double scale);
void launch_sr_apply(Handle* h, double lr, const double* delta);
bool sr_solve(Handle* h, int B, double lambda, double tol, int max_iterations, bool centered, int* iterations,
              double* residual, double* gnorm_out);
// general Ising specs / plain forward (spec.cu)
void spec_set(Handle* h, const double* alpha, const double* beta, const int32_t* pi, const int32_t* pj,
              const double* pv, int64_t np);
void spec_free(Handle* h);
void forward_plain(Handle* h, int B, double* d_cond, float* d_lterm, float* d_fterm, float* d_z1, double* d_lp_out);
void launch_spec_local(Handle* h, int B, const double* d_cached, double* d_local);
double* spec_local_buffer(Handle* h, int B);
double* spec_cached_buffer(Handle* h, int B);
void launch_given_umma(Handle* h, int B, double* cond, float* lterm, float* fterm);
void set_error(const std::string& msg);
int status_of(const std::exception& ex);
// hyper-parameters from h->d_step; gated: skip the update when the step's non-finite-logit flag is set
void launch_adam(Handle* h, float grad_scale, bool gated);
void launch_adam_part(Handle* h, float grad_scale, int part, cudaStream_t stream);  // 0: [W2|b2], 1: [W1T|b1]
void launch_set_step(Handle* h, uint64_t call, int64_t t, double lr, double b1, double b2, double eps);

// Kernel launch on the handle's stream; with Handle::pdl the launch carries the programmatic
// stream serialization attribute, so the kernel's prologue overlaps the previous kernel's tail
// (every step kernel calls ptx::pdl_wait() before touching global memory).
template <typename... KArgs, typename... Args>
void launch_k(Handle* H, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args);

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  Layout L;
  int64_t d = 0;  // reference parameter count
  std::vector<int32_t> degrees;
  std::vector<double> theta_host;  // reference-order copy (masked / dead entries)
  int64_t num_edges = 0;
  SpecState* spec = nullptr;  // general Ising spec (vqmc_gpu_set_spec): the local energy of TIM problems
  double* d_lstat = nullptr;  // general spec: [sum l, sum l^2, per segment (sum l, sum l^2)] of the last step
  int lstat_cap = 0;

  // model
  float* P = nullptr;      // live params [L.total]
  float* G = nullptr;      // live grads [L.total] + the rank statistics limbs [rstat_count(kMaxRanks)]
  float* h_rstat = nullptr;  // pinned host copy of the reduced limbs
  float last_grad_scale = 1.f;  // 1 / (workers * ranks) of the last train step (G holds the sum)
  bool last_grad_sr = false;     // the last step was SGD + SR: its reduced gradient is in cg_g
  float* Mo = nullptr;     // Adam m
  float* Vo = nullptr;     // Adam v
  // fp16 pair of [W2m | b2] ([n][hp18], column h = b2, zero padding): the B operand of the tail
  // GEMM (K-major, the bias rides along as column h against G1's ones column) and of dg1
  // (MN-major).  Refreshed by Adam after every update.
  __half* W2h = nullptr;
  __half* W2l = nullptr;
  int hp8 = 0, hp18 = 0, np8 = 0, hd18 = 0;  // 16-bit row strides: h, h + 1, n, Hd + 1 rounded up to 8
  int max_splits = 16;
  float* W1Tp = nullptr;   // [Hd][hp] padded head block of W1^T (head sampler staging)
  float* W2cp = nullptr;   // [h][Hdp] W2 head columns in completion order (padded)
  int head_hpk = 0, head_Hdp = 0;  // row strides of W1Tp / W2cp
  int32_t* d_comp_pos = nullptr;   // [h] completion slot of hidden unit k (inverse of comp_k)
  unsigned* d_done = nullptr;      // last-block counter of the Adam grad-norm reduction
  std::vector<int32_t> comp_off_host;  // [Hd + 1]
  bool head_fast = false;  // bit i completes exactly hidden unit i (head v3, lane-permuted staging)
  bool head_v4 = false;    // head_fast and the v4 sampler (tensor-core word updates; VQMC_HEAD=3 keeps v3)
  bool head_v5 = false;    // v4's staging with chain / tile warps specialised (VQMC_HEAD=4 keeps v4)
  Head4Stage h4{nullptr, nullptr, 0};  // v4 staging (head4.cuh)
  bool w1skip = false;     // deg_k <= k + 1 for all k (W1 columns below the current word are dead)
  int32_t* d_deg = nullptr;
  int32_t* d_comp_k = nullptr;    // hidden units sorted by degree
  int32_t* d_comp_off = nullptr;  // [Hd + 1]: units with degree i+1 at [off[i], off[i+1])
  int2* d_edges = nullptr;
  uint32_t* d_edges_bank = nullptr;  // byte offsets 4u | 4v << 16, bank-ordered, quad-interleaved (upload_edges)
  int64_t num_edges_bank = 0;        // entries incl. padding (multiple of 128)
  // dense-graph energy (energy_dense.cu): fp8 strictly-upper adjacency [n][32 W], node degrees, and
  // the fp8 expansion of the batch's spins [B][32 W]
  bool dense_energy = false;
  uint8_t* Uf8 = nullptr;
  uint8_t* Xf8 = nullptr;
  int32_t* d_degn = nullptr;
  int64_t xf8_cap = 0;

  // batch buffers (capacity cap_B)
  int cap_B = 0;
  uint32_t* X = nullptr;     // [B][W]
  float* G1 = nullptr;       // [B][h]  relu(z1)
  __half* Dh = nullptr;      // [B][np8] D = 0.5 (x - p_raw) * clampmask as an fp16 pair (hi)
  __half* Dl = nullptr;      // (lo): A operand of dg1 (K-major) and gW2 (MN-major)
  __half* G1h = nullptr;     // [B][hp18] fp16 pair of [G1 | 1] (tail GEMM A operand; column h = 1)
  __half* G1l = nullptr;
  __half* wG1h = nullptr;    // [B][hp18] fp16 pair of [w' (.) G1 | w'] (gW2 B operand)
  __half* wG1l = nullptr;
  double* lp_head = nullptr; // [B]
  float* thr = nullptr;      // [B][Hd8] logit thresholds of the head bits (head v3)
  double* lp_part = nullptr; // [max_tiles][B]
  double* log_psi = nullptr; // [B]
  int32_t* cut = nullptr;    // [B]
  int32_t* cpart = nullptr;  // [cut_chunks][B] per-edge-chunk partial cut counts (energy kernel)
  int cut_chunks = 1;
  int64_t cpart_cap = 0;
  double* local = nullptr;   // [B]
  float* w = nullptr;        // [B] REINFORCE weights w' = w / wscale (|w'| <= 1, fp16-safe)
  float* d_wscale = nullptr; // [1] wscale: power of two >= max |w| (the backward epilogues multiply by it)
  float* Epart = nullptr;    // [splits][B][h]
  __nv_bfloat16* dz1bh = nullptr;  // [B][hp8] bf16 pair of dz1 (gW1 operand)
  __nv_bfloat16* dz1bl = nullptr;
  __nv_bfloat16* Xfb = nullptr;    // [B][hd18] spins 0/1 of the head inputs + a ones column (gW1 operand)
  float* gw1_part = nullptr; // [kGw1MaxSplits][Hd + 1][h]
  double* cond = nullptr;    // [B][n] optional (log_psi with conditionals)
  double* uni = nullptr;     // [n][B] injected uniforms
  int64_t uni_cap = 0;
  int64_t cond_cap = 0;

  // scratch
  double* d_scal = nullptr;    // fp64 scratch: [0] = ||grad||^2
  int64_t* d_istat = nullptr;  // per worker segment s: [3s] cut_sum [3s+1] cut_sq_sum [3s+2] best
  int istat_cap = 0;
  double* d_gpart = nullptr;   // grad-norm partials
  // SR (sr.cu; allocated on first use): fp64 CG vectors in the live layout, the fp16 pair of the
  // CG direction's [W2 | b2] block, per-sample products q = grad log psi . p and their partials
  double *cg_x = nullptr, *cg_r = nullptr, *cg_p = nullptr, *cg_g = nullptr, *cg_ap = nullptr, *cg_part = nullptr;
  double* sr_S = nullptr;  // small models (d <= 2000): explicit fp64 score rows [B][total]
  double* sr_C = nullptr;  // and the Cholesky factor of the dense system (min(B, total)^2)
  size_t sr_S_cap = 0, sr_C_cap = 0;
  __half *SRh = nullptr, *SRl = nullptr;
  double *sr_q = nullptr, *sp_part = nullptr, *d_sr_scal = nullptr, *h_sr_scal = nullptr, *sr_q1 = nullptr;
  float *sr_dz1 = nullptr, *sr_p1f = nullptr;
  unsigned* d_pmax = nullptr;
  int sr_cap_B = 0;
  // SR's device-resident CG loop: one captured iteration under a conditional WHILE node
  // (VQMC_SR_HOST_LOOP=1 keeps the host-driven loop)
  bool sr_device_loop = true;
  cudaGraphExec_t sr_gexec = nullptr;
  struct SrGraphKey {
    bool valid = false;
    int B = 0, cap_B = 0, sr_cap_B = 0;
    bool centered = true;
    double lambda = 0.0, tol = 0.0;
    int max_it = 0;
    bool operator==(const SrGraphKey& o) const {
      return valid && o.valid && B == o.B && cap_B == o.cap_B && sr_cap_B == o.sr_cap_B && centered == o.centered &&
             lambda == o.lambda && tol == o.tol && max_it == o.max_it;
    }
  };
  SrGraphKey sr_gkey;
  int gpart_n = 0;
  uint32_t* d_flag = nullptr;  // sticky non-finite flag (logit overflow in the fp16-pair GEMMs)
  double* d_host_stage = nullptr;

  // pinned host staging for stats
  double* h_scal = nullptr;
  int64_t* h_istat = nullptr;  // pinned, istat_cap entries

  // per-step scalars and the captured step graph
  StepParams* d_step = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // exact configuration the graph was captured for (seed and stream0 are baked into its kernels'
  // arguments, so every field is compared; valid = false: no captured / warmed configuration)
  struct GraphKey {
    bool valid = false;
    int minibatch = 0, workers = 0, phase_timing = 0;
    int ktimer = 0;
    uint64_t seed = 0, stream0 = 0;
    bool operator==(const GraphKey& o) const {
      return valid && o.valid && minibatch == o.minibatch && workers == o.workers && phase_timing == o.phase_timing &&
             ktimer == o.ktimer && seed == o.seed && stream0 == o.stream0;
    }
  };
  GraphKey gkey;
  bool graph_enabled = true;
  bool graph_warm = false;      // one eager step runs before the first capture
  bool capturing = false;       // inside cudaStreamBeginCapture on this handle's stream
  uint64_t next_call = ~0ull;   // (call, t) the device counters will produce next
  int64_t next_t = -1;
  double cur_lr = -1, cur_b1 = -1, cur_b2 = -1, cur_eps = -1;
  void invalidate_graph();

  // comm: the [W2 | b2] part of the gradient (99% of the bytes) is all-reduced on cstream while dg1,
  // dz1 and gW1 run; the GEMMs then leave gemm_sm_reserve SMs free for NCCL's kernels
  void* nccl_comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_dg1 = nullptr, ev_dz1 = nullptr;
  int gemm_sm_reserve = 0;
  // concurrent backward: gW2 (and its all-reduce) on cstream with gw2_sms SMs while dg1 -> dz1 ->
  // gW1 use the rest (gemm_sm_cap limits the persistent GEMM grids; 0 = no cap)
  bool concurrent_bw = true;
  // (N = 10k sweep with PDL on and dg1's split count following this partition, ms per step at Adam
  // 110: gw2 56 0.185, 64 0.1768, 72 0.1789, 76 0.1780, 80 0.1749, 84 0.1754, 88 0.188, 96 0.191;
  // Adam 100 / 110 / 120 at gw2 80: 0.1755 / 0.1749 / 0.1767)
  // (N = 5000: 64 SMs 0.1448 vs 80 SMs 0.1498 ms: dg1's 12 pair tiles split 3 ways vs 2; N = 1000
  // and G(10^4, 3/4) within 1%: 80 from N = 8192 up, else 64 -- capi.cu vqmc_gpu_create)
  int gw2_sms = 64;
  // (started after dz1: 110 0.1707, 130 0.1696, 140 0.1702, 148 0.1700 ms)
  int adam_w2_sms = 130;  // SMs' worth of blocks for the [W2 | b2] Adam beside gW1 (VQMC_ADAM_SMS)
  int gemm_sm_cap = 0;
  int gw1_splits = 4;  // max split-K of the gW1 GEMM (1: direct epilogue, no finalize; VQMC_GW1_SPLITS; 4 measured best)

  // timing
  int phase_timing = 0;  // 0 off, 1 whole-step events, 2 per-phase events
  cudaEvent_t ev[6] = {};
  float phase_ms[5] = {0, 0, 0, 0, 0};

  // per-kernel event timing (bench roofline): pool of event pairs reused each step
  int ktimer = 0;  // 1: per-kernel events, serial backward; 2: timeline (events on both streams, concurrent schedule)
  static constexpr int kKtPool = 128;
  cudaEvent_t kt_start[kKtPool] = {}, kt_end[kKtPool] = {};
  const char* kt_name[kKtPool] = {};
  int kt_count = 0;

  int64_t launches = 0;
  bool pdl = true;  // programmatic dependent launch for the step kernels (VQMC_PDL=0 disables; -4 us per step)
  int tail_tiles = 0;  // column tiles of the last z2 launch (lp partials)
  int splits = 0;      // split-K factor of the dg1 GEMM

  void ensure_batch(int B);
  void ensure_uniforms(int64_t count);
  void ensure_cond(int64_t count);
  void ensure_cpart(int64_t count);
};

template <typename... KArgs, typename... Args>
void launch_k(Handle* H, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = H->stream;
  cudaLaunchAttribute at[1];
  if (H->pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  VQMC_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

}  // namespace vqmc_b200
