// C ABI of the B200 VQMC library: handle lifecycle, parameter layout
// conversion, the per-function entry points and the fused training step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "vqmc_b200.h"

namespace vqmc_b200 {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }

int status_of(const std::exception& ex) {
  if (dynamic_cast<const CudaError*>(&ex)) return VQMC_ERR_CUDA;
  if (dynamic_cast<const SrSolveError*>(&ex)) return VQMC_ERR_SR;
  if (dynamic_cast<const std::invalid_argument*>(&ex)) return VQMC_ERR_INVALID;
  return VQMC_ERR_NUMERIC;
}

// ---------------------------------------------------------------------------
// NCCL (dlopen'd so single-GPU use has no NCCL dependency).  Types follow nccl.h.
// ---------------------------------------------------------------------------
struct NcclUniqueId { char internal[128]; };
using ncclComm_t = void*;
enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0 };
struct NcclApi {
  bool loaded = false;
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
static NcclApi g_nccl;

static void load_nccl() {
  if (g_nccl.loaded) return;
  std::vector<std::string> cands;
  if (const char* e = std::getenv("VQMC_NCCL_LIB")) cands.push_back(e);
  cands.push_back("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2");
  cands.push_back("libnccl.so.2");
  for (const auto& p : cands) {
    void* h = dlopen(p.c_str(), RTLD_NOW | RTLD_GLOBAL);
    if (!h) continue;
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    if (g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce) {
      g_nccl.loaded = true;
      return;
    }
  }
  throw std::runtime_error("NCCL library not found (set VQMC_NCCL_LIB)");
}

static void nccl_check(int rc, const char* what) {
  if (rc != 0)
    throw std::runtime_error(std::string(what) + ": " +
                             (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "nccl error"));
}

// Sum over the ranks of the handle's communicator (no-op without one), on the handle's stream.
void comm_allreduce_sum(Handle* H, void* buf, size_t count, bool f64) {
  if (!H->nccl_comm) return;
  nccl_check(g_nccl.AllReduce(buf, buf, count, f64 ? ncclFloat64 : ncclFloat32, ncclSum, H->nccl_comm, H->stream),
             "ncclAllReduce (SR)");
}

// ---------------------------------------------------------------------------
// Buffers
// ---------------------------------------------------------------------------
template <class T>
static void dalloc(T** p, size_t count) {
  if (*p) VQMC_CUDA(cudaFree(*p));
  *p = nullptr;
  if (count) VQMC_CUDA(cudaMalloc((void**)p, count * sizeof(T)));
}

void Handle::ensure_batch(int B) {
  if (B <= cap_B) return;
  // stats_weights_kernel keeps the whole batch's weights in one CTA's shared memory
  if (B > kMaxBatch)
    throw std::invalid_argument("batch of " + std::to_string(B) + " samples exceeds the per-call maximum of " +
                                std::to_string(kMaxBatch) + " (split it over calls or GPUs)");
  invalidate_graph();
  const int n = L.n, h = L.h;
  const int max_tiles = 4 * ((n + 127) / 128 + 2);  // up to 4 epilogue partials per tail tile
  dalloc(&X, (size_t)B * L.W);
  dalloc(&G1, (size_t)B * h);
  dalloc(&Dh, (size_t)B * np8 + 128);
  dalloc(&Dl, (size_t)B * np8 + 128);
  dalloc(&G1h, (size_t)B * hp18 + 128);
  dalloc(&G1l, (size_t)B * hp18 + 128);
  dalloc(&wG1h, (size_t)B * hp18 + 128);
  dalloc(&wG1l, (size_t)B * hp18 + 128);
  {  // [G1 | 1]: the ones column h multiplies b2 in the tail GEMM; padding stays zero
    std::vector<__half> ones((size_t)B * hp18 + 128, __float2half(0.f));
    for (int b = 0; b < B; ++b) ones[(size_t)b * hp18 + h] = __float2half(1.f);
    VQMC_CUDA(cudaMemcpy(G1h, ones.data(), ones.size() * sizeof(__half), cudaMemcpyHostToDevice));
    VQMC_CUDA(cudaMemset(G1l, 0, ones.size() * sizeof(__half)));
  }
  dalloc(&lp_head, (size_t)B);
  dalloc(&thr, (size_t)B * ((L.Hd + 7) & ~7));
  dalloc(&lp_part, (size_t)max_tiles * B);
  dalloc(&log_psi, (size_t)B);
  dalloc(&cut, (size_t)B);
  dalloc(&local, (size_t)B);
  dalloc(&w, (size_t)B);
  dalloc(&Epart, (size_t)max_splits * B * h);
  dalloc(&dz1bh, (size_t)B * hp8 + 128);
  dalloc(&dz1bl, (size_t)B * hp8 + 128);
  dalloc(&Xfb, (size_t)B * hd18 + 128);
  VQMC_CUDA(cudaMemset(dz1bh, 0, ((size_t)B * hp8 + 128) * sizeof(__nv_bfloat16)));
  VQMC_CUDA(cudaMemset(dz1bl, 0, ((size_t)B * hp8 + 128) * sizeof(__nv_bfloat16)));
  VQMC_CUDA(cudaMemset(Xfb, 0, ((size_t)B * hd18 + 128) * sizeof(__nv_bfloat16)));
  VQMC_CUDA(cudaMemset(Dh, 0, ((size_t)B * np8 + 128) * sizeof(__half)));
  VQMC_CUDA(cudaMemset(Dl, 0, ((size_t)B * np8 + 128) * sizeof(__half)));
  cap_B = B;
}

void Handle::ensure_uniforms(int64_t count) {
  if (count <= uni_cap) return;
  dalloc(&uni, (size_t)count);
  uni_cap = count;
}

void Handle::ensure_cpart(int64_t count) {
  if (count <= cpart_cap) return;
  if (capturing) throw std::runtime_error("cpart reallocation during graph capture");
  invalidate_graph();
  dalloc(&cpart, (size_t)count);
  cpart_cap = count;
}

void Handle::ensure_cond(int64_t count) {
  if (count <= cond_cap) return;
  dalloc(&cond, (size_t)count);
  cond_cap = count;
}

static void upload_params(Handle* H, const double* theta) {
  const Layout& L = H->L;
  const int n = L.n, h = L.h, Hd = L.Hd;
  std::vector<float> P((size_t)L.total, 0.f);
  const double* W1 = theta;
  const double* b1 = W1 + (size_t)h * n;
  const double* W2 = b1 + h;
  const double* b2 = W2 + (size_t)n * h;
  for (int j = 0; j < Hd; ++j)
    for (int k = 0; k < h; ++k)
      P[L.off_w1t + (size_t)j * h + k] = (j + 1 <= H->degrees[k]) ? (float)W1[(size_t)k * n + j] : 0.f;
  for (int k = 0; k < h; ++k) P[L.off_b1 + k] = (float)b1[k];
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < h; ++k)
      P[L.off_w2 + (size_t)i * h + k] = (H->degrees[k] < i + 1) ? (float)W2[(size_t)i * h + k] : 0.f;
  for (int i = 0; i < n; ++i) P[L.off_b2 + i] = (float)b2[i];
  VQMC_CUDA(cudaMemcpyAsync(H->P, P.data(), P.size() * sizeof(float), cudaMemcpyHostToDevice, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  H->theta_host.assign(theta, theta + H->d);
  launch_params_refresh(H);
}

// live fp32 layout (device) -> reference order fp64; masked entries from `base`
static void live_to_reference(const Handle* H, const std::vector<float>& P, const double* base,
                              double* out) {
  const Layout& L = H->L;
  const int n = L.n, h = L.h, Hd = L.Hd;
  if (base) std::memcpy(out, base, sizeof(double) * H->d);
  else std::memset(out, 0, sizeof(double) * H->d);
  double* W1 = out;
  double* b1 = W1 + (size_t)h * n;
  double* W2 = b1 + h;
  double* b2 = W2 + (size_t)n * h;
  for (int j = 0; j < Hd; ++j)
    for (int k = 0; k < h; ++k)
      if (j + 1 <= H->degrees[k]) W1[(size_t)k * n + j] = P[L.off_w1t + (size_t)j * h + k];
  for (int k = 0; k < h; ++k) b1[k] = P[L.off_b1 + k];
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < h; ++k)
      if (H->degrees[k] < i + 1) W2[(size_t)i * h + k] = P[L.off_w2 + (size_t)i * h + k];
  for (int i = 0; i < n; ++i) b2[i] = P[L.off_b2 + i];
}

// reference order fp64 -> live layout fp64 (masked entries dropped)
static std::vector<double> reference_to_live(const Handle* H, const double* theta) {
  const Layout& L = H->L;
  const int n = L.n, h = L.h, Hd = L.Hd;
  std::vector<double> P((size_t)L.total, 0.0);
  const double* W1 = theta;
  const double* b1 = W1 + (size_t)h * n;
  const double* W2 = b1 + h;
  const double* b2 = W2 + (size_t)n * h;
  for (int j = 0; j < Hd; ++j)
    for (int k = 0; k < h; ++k)
      P[L.off_w1t + (size_t)j * h + k] = (j + 1 <= H->degrees[k]) ? W1[(size_t)k * n + j] : 0.0;
  for (int k = 0; k < h; ++k) P[L.off_b1 + k] = b1[k];
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < h; ++k)
      P[L.off_w2 + (size_t)i * h + k] = (H->degrees[k] < i + 1) ? W2[(size_t)i * h + k] : 0.0;
  for (int i = 0; i < n; ++i) P[L.off_b2 + i] = b2[i];
  return P;
}

// live layout fp64 -> reference order fp64 (masked entries 0)
static void live_to_reference_d(const Handle* H, const std::vector<double>& P, double* out) {
  const Layout& L = H->L;
  const int n = L.n, h = L.h, Hd = L.Hd;
  std::memset(out, 0, sizeof(double) * H->d);
  double* W1 = out;
  double* b1 = W1 + (size_t)h * n;
  double* W2 = b1 + h;
  double* b2 = W2 + (size_t)n * h;
  for (int j = 0; j < Hd; ++j)
    for (int k = 0; k < h; ++k)
      if (j + 1 <= H->degrees[k]) W1[(size_t)k * n + j] = P[L.off_w1t + (size_t)j * h + k];
  for (int k = 0; k < h; ++k) b1[k] = P[L.off_b1 + k];
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < h; ++k)
      if (H->degrees[k] < i + 1) W2[(size_t)i * h + k] = P[L.off_w2 + (size_t)i * h + k];
  for (int i = 0; i < n; ++i) b2[i] = P[L.off_b2 + i];
}

static std::vector<float> download(const Handle* H, const float* dptr, int64_t count) {
  std::vector<float> v((size_t)count);
  VQMC_CUDA(cudaMemcpyAsync(v.data(), dptr, count * sizeof(float), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  return v;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    VQMC_CUDA(cudaGetDevice(&prev));
    if (prev != dev) VQMC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Sticky device flag: a logit of the fp16-pair GEMMs was not finite (operand overflow).  The
// reference computes in fp64 and would not overflow here, so fail loudly (runtime_error, like
// the reference's non-finite local-energy check, estimator.hpp:85-87) instead of drawing junk.
// Bit 1: a general spec's local energy was not finite (estimator.hpp:85-87).
static void check_flag(Handle* H, uint32_t v) {
  if (!v) return;
  VQMC_CUDA(cudaMemsetAsync(H->d_flag, 0, sizeof(uint32_t), H->stream));
  H->next_call = ~0ull;  // (the device step counters are re-seeded from the caller's next call)
  if (v & 1u) throw NumericError("non-finite logit in the tail sampler (fp16 operand range exceeded)");
  throw NumericError("non-finite local energy (amplitude underflow?)");
}
static void sync_check_flag(Handle* H) {
  VQMC_CUDA(cudaMemcpyAsync(H->h_scal + 8, H->d_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  check_flag(H, *reinterpret_cast<const uint32_t*>(H->h_scal + 8));
}

// Side stream of the concurrent backward / gradient all-reduce (high priority) and its events.
static void ensure_side_stream(Handle* H) {
  if (H->cstream) return;
  int lo = 0, hi = 0;
  VQMC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  VQMC_CUDA(cudaStreamCreateWithPriority(&H->cstream, cudaStreamNonBlocking, hi));
  VQMC_CUDA(cudaEventCreateWithFlags(&H->ev_fork, cudaEventDisableTiming));
  VQMC_CUDA(cudaEventCreateWithFlags(&H->ev_join, cudaEventDisableTiming));
  VQMC_CUDA(cudaEventCreateWithFlags(&H->ev_dg1, cudaEventDisableTiming));
  VQMC_CUDA(cudaEventCreateWithFlags(&H->ev_dz1, cudaEventDisableTiming));
}

static void check_B(int B) {
  if (B < 1) throw std::invalid_argument("batch size must be >= 1");
}

// The statistics / REINFORCE-weights kernel keeps the whole batch's weights in shared memory
// (4 bytes per sample per CTA): the fused step and evaluate accept batches up to that limit
// (~56K samples per GPU handle; the reference has no cap, so fail with a clear message).
static void check_stats_batch(int B) {
  int dev = 0, optin = 0;
  VQMC_CUDA(cudaGetDevice(&dev));
  VQMC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int64_t cap = (optin - 4096) / (int64_t)sizeof(float);  // (the kernel's static shared memory)
  if ((int64_t)B > cap)
    throw std::invalid_argument("batch of " + std::to_string(B) + " samples exceeds the per-GPU statistics limit of " +
                                std::to_string(cap) + " (split the batch over more workers' handles or GPUs)");
}

static void upload_bits(Handle* H, const uint32_t* bits, int B) {
  VQMC_CUDA(cudaMemcpyAsync(H->X, bits, (size_t)B * H->L.W * sizeof(uint32_t), cudaMemcpyHostToDevice,
                            H->stream));
}

// Sampling into the handle's batch buffers (X, G1, D, log_psi).  The batch is
// `workers` segments of B / workers rows; segment s draws from stream
// (stream0 + s) (trainer.cpp:126: worker w uses make_stream(seed, w + 1)).
static void sample_into(Handle* H, int B, int workers, const double* uniforms_host, uint64_t seed,
                        uint64_t stream0, uint64_t call, bool device_call = false, bool want_log_psi = true) {
  H->ensure_batch(B);
  const double* du = nullptr;
  if (uniforms_host) {
    H->ensure_uniforms((int64_t)H->L.n * B);
    VQMC_CUDA(cudaMemcpyAsync(H->uni, uniforms_host, (size_t)H->L.n * B * sizeof(double),
                              cudaMemcpyHostToDevice, H->stream));
    du = H->uni;
  }
  RngSpec rng{seed, stream0, call, B / workers, device_call ? H->d_step : nullptr};
  launch_head_v2(H, B, du, rng, false, nullptr);  // head and tail together write every word of X
  launch_z2(H, B, H->L.Hd, du, rng, false, nullptr, want_log_psi);
  if (want_log_psi) launch_finalize_logpsi(H, B, H->tail_tiles);  // the training step never reads log psi
}

// Forward from configurations already in H->X (models.cpp:51-70): layer 1 and the tcgen05
// layer-2 GEMM with the given-bits epilogue (spec.cu), log psi into H->log_psi.
static void forward_given(Handle* H, int B, double* cond) {
  forward_plain(H, B, cond, nullptr, nullptr, nullptr, H->log_psi);
}

// The step's host-visible results live in one device block (read back with one copy):
// [0] ||g||^2 (double), [8] the non-finite-logit flag (uint32), [16 ...] per-segment integer cut
// statistics (3 int64 per segment); mirrored by a pinned host block of the same layout.
static void ensure_istat(Handle* H, int segs) {
  if (segs <= H->istat_cap) return;
  const size_t words = 16 + (size_t)3 * segs;  // 8-byte words
  if (H->d_scal) VQMC_CUDA(cudaFree(H->d_scal));
  VQMC_CUDA(cudaMalloc((void**)&H->d_scal, words * 8));
  VQMC_CUDA(cudaMemset(H->d_scal, 0, words * 8));
  H->d_flag = reinterpret_cast<uint32_t*>(H->d_scal + 8);
  H->d_istat = reinterpret_cast<int64_t*>(H->d_scal + 16);
  if (H->h_scal) VQMC_CUDA(cudaFreeHost(H->h_scal));
  VQMC_CUDA(cudaMallocHost((void**)&H->h_scal, words * 8));
  H->h_istat = reinterpret_cast<int64_t*>(H->h_scal + 16);
  H->istat_cap = segs;
}

// one copy of the step's results (||g||^2, flag, cut statistics of `segs` segments, and with a
// communicator the reduced statistics limbs of all ranks); blocks
// The step's scalar results (grad norm, flag, per-segment cut sums; multi-GPU: the all-reduced
// statistics limbs) into the pinned host mirrors.  Captured into the step's graph, so a replay
// ends with them already copied.
static void enqueue_results_copy(Handle* H, int segs) {
  VQMC_CUDA(cudaMemcpyAsync(H->h_scal, H->d_scal, (16 + (size_t)3 * segs) * 8, cudaMemcpyDeviceToHost, H->stream));
  if (H->nccl_comm)
    VQMC_CUDA(cudaMemcpyAsync(H->h_rstat, H->G + H->L.total, rstat_count(H->nranks) * sizeof(float),
                              cudaMemcpyDeviceToHost, H->stream));
}
static void read_step_results(Handle* H, int segs, bool copied = false) {
  if (!copied) enqueue_results_copy(H, segs);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));  // (a busy-wait measured the same)
  check_flag(H, *reinterpret_cast<const uint32_t*>(H->h_scal + 8));
}

// Pooled cut statistics of the step: this rank's segments, or (communicator) every rank's, decoded
// from the all-reduced limbs (sums exact; best = max over the ranks' slots).
struct CutTotals {
  int64_t cs = 0, cq = 0, best = 0, N = 0;
};
static CutTotals step_totals(const Handle* H, int segs, int B) {
  CutTotals t;
  if (H->nccl_comm) {
    auto limbs = [&](int off, int cnt) {
      uint64_t v = 0;
      for (int k = 0; k < cnt; ++k) v += (uint64_t)llrintf(H->h_rstat[off + k]) << (16 * k);
      return v;
    };
    t.cs = (int64_t)limbs(0, 3);
    t.cq = (int64_t)limbs(3, 4);
    for (int r = 0; r < H->nranks; ++r) t.best = std::max(t.best, (int64_t)limbs(7 + 2 * r, 2));
    t.N = (int64_t)B * H->nranks;
    return t;
  }
  for (int s = 0; s < segs; ++s) {
    t.cs += H->h_istat[3 * s];
    t.cq += H->h_istat[3 * s + 1];
    t.best = std::max(t.best, H->h_istat[3 * s + 2]);
  }
  t.N = B;
  return t;
}

// Pooled mean / unbiased variance of N Max-Cut local energies l = (E - 2c)/4
// from exact integer sums of c and c^2 (estimator.hpp:94-100; the fp64
// two-pass result is exact for Max-Cut whenever its partial sums are, and
// this evaluates the same rational with one rounding).
static void pooled_stats(int64_t E, int64_t N, int64_t cs, int64_t cq, double* mean, double* var) {
  const __int128 num = (__int128)N * E - 2 * (__int128)cs;  // 4 * sum(l)
  *mean = ((double)num * 0.25) / (double)N;
  const __int128 ssn = (__int128)N * cq - (__int128)cs * cs;  // 4 N * sum (l - mean)^2
  const double ss = (double)ssn / (4.0 * (double)N);
  *var = N > 1 ? ss / (double)(N - 1) : 0.0;
}

static void grad_to_host(Handle* H, double* grad_out) {
  const auto g = download(H, H->G, H->L.total);
  live_to_reference(H, g, nullptr, grad_out);
}

// HamiltonianSpec::validate for a Max-Cut pair list (hamiltonian.cpp:36-54).
static void validate_edges(int n, const int32_t* edges, int64_t num_edges) {
  if (num_edges < 0) throw std::invalid_argument("num_edges must be >= 0");
  std::vector<int64_t> keys((size_t)num_edges);
  for (int64_t t = 0; t < num_edges; ++t) {
    const int i = edges[2 * t], j = edges[2 * t + 1];
    if (i < 0 || j >= n || i >= j) throw std::invalid_argument("pair indices must satisfy 0 <= i < j < n");
    keys[t] = (int64_t)i * n + j;
  }
  std::sort(keys.begin(), keys.end());
  if (std::adjacent_find(keys.begin(), keys.end()) != keys.end()) throw std::invalid_argument("duplicate pair");
}

// Edge list for the bit-sliced cut kernel: entries u | v << 16 (n <= 65536; swizzled indices, see
// maxcut_cut_kernel) grouped into aligned batches of 32 in which the u's are pairwise distinct
// mod 32 and so are the v's (orientation is
// free: the cut term is symmetric), so a warp's two shared-memory lookups per edge hit 32 distinct
// banks.  Greedy first fit over a window of open batches; unfilled slots point at two of the kernel's
// 32 zero words (one per bank) on banks still free (XOR = 0: no contribution).  The order of the integer sum
// does not matter (exact).
static std::vector<uint32_t> bank_order_edges(int W, const int32_t* edges, int64_t num_edges) {
  struct Batch {
    uint32_t lu = 0, lv = 0;
    uint32_t e[32];
    int cnt = 0;
  };
  std::vector<Batch> batches;
  std::vector<int> open;  // indices of batches that are not full (window)
  // open-batch window: 256 packs a random 3-regular N = 10k instance to 5% padding (48: 16%)
  const size_t kWindow = num_edges <= 300000 ? 256 : 48;
  for (int64_t t = 0; t < num_edges; ++t) {
    // swizzled word indices of the cut kernel's transposed spins: node i at i ^ (((i >> 5) & 7) << 2)
    const uint32_t u0 = (uint32_t)edges[2 * t], v0 = (uint32_t)edges[2 * t + 1];
    const uint32_t u = u0 ^ (((u0 >> 5) & 7u) << 2), v = v0 ^ (((v0 >> 5) & 7u) << 2);
    const uint32_t bu = 1u << (u & 31), bv = 1u << (v & 31);
    bool placed = false;
    for (size_t k = open.size(); k-- > 0 && !placed;) {
      Batch& b = batches[open[k]];
      if (!(b.lu & bu) && !(b.lv & bv)) {
        b.lu |= bu, b.lv |= bv, b.e[b.cnt++] = u | v << 16;
        placed = true;
      } else if (!(b.lu & bv) && !(b.lv & bu)) {
        b.lu |= bv, b.lv |= bu, b.e[b.cnt++] = v | u << 16;
        placed = true;
      }
      if (placed && b.cnt == 32) open.erase(open.begin() + (long)k);
    }
    if (!placed) {
      batches.emplace_back();
      Batch& b = batches.back();
      b.lu = bu, b.lv = bv, b.e[b.cnt++] = u | v << 16;
      open.push_back((int)batches.size() - 1);
      if (open.size() > kWindow) open.erase(open.begin());  // oldest leaves the window (padded later)
    }
  }
  const uint32_t zero = 32u * (uint32_t)W;  // 32 zero words after the transposed spins (kernel)
  do batches.emplace_back();  // whole blocks of 4 batches (at least one)
  while (batches.size() % 4);
  for (Batch& b : batches) {
    for (int k = b.cnt; k < 32; ++k) {  // pad: a zero word on a free bank on each side (XOR = 0)
      const uint32_t pu = (uint32_t)__builtin_ctz(~b.lu), pv = (uint32_t)__builtin_ctz(~b.lv);
      b.lu |= 1u << pu, b.lv |= 1u << pv;
      b.e[k] = (zero + pu) | (zero + pv) << 16;
    }
  }
  // entries as byte offsets (4 u | 4 v << 16; 32 W + 32 <= 16384 words), and within each block of
  // 128 entries lane l's 16-byte quad holds entry l of the block's 4 batches: the kernel's warp reads
  // one quad per lane and its q-th lookups are batch q's (conflict-free) entries
  std::vector<uint32_t> out(batches.size() * 32);
  for (size_t blk = 0; blk < batches.size() / 4; ++blk)
    for (int q = 0; q < 4; ++q)
      for (int l = 0; l < 32; ++l) {
        const uint32_t e = batches[4 * blk + q].e[l];
        out[128 * blk + 4 * l + q] = (e & 0xFFFFu) * 4u | ((e >> 16) * 4u) << 16;
      }
  return out;
}

static void upload_edges(Handle* H, const int32_t* edges, int64_t num_edges) {
  if (H->d_edges) VQMC_CUDA(cudaFree(H->d_edges));
  H->d_edges = nullptr;
  if (H->d_edges_bank) VQMC_CUDA(cudaFree(H->d_edges_bank));
  H->d_edges_bank = nullptr;
  H->num_edges_bank = 0;
  H->num_edges = num_edges;
  if (32 * H->L.W + 32 <= 16384 && !dense_energy_preferred(H->L.n, num_edges)) {
    const std::vector<uint32_t> pk = bank_order_edges(H->L.W, edges, num_edges);
    VQMC_CUDA(cudaMalloc((void**)&H->d_edges_bank, pk.size() * sizeof(uint32_t)));
    VQMC_CUDA(cudaMemcpy(H->d_edges_bank, pk.data(), pk.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    H->num_edges_bank = (int64_t)pk.size();
  }
  if (num_edges > 0) {
    // (+2 entries: the energy kernel's bulk copies round a chunk up to an even edge count)
    VQMC_CUDA(cudaMalloc((void**)&H->d_edges, (num_edges + 2) * sizeof(int2)));
    VQMC_CUDA(cudaMemset(H->d_edges, 0, (num_edges + 2) * sizeof(int2)));
    VQMC_CUDA(cudaMemcpy(H->d_edges, edges, num_edges * sizeof(int2), cudaMemcpyHostToDevice));
  }
  setup_dense_energy(H);  // dense instances (e.g. the reference's G(n, 3/4)): the tensor-core quadratic form
}

}  // namespace vqmc_b200

using namespace vqmc_b200;

#define API_TRY try {
#define API_CATCH                     \
  }                                   \
  catch (const std::exception& ex) {  \
    set_error(ex.what());             \
    return status_of(ex);             \
  }                                   \
  return VQMC_OK;

extern "C" {

const char* vqmc_last_error(void) { return g_error.c_str(); }

int vqmc_gpu_device_count(int* count) {
  API_TRY
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  *count = c;
  API_CATCH
}

int vqmc_gpu_create(int device, int n, int h, const int32_t* degrees, const double* theta,
                    const int32_t* edges, int64_t num_edges, int max_batch, vqmc_gpu_t** out) {
  Handle* H = nullptr;
  API_TRY
  if (n < 2) throw std::invalid_argument("MADE requires n >= 2");
  if (h < 1) throw std::invalid_argument("MADE requires h >= 1");
  if (h > kMaxHidden) throw std::invalid_argument("hidden width > 1024 is not supported on the GPU path");
  if (num_edges < 0) throw std::invalid_argument("num_edges must be >= 0");
  int Hd = 0;
  for (int k = 0; k < h; ++k) {
    if (degrees[k] < 1 || degrees[k] > n - 1) throw std::invalid_argument("degrees must lie in [1, n-1]");
    Hd = std::max(Hd, (int)degrees[k]);
  }
  validate_edges(n, edges, num_edges);
  H = new Handle();
  H->device = device;
  DeviceGuard dg(device);
  VQMC_CUDA(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
  if (const char* e = std::getenv("VQMC_PDL")) H->pdl = e[0] == '1';
  if (const char* e = std::getenv("VQMC_SERIAL_BW")) H->concurrent_bw = e[0] != '1';
  H->gw2_sms = n >= 8192 ? 80 : 64;  // (gW2's 2 x ceil(n / 128) pair tiles in whole rounds; internal.cuh)
  if (const char* e = std::getenv("VQMC_GW2_SMS")) H->gw2_sms = std::max(2, atoi(e));
  if (const char* e = std::getenv("VQMC_GW1_SPLITS")) H->gw1_splits = atoi(e);
  if (const char* e = std::getenv("VQMC_ADAM_SMS")) H->adam_w2_sms = std::max(2, atoi(e));
  H->L.init(n, h, Hd);
  if (H->L.total >= (int64_t(1) << 31)) throw std::invalid_argument("model too large for the device layout (> 2^31 live parameters)");
  H->hp8 = (h + 7) & ~7;
  H->hp18 = (h + 1 + 7) & ~7;
  H->np8 = (n + 15) & ~15;  // (32-byte rows: the sampler epilogue writes D with 256-bit stores)
  H->hd18 = (Hd + 1 + 7) & ~7;
  H->d = 2LL * h * n + h + n;
  H->degrees.assign(degrees, degrees + h);
  H->num_edges = num_edges;
  dalloc(&H->P, (size_t)H->L.total);
  dalloc(&H->G, (size_t)H->L.total + rstat_count(kMaxRanks));
  dalloc(&H->Mo, (size_t)H->L.total);
  dalloc(&H->Vo, (size_t)H->L.total);
  VQMC_CUDA(cudaMemsetAsync(H->G, 0, (H->L.total + rstat_count(kMaxRanks)) * sizeof(float), H->stream));
  VQMC_CUDA(cudaMallocHost((void**)&H->h_rstat, rstat_count(kMaxRanks) * sizeof(float)));
  VQMC_CUDA(cudaMemsetAsync(H->Mo, 0, H->L.total * sizeof(float), H->stream));
  VQMC_CUDA(cudaMemsetAsync(H->Vo, 0, H->L.total * sizeof(float), H->stream));
  dalloc(&H->gw1_part, (size_t)kGw1MaxSplits * (Hd + 1) * h);
  dalloc(&H->W2h, (size_t)n * H->hp18 + 128);
  dalloc(&H->W2l, (size_t)n * H->hp18 + 128);
  VQMC_CUDA(cudaMemset(H->W2h, 0, ((size_t)n * H->hp18 + 128) * sizeof(__half)));
  VQMC_CUDA(cudaMemset(H->W2l, 0, ((size_t)n * H->hp18 + 128) * sizeof(__half)));
  dalloc(&H->d_deg, (size_t)h);
  VQMC_CUDA(cudaMemcpy(H->d_deg, degrees, h * sizeof(int32_t), cudaMemcpyHostToDevice));
  {  // completion lists: hidden units by degree
    std::vector<int32_t> off(Hd + 1, 0), ks;
    for (int k = 0; k < h; ++k) off[degrees[k]]++;  // degree d completes at step d-1 -> slot d-1
    // off[i+1] counts units with degree i+1; prefix sum
    std::vector<int32_t> cnt(Hd + 1, 0);
    for (int k = 0; k < h; ++k) cnt[degrees[k] - 1]++;
    off.assign(Hd + 1, 0);
    for (int i = 0; i < Hd; ++i) off[i + 1] = off[i] + cnt[i];
    ks.resize(h);
    std::vector<int32_t> pos(off.begin(), off.end() - 1);
    for (int k = 0; k < h; ++k) ks[pos[degrees[k] - 1]++] = k;
    dalloc(&H->d_comp_k, (size_t)h);
    dalloc(&H->d_comp_off, (size_t)Hd + 1);
    VQMC_CUDA(cudaMemcpy(H->d_comp_k, ks.data(), h * sizeof(int32_t), cudaMemcpyHostToDevice));
    VQMC_CUDA(cudaMemcpy(H->d_comp_off, off.data(), (Hd + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
    H->comp_off_host = off;
    H->w1skip = true;
    for (int k = 0; k < h; ++k) H->w1skip = H->w1skip && degrees[k] <= k + 1;
    H->head_fast = true;
    for (int i = 0; i < Hd; ++i) H->head_fast = H->head_fast && off[i + 1] - off[i] == 1 && ks[off[i]] == i;
    // staged head rows: v3 (fast structure) uses 128-float lane groups, v2 a power-of-two word count
    const int kp = H->head_fast ? 128 * ((h + 127) / 128)
                                : 32 * ((h + 31) / 32 <= 1 ? 1 : (h + 31) / 32 <= 2 ? 2 : (h + 31) / 32 <= 4 ? 4
                                        : (h + 31) / 32 <= 8 ? 8 : (h + 31) / 32 <= 16 ? 16 : 32);
    // rows padded to a multiple of 8 with zero rows (the v3 head runs whole 8-bit ring slots)
    const size_t r1 = (size_t)((Hd + 7) & ~7), r2 = (size_t)((h + 7) & ~7);
    dalloc(&H->W1Tp, r1 * kp);
    dalloc(&H->W2cp, r2 * kp);
    VQMC_CUDA(cudaMemset(H->W1Tp, 0, r1 * kp * sizeof(float)));
    VQMC_CUDA(cudaMemset(H->W2cp, 0, r2 * kp * sizeof(float)));
    H->head_hpk = kp;
    H->head_Hdp = H->head_fast ? kp : 32 * ((Hd + 31) / 32);
    const char* hv = std::getenv("VQMC_HEAD");  // "3": keep the v3 head sampler (A/B measurements)
    H->head_v4 = H->head_fast && !(hv && hv[0] == '3');
    H->head_v5 = H->head_v4 && !(hv && hv[0] == '4');
    if (H->head_v4) {
      const int KG = kp / 128, nwords = (h + 31) / 32;
      const size_t af = (size_t)nwords * KG * 2 * 8192, tri = (size_t)nwords * 32 * 64;  // halves, floats
      dalloc(&H->h4.AF, af);
      dalloc(&H->h4.TRI, tri);
      VQMC_CUDA(cudaMemset(H->h4.AF, 0, af * sizeof(__half)));
      VQMC_CUDA(cudaMemset(H->h4.TRI, 0, tri * sizeof(float)));
      H->h4.KG = KG;
    }
    std::vector<int32_t> cpos(h);
    for (int c = 0; c < h; ++c) cpos[ks[c]] = c;
    dalloc(&H->d_comp_pos, (size_t)h);
    VQMC_CUDA(cudaMemcpy(H->d_comp_pos, cpos.data(), h * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  upload_edges(H, edges, num_edges);
  dalloc(&H->d_step, 1);
  dalloc(&H->d_done, 1);
  VQMC_CUDA(cudaMemset(H->d_done, 0, sizeof(unsigned)));
  dalloc(&H->d_wscale, 1);
  ensure_istat(H, 64);  // (d_scal, d_flag, d_istat and their host mirror)
  H->gpart_n = 148 * 8;  // Adam ||g||^2 partials: part 0 (<= half) + part 1, or one whole launch (<= 592)
  dalloc(&H->d_gpart, (size_t)H->gpart_n);
  for (auto& e : H->ev) VQMC_CUDA(cudaEventCreate(&e));
  for (int i = 0; i < Handle::kKtPool; ++i) {
    VQMC_CUDA(cudaEventCreate(&H->kt_start[i]));
    VQMC_CUDA(cudaEventCreate(&H->kt_end[i]));
  }
  H->ensure_batch(std::max(2, max_batch));
  upload_params(H, theta);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  *out = reinterpret_cast<vqmc_gpu_t*>(H);
  H = nullptr;
  }
  catch (const std::exception& ex) {
    set_error(ex.what());
    delete H;
    return status_of(ex);
  }
  return VQMC_OK;
}

int vqmc_gpu_destroy(vqmc_gpu_t* g) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  if (!H) return VQMC_OK;
  DeviceGuard dg(H->device);
  cudaStreamSynchronize(H->stream);
  H->invalidate_graph();
  if (H->nccl_comm && g_nccl.CommDestroy) g_nccl.CommDestroy(H->nccl_comm);
  if (H->cstream) cudaStreamDestroy(H->cstream);
  if (H->ev_fork) cudaEventDestroy(H->ev_fork);
  if (H->ev_join) cudaEventDestroy(H->ev_join);
  if (H->ev_dg1) cudaEventDestroy(H->ev_dg1);
  if (H->ev_dz1) cudaEventDestroy(H->ev_dz1);
  free_sr(H);
  free_dense_energy(H);
  spec_free(H);
  if (H->d_lstat) cudaFree(H->d_lstat);
  if (H->d_edges_bank) cudaFree(H->d_edges_bank);
  void* ptrs[] = {H->P, H->G, H->Mo, H->Vo, H->W1Tp, H->W2cp, H->W2h, H->W2l, H->d_deg, H->d_comp_k,
                  H->d_comp_off, H->d_edges, H->X, H->G1, H->G1h, H->G1l, H->wG1h, H->wG1l, H->Dh, H->Dl,
                  H->lp_head, H->thr, H->lp_part, H->log_psi, H->cut, H->cpart, H->local, H->w, H->d_wscale,
                  H->Epart, H->dz1bh, H->dz1bl, H->Xfb, H->gw1_part, H->cond, H->uni, H->d_scal,
                  H->d_gpart, H->d_step, H->d_done, H->d_comp_pos, H->h4.AF, H->h4.TRI};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (H->h_scal) cudaFreeHost(H->h_scal);
  if (H->h_rstat) cudaFreeHost(H->h_rstat);
  for (auto& e : H->ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < Handle::kKtPool; ++i) {
    if (H->kt_start[i]) cudaEventDestroy(H->kt_start[i]);
    if (H->kt_end[i]) cudaEventDestroy(H->kt_end[i]);
  }
  cudaStreamDestroy(H->stream);
  delete H;
  API_CATCH
}

int vqmc_gpu_set_edges(vqmc_gpu_t* g, const int32_t* edges, int64_t num_edges) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  validate_edges(H->L.n, edges, num_edges);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  H->invalidate_graph();
  upload_edges(H, edges, num_edges);
  API_CATCH
}

int vqmc_gpu_param_count(const vqmc_gpu_t* g, int64_t* d) {
  API_TRY
  *d = reinterpret_cast<const Handle*>(g)->d;
  API_CATCH
}

int vqmc_gpu_set_params(vqmc_gpu_t* g, const double* theta) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  upload_params(H, theta);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_get_params(vqmc_gpu_t* g, double* theta) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  const auto P = download(H, H->P, H->L.total);
  live_to_reference(H, P, H->theta_host.data(), theta);
  API_CATCH
}

int vqmc_gpu_sample(vqmc_gpu_t* g, int B, const double* uniforms, uint64_t seed, uint64_t stream,
                    uint64_t call, uint32_t* bits_out, double* log_psi_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  check_B(B);
  sample_into(H, B, 1, uniforms, seed, stream, call);
  if (bits_out)
    VQMC_CUDA(cudaMemcpyAsync(bits_out, H->X, (size_t)B * H->L.W * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, H->stream));
  if (log_psi_out)
    VQMC_CUDA(cudaMemcpyAsync(log_psi_out, H->log_psi, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost,
                              H->stream));
  VQMC_CUDA(cudaMemcpyAsync(H->h_scal + 8, H->d_flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  check_flag(H, *reinterpret_cast<const uint32_t*>(H->h_scal + 8));
  API_CATCH
}

int vqmc_gpu_log_psi(vqmc_gpu_t* g, const uint32_t* bits, int B, double* log_psi_out, double* cond_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  check_B(B);
  H->ensure_batch(B);
  upload_bits(H, bits, B);
  double* cond = nullptr;
  if (cond_out) {
    H->ensure_cond((int64_t)B * H->L.n);
    cond = H->cond;
  }
  forward_given(H, B, cond);
  if (log_psi_out)
    VQMC_CUDA(cudaMemcpyAsync(log_psi_out, H->log_psi, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost,
                              H->stream));
  if (cond_out)
    VQMC_CUDA(cudaMemcpyAsync(cond_out, cond, (size_t)B * H->L.n * sizeof(double), cudaMemcpyDeviceToHost,
                              H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_maxcut_energy(vqmc_gpu_t* g, const uint32_t* bits, int B, int32_t* cut_out, double* local_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  check_B(B);
  H->ensure_batch(B);
  upload_bits(H, bits, B);
  launch_energy(H, B);
  launch_cuts_reduce(H, B);
  std::vector<int32_t> cuts((size_t)B);
  VQMC_CUDA(cudaMemcpyAsync(cuts.data(), H->cut, (size_t)B * sizeof(int32_t), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  if (cut_out) std::memcpy(cut_out, cuts.data(), (size_t)B * sizeof(int32_t));
  if (local_out)  // l_b = (|E| - 2 cut_b) / 4 (exact in fp64), as the device statistics use it
    for (int b = 0; b < B; ++b) local_out[b] = 0.25 * ((double)H->num_edges - 2.0 * (double)cuts[b]);
  API_CATCH
}

int vqmc_gpu_set_spec(vqmc_gpu_t* g, const double* alpha, const double* beta, const int32_t* pair_i,
                      const int32_t* pair_j, const double* pair_value, int64_t num_pairs) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  spec_set(H, alpha, beta, pair_i, pair_j, pair_value, num_pairs);
  API_CATCH
}

int vqmc_gpu_clear_spec(vqmc_gpu_t* g) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  spec_free(H);
  H->invalidate_graph();
  API_CATCH
}

int vqmc_gpu_local_energy(vqmc_gpu_t* g, const uint32_t* bits, int B, const double* cached_log_psi,
                          double* local_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  check_B(B);
  if (!H->spec) return vqmc_gpu_maxcut_energy(g, bits, B, nullptr, local_out);  // the diagonal branch
  H->ensure_batch(B);
  upload_bits(H, bits, B);
  const double* dc = nullptr;
  if (cached_log_psi) {
    double* c = spec_cached_buffer(H, B);
    VQMC_CUDA(cudaMemcpyAsync(c, cached_log_psi, (size_t)B * sizeof(double), cudaMemcpyHostToDevice, H->stream));
    dc = c;
  }
  double* dl = spec_local_buffer(H, B);
  launch_spec_local(H, B, dc, dl);
  if (local_out)
    VQMC_CUDA(cudaMemcpyAsync(local_out, dl, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  sync_check_flag(H);
  API_CATCH
}

int vqmc_gpu_weighted_grad(vqmc_gpu_t* g, const uint32_t* bits, const double* weights, int B,
                           double* grad_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  check_B(B);
  H->ensure_batch(B);
  upload_bits(H, bits, B);
  // normalised weights w' = w / wscale, wscale = 2^e >= max |w| (as stats_weights_kernel does)
  double wmax = 0.0;
  for (int b = 0; b < B; ++b) wmax = std::max(wmax, std::fabs((double)(float)weights[b]));
  int e = 0;
  if (wmax > 0.0) std::frexp(wmax, &e);
  const float sc = std::ldexp(1.f, e);
  std::vector<float> wf(B);
  for (int b = 0; b < B; ++b) wf[b] = std::ldexp((float)weights[b], -e);
  VQMC_CUDA(cudaMemcpyAsync(H->w, wf.data(), B * sizeof(float), cudaMemcpyHostToDevice, H->stream));
  VQMC_CUDA(cudaMemcpyAsync(H->d_wscale, &sc, sizeof(float), cudaMemcpyHostToDevice, H->stream));
  forward_given(H, B, nullptr);
  launch_backward(H, B);
  grad_to_host(H, grad_out);
  API_CATCH
}

int vqmc_gpu_gradient_from_locals(vqmc_gpu_t* g, const uint32_t* bits, const double* local, int B,
                                  double* grad_out) {
  API_TRY
  if (B < 2) throw std::invalid_argument("gradient estimate needs at least two samples");
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += local[b];
  const double mean = s / (double)B;
  std::vector<double> w(B);
  for (int b = 0; b < B; ++b) w[b] = 2.0 * (local[b] - mean) / (double)B;
  return vqmc_gpu_weighted_grad(g, bits, w.data(), B, grad_out);
  API_CATCH
}

int vqmc_gpu_adam_step(vqmc_gpu_t* g, const double* grad, double lr, double beta1, double beta2, double eps,
                       int64_t t) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (t < 1) throw std::invalid_argument("adam step count must be >= 1");
  if (grad) {
    const Layout& L = H->L;
    const int n = L.n, h = L.h;
    std::vector<float> G((size_t)L.total, 0.f);
    const double* gW1 = grad;
    const double* gb1 = gW1 + (size_t)h * n;
    const double* gW2 = gb1 + h;
    const double* gb2 = gW2 + (size_t)n * h;
    for (int j = 0; j < L.Hd; ++j)
      for (int k = 0; k < h; ++k)
        G[L.off_w1t + (size_t)j * h + k] = (j + 1 <= H->degrees[k]) ? (float)gW1[(size_t)k * n + j] : 0.f;
    for (int k = 0; k < h; ++k) G[L.off_b1 + k] = (float)gb1[k];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < h; ++k)
        G[L.off_w2 + (size_t)i * h + k] = (H->degrees[k] < i + 1) ? (float)gW2[(size_t)i * h + k] : 0.f;
    for (int i = 0; i < n; ++i) G[L.off_b2 + i] = (float)gb2[i];
    VQMC_CUDA(cudaMemcpyAsync(H->G, G.data(), G.size() * sizeof(float), cudaMemcpyHostToDevice, H->stream));
  }
  launch_set_step(H, 0, t, lr, beta1, beta2, eps);
  H->next_call = ~0ull;  // the next train step must re-seed the device counters
  launch_adam(H, 1.0f, /*gated=*/false);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_adam_reset(vqmc_gpu_t* g) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  VQMC_CUDA(cudaMemsetAsync(H->Mo, 0, H->L.total * sizeof(float), H->stream));
  VQMC_CUDA(cudaMemsetAsync(H->Vo, 0, H->L.total * sizeof(float), H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_comm_unique_id(uint8_t id_out[128]) {
  API_TRY
  load_nccl();
  NcclUniqueId id;
  nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id_out, id.internal, 128);
  API_CATCH
}

int vqmc_gpu_comm_init(vqmc_gpu_t* g, const uint8_t id[128], int nranks, int rank) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad nranks/rank");
  if (nranks > kMaxRanks) throw std::invalid_argument("at most 256 ranks (exact fp32 statistics limbs)");
  H->nranks = nranks;
  H->rank = rank;
  // nranks == 1 needs no communicator; VQMC_NCCL_SELF=1 still creates one (a one-rank NCCL
  // all-reduce) so the overlapped-collective path can be exercised on a single GPU
  const char* self = std::getenv("VQMC_NCCL_SELF");
  if (nranks == 1 && !(self && self[0] == '1')) return VQMC_OK;
  load_nccl();
  NcclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  ncclComm_t comm = nullptr;
  nccl_check(g_nccl.CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  H->nccl_comm = comm;
  ensure_side_stream(H);
  H->gemm_sm_reserve = 16;  // SMs left to NCCL while the backward GEMMs overlap the all-reduce
  H->invalidate_graph();
  API_CATCH
}

}  // extern "C"

namespace vqmc_b200 {

void Handle::invalidate_graph() {
  if (gexec) cudaGraphExecDestroy(gexec);
  gexec = nullptr;
  gkey = GraphKey{};
  graph_warm = false;
}

// The work of one training step (worker_body, trainer.cpp:150-282) on the handle's stream.
// The Philox counter and the Adam step are taken from H->d_step, which the first kernel
// advances, so the same sequence can be captured once and replayed as a CUDA graph.
static void enqueue_train_step(Handle* H, int minibatch, int workers, const double* uniforms, uint64_t seed,
                               uint64_t stream0) {
  const int B = minibatch * workers;
  H->kt_count = 0;
  const bool tm = H->phase_timing >= 2, t0 = H->phase_timing >= 1;
  if (t0) record_event(H, H->ev[0]);
  sample_into(H, B, workers, uniforms, seed, stream0, 0, /*device_call=*/true, /*want_log_psi=*/false);
  if (tm) record_event(H, H->ev[1]);
  launch_energy(H, B);                                // local_energy_batch (:161)
  launch_weights_from_locals(H, B, minibatch, true);  // gradient_from_locals weights (:164) + w' G1 operand
  if (tm) record_event(H, H->ev[2]);
  const Layout& L = H->L;
  if (H->concurrent_bw && H->ktimer != 1) {
    // weighted_grad_log_psi with its two independent halves concurrent: gW2 / gb2 (and, multi-GPU,
    // their all-reduce: 99% of the gradient bytes) on cstream with gw2_sms SMs, dg1 -> dz1 -> gW1
    // on the main stream with the rest; then the small W1 / b1 all-reduce and the join.
    // allreduce_mean (:187) is summed here and divided by L in Adam.
    ensure_side_stream(H);
    const int avail = gemm_sms(nullptr) - H->gemm_sm_reserve;
    VQMC_CUDA(cudaEventRecord(H->ev_fork, H->stream));
    VQMC_CUDA(cudaStreamWaitEvent(H->cstream, H->ev_fork, 0));
    H->gemm_sm_cap = std::min(H->gw2_sms, avail - 16);
    launch_gw2_umma(H, B, /*wg1_done=*/true, H->cstream);
    if (H->nccl_comm)
      nccl_check(g_nccl.AllReduce(H->G + L.off_w2, H->G + L.off_w2,
                                  (size_t)(L.total - L.off_w2) + rstat_count(H->nranks), ncclFloat32, ncclSum,
                                  H->nccl_comm, H->cstream),
                 "ncclAllReduce (W2, b2, cut statistics)");
    H->gemm_sm_cap = avail - std::min(H->gw2_sms, avail - 16);
    launch_dg1_umma(H, B);  // the step's last read of the W2 operand pairs
    VQMC_CUDA(cudaEventRecord(H->ev_dg1, H->stream));
    const float gs = 1.0f / (float)(workers * H->nranks);
    // adam_step (:221) on [W2 | b2] once its gradient is reduced and dz1 (after dg1, the last
    // reader of the W2 pairs) is done: gW1's CTAs, enqueued first, take the SMs before Adam's
    // blocks fill them (gW1 15 vs 29 us; step -2 us vs starting Adam right after dg1)
    launch_backward_after_dg1(H, B, H->ev_dz1);
    VQMC_CUDA(cudaStreamWaitEvent(H->cstream, H->ev_dz1, 0));
    launch_adam_part(H, gs, 0, H->cstream);
    VQMC_CUDA(cudaEventRecord(H->ev_join, H->cstream));
    H->gemm_sm_cap = 0;
    if (tm) record_event(H, H->ev[3]);
    if (H->nccl_comm)
      nccl_check(g_nccl.AllReduce(H->G, H->G, (size_t)L.off_w2, ncclFloat32, ncclSum, H->nccl_comm, H->stream),
                 "ncclAllReduce (W1, b1)");
    if (tm) record_event(H, H->ev[4]);
    launch_adam_part(H, gs, 1, H->stream);  // [W1T | b1]
    VQMC_CUDA(cudaStreamWaitEvent(H->stream, H->ev_join, 0));
    if (t0) record_event(H, H->ev[5]);
    return;
  } else {
    launch_backward(H, B, /*wg1_done=*/true);  // weighted_grad_log_psi (serial; per-kernel timing)
    if (tm) record_event(H, H->ev[3]);
    if (H->nccl_comm)
      nccl_check(g_nccl.AllReduce(H->G, H->G, (size_t)L.total + rstat_count(H->nranks), ncclFloat32, ncclSum,
                                  H->nccl_comm, H->stream),
                 "ncclAllReduce");
    if (tm) record_event(H, H->ev[4]);
  }
  launch_adam(H, 1.0f / (float)(workers * H->nranks), /*gated=*/true);  // adam_step (:221)
  if (t0) record_event(H, H->ev[5]);
}

// The same iteration on a general spec (TIM): the sampler keeps log psi (the cached value of the
// off-diagonal ratios, trainer.cpp:157-162), fp64 local energies with the flipped-neighbour
// branch (spec.cu), weights from them, the serial backward, the gradient all-reduce plus a small
// fp64 one of the energy sums, and Adam (skipped when the step's flag is set).
static void enqueue_train_step_spec(Handle* H, int minibatch, int workers, const double* uniforms, uint64_t seed,
                                    uint64_t stream0) {
  const int B = minibatch * workers;
  H->kt_count = 0;
  const bool tm = H->phase_timing >= 2, t0 = H->phase_timing >= 1;
  if (t0) record_event(H, H->ev[0]);
  sample_into(H, B, workers, uniforms, seed, stream0, 0, /*device_call=*/true, /*want_log_psi=*/true);
  if (tm) record_event(H, H->ev[1]);
  double* dl = spec_local_buffer(H, B);
  launch_spec_local(H, B, H->log_psi, dl);                                 // local_energy_batch (:161)
  launch_weights_from_locals(H, B, minibatch, true, dl, H->d_lstat);      // gradient_from_locals (:164)
  if (tm) record_event(H, H->ev[2]);
  launch_backward(H, B, /*wg1_done=*/true);
  if (tm) record_event(H, H->ev[3]);
  if (H->nccl_comm) {
    nccl_check(g_nccl.AllReduce(H->G, H->G, (size_t)H->L.total, ncclFloat32, ncclSum, H->nccl_comm, H->stream),
               "ncclAllReduce");
    nccl_check(g_nccl.AllReduce(H->d_lstat, H->d_lstat, 2, ncclFloat64, ncclSum, H->nccl_comm, H->stream),
               "ncclAllReduce (energy sums)");
  }
  if (tm) record_event(H, H->ev[4]);
  launch_adam(H, 1.0f / (float)(workers * H->nranks), /*gated=*/true);
  if (t0) record_event(H, H->ev[5]);
}

}  // namespace vqmc_b200

extern "C" {

int vqmc_gpu_train_step(vqmc_gpu_t* g, int minibatch, int workers, const double* uniforms, uint64_t seed,
                        uint64_t stream0, uint64_t call, double lr, double beta1, double beta2, double eps,
                        int64_t t, vqmc_step_stats_t* stats_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (minibatch < 2) throw std::invalid_argument("minibatch must be >= 2");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (t < 1) throw std::invalid_argument("adam step count must be >= 1");
  if ((int64_t)minibatch * workers > INT32_MAX) throw std::invalid_argument("batch too large");
  const int B = minibatch * workers;
  check_stats_batch(B);
  H->last_grad_scale = 1.0f / (float)(workers * H->nranks);
  H->last_grad_sr = false;
  if (B > H->cap_B) H->invalidate_graph();
  H->ensure_batch(B);
  if (workers > H->istat_cap) H->invalidate_graph();
  ensure_istat(H, workers);
  // device step counters describe the step about to run; Adam advances them at the step's end
  if (call != H->next_call || t != H->next_t || lr != H->cur_lr || beta1 != H->cur_b1 || beta2 != H->cur_b2 ||
      eps != H->cur_eps) {
    launch_set_step(H, call, t, lr, beta1, beta2, eps);
    H->cur_lr = lr;
    H->cur_b1 = beta1;
    H->cur_b2 = beta2;
    H->cur_eps = eps;
  }
  if (H->spec) {  // general spec (TIM): eager, no captured graph
    if (2 + 2 * workers > H->lstat_cap) {
      if (H->d_lstat) VQMC_CUDA(cudaFree(H->d_lstat));
      H->d_lstat = nullptr;
      VQMC_CUDA(cudaMalloc((void**)&H->d_lstat, (size_t)(2 + 2 * workers) * sizeof(double)));
      H->lstat_cap = 2 + 2 * workers;
    }
    enqueue_train_step_spec(H, minibatch, workers, uniforms, seed, stream0);
    H->next_call = call + 1;
    H->next_t = t + 1;
    if (stats_out) {
      read_step_results(H, workers);
      double ls[2];
      VQMC_CUDA(cudaMemcpy(ls, H->d_lstat, sizeof(ls), cudaMemcpyDeviceToHost));
      const double N = (double)B * H->nranks;
      const double mean = ls[0] / N;
      stats_out->energy_mean = mean;
      stats_out->energy_var = N > 1 ? std::max(0.0, (ls[1] - N * mean * mean) / (N - 1)) : 0.0;
      stats_out->grad_norm = std::sqrt(H->h_scal[0]);
      stats_out->cut_sum = 0;
      stats_out->cut_sq_sum = 0;
      stats_out->best_cut = 0;
      stats_out->batch = (int32_t)N;
    }
    return VQMC_OK;
  }
  const bool graphable = H->graph_enabled && uniforms == nullptr;
  Handle::GraphKey key;
  key.valid = true;
  key.minibatch = minibatch;
  key.workers = workers;
  key.phase_timing = H->phase_timing;
  key.ktimer = H->ktimer;
  key.seed = seed;
  key.stream0 = stream0;
  bool copied = false;
  if (!graphable) {
    enqueue_train_step(H, minibatch, workers, uniforms, seed, stream0);
  } else if (H->gexec && H->gkey == key) {
    VQMC_CUDA(cudaGraphLaunch(H->gexec, H->stream));  // replay the captured step
    copied = true;
  } else if (!H->graph_warm || !(H->gkey == key)) {
    if (H->gexec) {
      cudaGraphExecDestroy(H->gexec);
      H->gexec = nullptr;
    }
    enqueue_train_step(H, minibatch, workers, uniforms, seed, stream0);  // eager warm-up step
    H->graph_warm = true;
    H->gkey = key;
  } else {
    cudaGraph_t graph = nullptr;
    VQMC_CUDA(cudaStreamBeginCapture(H->stream, cudaStreamCaptureModeThreadLocal));
    H->capturing = true;
    try {
      enqueue_train_step(H, minibatch, workers, uniforms, seed, stream0);
      enqueue_results_copy(H, workers);  // (the replay ends with the scalars on the host)
      H->capturing = false;
    } catch (...) {
      H->capturing = false;
      cudaStreamEndCapture(H->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    VQMC_CUDA(cudaStreamEndCapture(H->stream, &graph));
    VQMC_CUDA(cudaGraphInstantiate(&H->gexec, graph, 0));
    cudaGraphDestroy(graph);
    H->gkey = key;
    VQMC_CUDA(cudaGraphLaunch(H->gexec, H->stream));
    copied = true;
  }
  H->next_call = call + 1;
  H->next_t = t + 1;
  if (stats_out) {
    read_step_results(H, workers, copied);
    const CutTotals t = step_totals(H, workers, B);
    pooled_stats(H->num_edges, t.N, t.cs, t.cq, &stats_out->energy_mean, &stats_out->energy_var);
    stats_out->grad_norm = std::sqrt(H->h_scal[0]);
    stats_out->cut_sum = t.cs;
    stats_out->cut_sq_sum = t.cq;
    stats_out->best_cut = (int32_t)t.best;
    stats_out->batch = (int32_t)t.N;
  }
  API_CATCH
}

int vqmc_gpu_sr_direction(vqmc_gpu_t* g, const uint32_t* bits, int B, const double* grad, double lambda, double tol,
                          int max_iterations, int centered, double* delta_out, int* iterations_out,
                          double* residual_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (B < 2) throw std::invalid_argument("Fisher needs at least two samples");  // estimator.hpp:153
  if (max_iterations < 0) throw std::invalid_argument("max_iterations must be >= 0");
  H->ensure_batch(B);
  ensure_sr(H, B);
  upload_bits(H, bits, B);
  forward_given(H, B, nullptr);  // G1, D of the configurations
  launch_dg1_umma(H, B);         // D . W2m partials (dz1 of the scores)
  const std::vector<double> gl = reference_to_live(H, grad);
  VQMC_CUDA(cudaMemcpyAsync(H->cg_g, gl.data(), gl.size() * sizeof(double), cudaMemcpyHostToDevice, H->stream));
  int it = 0;
  double res = 0.0;
  const bool ok = sr_solve(H, B, lambda, tol, max_iterations, centered != 0, &it, &res, nullptr);
  if (iterations_out) *iterations_out = it;
  if (residual_out) *residual_out = res;
  if (!ok)
    throw SrSolveError("SR conjugate gradient did not converge (relative residual " + std::to_string(res) +
                       " after " + std::to_string(it) + " iterations)");
  std::vector<double> x((size_t)H->L.total);
  VQMC_CUDA(cudaMemcpyAsync(x.data(), H->cg_x, x.size() * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  live_to_reference_d(H, x, delta_out);
  API_CATCH
}

// Test hook: the explicit fp64 score rows of the small-model SR path (d <= 2000), uncentred,
// reference order [B][d]: forward + dg1 of `bits`, then the score kernel.
int vqmc_test_sr_scores(vqmc_gpu_t* g, const uint32_t* bits, int B, double* out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (H->d > 2000) throw std::invalid_argument("explicit scores only for d <= 2000");
  H->ensure_batch(B);
  ensure_sr(H, B);
  upload_bits(H, bits, B);
  forward_given(H, B, nullptr);
  launch_dg1_umma(H, B);
  sr_build_scores(H, B, false);
  const int64_t total = H->L.total;
  std::vector<double> S((size_t)B * total);
  VQMC_CUDA(cudaMemcpyAsync(S.data(), H->sr_S, S.size() * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  for (int b = 0; b < B; ++b) {
    std::vector<double> row(S.begin() + (size_t)b * total, S.begin() + (size_t)(b + 1) * total);
    live_to_reference_d(H, row, out + (size_t)b * H->d);
  }
  API_CATCH
}

int vqmc_gpu_train_step_sr(vqmc_gpu_t* g, int minibatch, int workers, const double* uniforms, uint64_t seed,
                           uint64_t stream0, uint64_t call, double lr, double lambda, double tol, int max_iterations,
                           int fallback, int centered, vqmc_step_stats_t* stats_out, int* iterations_out,
                           double* residual_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (minibatch < 2) throw std::invalid_argument("minibatch must be >= 2");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (max_iterations < 0) throw std::invalid_argument("max_iterations must be >= 0");
  if (H->nranks > 1 && H->d <= 2000)
    throw std::invalid_argument("multi-GPU SR needs the CG path (reference d > 2000)");
  if ((int64_t)minibatch * workers > INT32_MAX) throw std::invalid_argument("batch too large");
  const int B = minibatch * workers;
  check_stats_batch(B);
  H->ensure_batch(B);
  ensure_istat(H, workers);
  ensure_sr(H, B);
  launch_set_step(H, call, 1, lr, 0.9, 0.999, 1e-8);  // (the sampler's Philox call; t / Adam unused)
  H->next_call = ~uint64_t(0);                         // an ADAM step after this one resets the counters
  // phase 1: sample, local energies, REINFORCE weights, gradient (trainer.cpp:155-168)
  sample_into(H, B, workers, uniforms, seed, stream0, 0, /*device_call=*/true, /*want_log_psi=*/false);
  launch_energy(H, B);
  launch_weights_from_locals(H, B, minibatch, true);
  launch_backward(H, B, /*wg1_done=*/true);
  // phase 2: allreduce_mean (the segments' and ranks' summed gradient / L, and the statistics limbs)
  // and the natural-gradient solve over the pooled scores of every rank (trainer.cpp:187-199)
  if (H->nccl_comm) comm_allreduce_sum(H, H->G, (size_t)H->L.total + rstat_count(H->nranks), false);
  read_step_results(H, workers);
  const CutTotals tot = step_totals(H, workers, B);
  launch_sr_grad_from_G(H, 1.0 / ((double)workers * H->nranks));
  H->last_grad_sr = true;
  int it = 0;
  double res = 0.0, gnorm = 0.0;
  const bool ok = sr_solve(H, B, lambda, tol, max_iterations, centered != 0, &it, &res, &gnorm);
  if (iterations_out) *iterations_out = it;
  if (residual_out) *residual_out = res;
  if (!ok && !fallback)
    throw SrSolveError("SR conjugate gradient did not converge (relative residual " + std::to_string(res) +
                       " after " + std::to_string(it) + " iterations)");
  // phase 3: sgd_step with the natural direction (or the raw gradient on a tolerated failure)
  launch_sr_apply(H, lr, ok ? H->cg_x : H->cg_g);
  launch_params_refresh(H);
  H->invalidate_graph();
  if (stats_out) {
    pooled_stats(H->num_edges, tot.N, tot.cs, tot.cq, &stats_out->energy_mean, &stats_out->energy_var);
    stats_out->grad_norm = gnorm;
    stats_out->cut_sum = tot.cs;
    stats_out->cut_sq_sum = tot.cq;
    stats_out->best_cut = (int32_t)tot.best;
    stats_out->batch = (int32_t)tot.N;
  }
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_last_cuts(vqmc_gpu_t* g, int32_t* cuts_out, int B) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (B > H->cap_B) throw std::invalid_argument("B exceeds the batch capacity");
  VQMC_CUDA(cudaMemcpyAsync(cuts_out, H->cut, (size_t)B * sizeof(int32_t), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_last_samples(vqmc_gpu_t* g, uint32_t* bits_out, int B) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (B < 0 || B > H->cap_B) throw std::invalid_argument("B exceeds the batch capacity");
  VQMC_CUDA(cudaMemcpyAsync(bits_out, H->X, (size_t)B * H->L.W * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int vqmc_gpu_last_gradient(vqmc_gpu_t* g, double* grad_out) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (H->last_grad_sr) {  // SGD + SR step: the reduced gradient is the CG right-hand side (fp64)
    std::vector<double> x((size_t)H->L.total);
    VQMC_CUDA(cudaMemcpyAsync(x.data(), H->cg_g, x.size() * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
    VQMC_CUDA(cudaStreamSynchronize(H->stream));
    live_to_reference_d(H, x, grad_out);
  } else {
    auto G = download(H, H->G, H->L.total);
    for (auto& v : G) v *= H->last_grad_scale;  // (the step keeps the sum; Adam applies 1 / L on the fly)
    live_to_reference(H, G, nullptr, grad_out);
  }
  API_CATCH
}

int vqmc_gpu_evaluate(vqmc_gpu_t* g, int B, const double* uniforms, uint64_t seed, uint64_t stream,
                      uint64_t call, double out[4]) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  DeviceGuard dg(H->device);
  if (B < 2) throw std::invalid_argument("variance needs at least two samples");
  check_stats_batch(B);
  sample_into(H, B, 1, uniforms, seed, stream, call);
  if (H->spec) {  // general spec: energy and std of the fp64 local energies; no cut (trainer.cpp:91-108)
    double* dl = spec_local_buffer(H, B);
    launch_spec_local(H, B, H->log_psi, dl);
    std::vector<double> l((size_t)B);
    VQMC_CUDA(cudaMemcpyAsync(l.data(), dl, (size_t)B * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
    sync_check_flag(H);
    double sum = 0.0;
    for (double v : l) sum += v;
    const double mean = sum / (double)B;
    double ss = 0.0;
    for (double v : l) ss += (v - mean) * (v - mean);
    out[0] = mean;
    out[1] = std::sqrt(ss / (double)(B - 1));
    out[2] = 0.0;
    out[3] = 0.0;
    return VQMC_OK;
  }
  launch_energy(H, B);
  launch_weights_from_locals(H, B, B);
  VQMC_CUDA(cudaMemcpyAsync(H->h_istat, H->d_istat, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  double mean, var;
  pooled_stats(H->num_edges, B, H->h_istat[0], H->h_istat[1], &mean, &var);
  out[0] = mean;
  out[1] = std::sqrt(var);
  out[2] = std::max(0.0, (double)H->h_istat[2]);  // best = max(0.0, cuts), trainer.cpp:98-104
  out[3] = (double)H->h_istat[0] / (double)B;     // total / rows (exact integer total)
  API_CATCH
}

int vqmc_pooled_stats(int64_t num_edges, int64_t N, int64_t cut_sum, int64_t cut_sq_sum, double* mean,
                      double* var) {
  API_TRY
  if (N < 2) throw std::invalid_argument("variance needs at least two samples");
  pooled_stats(num_edges, N, cut_sum, cut_sq_sum, mean, var);
  API_CATCH
}

int vqmc_gpu_synchronize(vqmc_gpu_t* g) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  API_CATCH
}

int64_t vqmc_gpu_launch_count(const vqmc_gpu_t* g) { return reinterpret_cast<const Handle*>(g)->launches; }

int vqmc_gpu_set_graph(vqmc_gpu_t* g, int enable) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  H->graph_enabled = enable != 0;
  H->invalidate_graph();
  API_CATCH
}

int vqmc_gpu_set_phase_timing(vqmc_gpu_t* g, int enable) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  H->phase_timing = enable < 0 ? 0 : enable > 2 ? 2 : enable;
  API_CATCH
}

int vqmc_gpu_set_kernel_timing(vqmc_gpu_t* g, int enable) {
  API_TRY
  reinterpret_cast<Handle*>(g)->ktimer = enable <= 0 ? 0 : enable >= 2 ? 2 : 1;
  API_CATCH
}

int vqmc_gpu_kernel_timeline(vqmc_gpu_t* g, char* names_out, float* start_ms, float* end_ms, int cap, int* count) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  if (H->phase_timing < 1) throw std::invalid_argument("kernel timeline needs phase timing >= 1 (the step-start event)");
  VQMC_CUDA(cudaDeviceSynchronize());
  const int c = std::min(cap, H->kt_count);
  for (int i = 0; i < c; ++i) {
    VQMC_CUDA(cudaEventElapsedTime(&start_ms[i], H->ev[0], H->kt_start[i]));
    VQMC_CUDA(cudaEventElapsedTime(&end_ms[i], H->ev[0], H->kt_end[i]));
    std::strncpy(names_out + 32 * i, H->kt_name[i], 31);
    names_out[32 * i + 31] = 0;
  }
  *count = c;
  API_CATCH
}

int vqmc_gpu_kernel_times(vqmc_gpu_t* g, char* names_out, float* ms_out, int cap, int* count) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  const int c = std::min(cap, H->kt_count);
  for (int i = 0; i < c; ++i) {
    VQMC_CUDA(cudaEventElapsedTime(&ms_out[i], H->kt_start[i], H->kt_end[i]));
    std::strncpy(names_out + 32 * i, H->kt_name[i], 31);
    names_out[32 * i + 31] = 0;
  }
  *count = c;
  API_CATCH
}

int vqmc_gpu_phase_times(vqmc_gpu_t* g, float out_ms[5]) {
  API_TRY
  Handle* H = reinterpret_cast<Handle*>(g);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  if (H->phase_timing >= 2) {
    for (int i = 0; i < 5; ++i) VQMC_CUDA(cudaEventElapsedTime(&out_ms[i], H->ev[i], H->ev[i + 1]));
  } else {
    VQMC_CUDA(cudaEventElapsedTime(&out_ms[0], H->ev[0], H->ev[5]));  // level 1: whole step only
    for (int i = 1; i < 5; ++i) out_ms[i] = 0.f;
  }
  API_CATCH
}

}  // extern "C"
