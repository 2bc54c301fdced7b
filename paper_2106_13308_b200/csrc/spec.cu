// General Ising specs (the TIM branch of the reference) and the plain forward of given
// configurations, for sm_100a.
//
//   H = -sum_i (alpha_i X_i + beta_i Z_i) - sum_{i<j} beta_ij Z_i Z_j      hamiltonian.hpp:26-44
//   l(x) = H_xx - sum_{k: alpha_k > 0} alpha_k psi(x ^ e_k) / psi(x)        estimator.hpp:43-90
//
// The reference evaluates every flipped neighbour with a full forward pass (B s rows of n
// conditionals, chunked).  Here the MADE structure does most of that work once:
//   * a flip of bit k >= Hd (the largest hidden degree) changes no hidden unit, so
//     log psi(x ^ e_k) - log psi(x) = (log p_k(1 - x_k) - log p_k(x_k)) / 2 comes from the base
//     forward's logit of output k alone (fterm);
//   * a flip of bit k < Hd changes z1 by +-W1m[:, k] (one rank-1 update of the base z1) and only
//     the conditionals of outputs i >= k: the neighbour rows [relu(z1 +- W1m[:, k]) | 1] go through
//     the tcgen05 pair GEMM with [W2m | b2] (launch_nbr_umma) whose epilogue sums
//     log p_i(x'_i) for i >= k; the base's suffix sum of the same terms is subtracted.
// The diagonal H_xx is an fp64 sum over the pair list on bit-sliced spins (32 samples per word).
//
// Plain forward (made_forward + log_prob, models.cpp:51-70, for log_psi / weighted_grad / SR /
// TIM): z1_given_kernel writes [G1 | 1] (fp32 and the fp16 pair), the spins' bf16 operand of gW1
// and optionally z1; launch_given_umma runs the layer-2 GEMM over every output with the
// given-bits epilogue.  No sampling chain is involved.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace vqmc_b200 {

#define SPEC_LAUNCH_CHECK() VQMC_CUDA(cudaGetLastError())

int launch_nbr_umma(Handle* H, int rows, int Bc, int b0, const int32_t* sites, const __half* Nh, const __half* Nl,
                    double* part);
void launch_given_umma(Handle* H, int B, double* cond, float* lterm, float* fterm);

template <class T>
static void salloc(T** p, size_t count) {
  if (*p) VQMC_CUDA(cudaFree(*p));
  *p = nullptr;
  if (count) VQMC_CUDA(cudaMalloc((void**)p, count * sizeof(T)));
}
template <class T>
static void sfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// ===========================================================================
// Layer 1 of given configurations: z1[b][k] = b1[k] + sum_{j < Hd} x_bj W1T[j][k] (the live W1T
// holds only inputs below the largest degree; masked entries are exact zeros).  kS samples per
// CTA (spins staged as floats in shared memory), one thread per hidden unit.
// ===========================================================================
constexpr int kZ1S = 8;
__global__ void __launch_bounds__(1024) z1_given_kernel(int B, int h, int Hd, int W, int hp, int hd1p,
                                                        const uint32_t* __restrict__ X,
                                                        const float* __restrict__ W1T, const float* __restrict__ b1,
                                                        float* __restrict__ G1, __half* __restrict__ G1h,
                                                        __half* __restrict__ G1l, __nv_bfloat16* __restrict__ Xf,
                                                        float* __restrict__ Z1) {
  __shared__ __align__(16) float xs[kZ1S][kMaxHidden];
  const int b0 = blockIdx.x * kZ1S, tid = threadIdx.x;
  const int Hd4 = (Hd + 3) & ~3;
  for (int t = tid; t < kZ1S * Hd4; t += blockDim.x) {
    const int s = t / Hd4, j = t % Hd4, b = b0 + s;
    float x = 0.f;
    if (b < B && j < Hd) {
      x = (float)((X[(size_t)b * W + (j >> 5)] >> (j & 31)) & 1u);
      Xf[(size_t)b * hd1p + j] = __float2bfloat16_rn(x);
    }
    xs[s][j] = x;
    if (b < B && j == 0) Xf[(size_t)b * hd1p + Hd] = __float2bfloat16_rn(1.f);  // ones column: gb1
  }
  __syncthreads();
  for (int k = tid; k < h; k += blockDim.x) {
    float acc[kZ1S];
    const float bk = b1[k];
#pragma unroll
    for (int s = 0; s < kZ1S; ++s) acc[s] = bk;
    for (int j = 0; j < Hd4; j += 4) {
      float w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = j + u < Hd ? W1T[(size_t)(j + u) * h + k] : 0.f;
#pragma unroll
      for (int s = 0; s < kZ1S; ++s) {
        const float4 xv = *reinterpret_cast<const float4*>(&xs[s][j]);
        acc[s] = fmaf(xv.x, w[0], acc[s]);
        acc[s] = fmaf(xv.y, w[1], acc[s]);
        acc[s] = fmaf(xv.z, w[2], acc[s]);
        acc[s] = fmaf(xv.w, w[3], acc[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < kZ1S; ++s) {
      const int b = b0 + s;
      if (b >= B) break;
      const float g = fmaxf(acc[s], 0.f);
      G1[(size_t)b * h + k] = g;
      ptx::split_f16(g, G1h[(size_t)b * hp + k], G1l[(size_t)b * hp + k]);
      if (Z1) Z1[(size_t)b * h + k] = acc[s];
    }
  }
}

// Small batches (B < 64): one warp per (sample, hidden unit), lanes over the inputs (fixed-order
// shuffle reduction): the CTA-per-8-samples kernel above would leave almost every SM idle.
__global__ void __launch_bounds__(256) z1_given_small_kernel(int B, int h, int Hd, int W, int hp, int hd1p,
                                                             const uint32_t* __restrict__ X,
                                                             const float* __restrict__ W1T,
                                                             const float* __restrict__ b1, float* __restrict__ G1,
                                                             __half* __restrict__ G1h, __half* __restrict__ G1l,
                                                             __nv_bfloat16* __restrict__ Xf,
                                                             float* __restrict__ Z1) {
  const int wid = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (wid < B * ((Hd + 31) / 32)) {  // (the first warps also write the spins' bf16 operand)
    const int b = wid / ((Hd + 31) / 32), j = 32 * (wid % ((Hd + 31) / 32)) + lane;
    if (j < Hd) Xf[(size_t)b * hd1p + j] = __float2bfloat16_rn((float)((X[(size_t)b * W + (j >> 5)] >> (j & 31)) & 1u));
    if (j == 0) Xf[(size_t)b * hd1p + Hd] = __float2bfloat16_rn(1.f);  // ones column: gb1
  }
  if (wid >= B * h) return;
  const int b = wid / h, k = wid % h;
  float acc = 0.f;
  for (int j = lane; j < Hd; j += 32)
    if ((X[(size_t)b * W + (j >> 5)] >> (j & 31)) & 1u) acc += W1T[(size_t)j * h + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) {
    const float z = acc + b1[k];
    const float g = fmaxf(z, 0.f);
    G1[(size_t)b * h + k] = g;
    ptx::split_f16(g, G1h[(size_t)b * hp + k], G1l[(size_t)b * hp + k]);
    if (Z1) Z1[(size_t)b * h + k] = z;
  }
}

// log_psi[b] = (lp_head[b] (optional) + sum of the row's partials) / 2
__global__ void finalize_lp_kernel(int B, int tiles, const double* __restrict__ lp_part,
                                   double* __restrict__ out) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  double s = 0.0;
  for (int t = lane; t < tiles; t += 32) s += lp_part[(size_t)t * B + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) out[b] = 0.5 * s;  // log_psi_batch = log_prob / 2 (models.cpp:126-128)
}

// Forward of the configurations in H->X: [G1 | 1], D, log psi (into lp_out), optional p and
// per-output log terms / flip deltas and z1.
void forward_plain(Handle* H, int B, double* cond, float* lterm, float* fterm, float* Z1, double* lp_out) {
  const Layout& L = H->L;
  {
    KScope ks(H, "z1_given");
    if (B < 64) {
      const int64_t warps = std::max<int64_t>((int64_t)B * L.h, (int64_t)B * ((L.Hd + 31) / 32));
      z1_given_small_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, H->stream>>>(
          B, L.h, L.Hd, L.W, H->hp18, H->hd18, H->X, H->P + L.off_w1t, H->P + L.off_b1, H->G1, H->G1h, H->G1l,
          H->Xfb, Z1);
    } else {
      const int threads = std::min(1024, (L.h + 31) & ~31);
      z1_given_kernel<<<(B + kZ1S - 1) / kZ1S, threads, 0, H->stream>>>(
          B, L.h, L.Hd, L.W, H->hp18, H->hd18, H->X, H->P + L.off_w1t, H->P + L.off_b1, H->G1, H->G1h, H->G1l,
          H->Xfb, Z1);
    }
    SPEC_LAUNCH_CHECK();
    H->launches++;
  }
  launch_given_umma(H, B, cond, lterm, fterm);
  H->launches++;
  {
    KScope ks(H, "finalize_logpsi");
    finalize_lp_kernel<<<(B + 7) / 8, 256, 0, H->stream>>>(B, H->tail_tiles, H->lp_part, lp_out);
    SPEC_LAUNCH_CHECK();
    H->launches++;
  }
}

// ===========================================================================
// Diagonal energy (hamiltonian.cpp:61-69).  G <= 32 samples per CTA as bit-sliced node words
// T[i] (bit l = spin i of sample b0 + l, one ballot per node); threads stream the CTA's chunk of
// the pair list with coalesced loads and every thread keeps G fp64 accumulators:
//   -beta_i s_i = x_i ? beta_i : -beta_i,   -v s_i s_j = (x_i ^ x_j) ? v : -v
//   = 2 sum_{bit set} v - sum v   (one predicated add per sample and pair).
// Dense mode (the complete row-major pair list of random_tim): only the values are read, the
// indices follow from the position; a warp walks row i (lanes over j) and its mirror row
// n - 2 - i, so every warp task has n - 1 pairs.  Partials per (chunk, sample).
// ===========================================================================
// Bit-sliced spins of G-sample groups: Tg[g][i] bit l = spin i of sample g G + l (one warp per
// 32 nodes: lane l loads sample l's word, 32 ballots transpose it).
__global__ void spec_slice_kernel(int B, int n, int W, int G, const uint32_t* __restrict__ X,
                                  uint32_t* __restrict__ Tg) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // word column
  const int g = blockIdx.y;
  if (w >= W) return;
  const int b = g * G + lane;
  const uint32_t xw = lane < G && b < B ? X[(size_t)b * W + w] : 0u;
  uint32_t mine = 0;
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const uint32_t word = __ballot_sync(kFull, (xw >> t) & 1u);
    if (lane == t) mine = word;
  }
  if (32 * w + lane < n) Tg[(size_t)g * n + 32 * w + lane] = mine;
}

template <int G>
__global__ void __launch_bounds__(256) spec_diag_kernel(int B, int n, const uint32_t* __restrict__ Tg,
                                                        const double* __restrict__ beta, int dense, int64_t np,
                                                        int64_t per_chunk, const int32_t* __restrict__ pi,
                                                        const int32_t* __restrict__ pj,
                                                        const double* __restrict__ pv, double* __restrict__ dpart) {
  extern __shared__ uint32_t T[];  // [n]
  __shared__ double red[8][G];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b0 = blockIdx.x * G;
  for (int i = tid; i < n; i += blockDim.x) T[i] = Tg[(size_t)blockIdx.x * n + i];
  __syncthreads();
  double acc[G];
#pragma unroll
  for (int l = 0; l < G; ++l) acc[l] = 0.0;
  double vsum = 0.0;
  auto add = [&](uint32_t w, double v) {
    vsum += v;
#pragma unroll
    for (int l = 0; l < G; ++l)
      if ((w >> l) & 1u) acc[l] += v;
  };
  if (blockIdx.y == 0)
    for (int i = tid; i < n; i += blockDim.x) add(T[i], beta[i]);  // x_i ? +beta : -beta
  if (dense) {
    // row pairs (i, n - 2 - i), i < (n - 1) / 2 (+ the middle row when n - 1 is odd); 16 loads in
    // flight per lane for <= 4 samples per CTA, else 8 (at B = 4 the walk is a pure stream of the
    // n^2/2 values: latency-bound)
    const int64_t r0 = (int64_t)blockIdx.y * per_chunk, r1 = min((int64_t)(n / 2), r0 + per_chunk);
    for (int64_t rp = r0 + warp; rp < r1; rp += 8) {
      for (int half = 0; half < 2; ++half) {
        const int i = half ? n - 2 - (int)rp : (int)rp;
        if (half && i <= (int)rp) break;  // (the middle row is walked once)
        const double* row = pv + ((int64_t)i * n - (int64_t)i * (i + 1) / 2) - (i + 1);  // row[j], j > i
        const uint32_t ti = T[i];
        int j = i + 1 + lane;
        constexpr int D = G <= 4 ? 16 : 8;  // loads in flight per lane (few accumulators: go deeper)
        for (; j + 32 * (D - 1) < n; j += 32 * D) {
          double v[D];
#pragma unroll
          for (int u = 0; u < D; ++u) v[u] = row[j + 32 * u];
#pragma unroll
          for (int u = 0; u < D; ++u) add(ti ^ T[j + 32 * u], v[u]);
        }
        for (; j + 224 < n; j += 256) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = row[j + 32 * u];
#pragma unroll
          for (int u = 0; u < 8; ++u) add(ti ^ T[j + 32 * u], v[u]);
        }
        for (; j + 96 < n; j += 128) {
          const double v0 = row[j], v1 = row[j + 32], v2 = row[j + 64], v3 = row[j + 96];
          add(ti ^ T[j], v0);
          add(ti ^ T[j + 32], v1);
          add(ti ^ T[j + 64], v2);
          add(ti ^ T[j + 96], v3);
        }
        for (; j < n; j += 32) add(ti ^ T[j], row[j]);
      }
    }
  } else {
    const int64_t p0 = (int64_t)blockIdx.y * per_chunk, p1 = min(np, p0 + per_chunk);
#pragma unroll 4
    for (int64_t p = p0 + tid; p < p1; p += blockDim.x) add(T[pi[p]] ^ T[pj[p]], pv[p]);
  }
  // sample l: 2 acc_l - vsum (vsum covers the fields and the pairs this thread saw)
#pragma unroll
  for (int l = 0; l < G; ++l) {
    double v = 2.0 * acc[l] - vsum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) red[warp][l] = v;
  }
  __syncthreads();
  if (tid < G) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][tid];
    if (b0 + tid < B) dpart[(size_t)blockIdx.y * B + b0 + tid] = s;
  }
}

// ===========================================================================
// Neighbour rows: row r = t * Bc + (b - b0), site k = sites[t] < Hd:
//   [G1' | 1] = [relu(z1_b + (x_bk ? -1 : 1) W1T[k]) | 1]   (fp16 pair, row stride hp)
// One warp per group of kNbrR rows (the rows' site / spin / z1 / W1T loads all in flight before
// use): coalesced z1 / W1T reads, 4-byte (half2) stores.
// ===========================================================================
constexpr int kNbrR = 4;
__global__ void __launch_bounds__(256) nbr_build_kernel(int rows, int Bc, int b0, int h, int hp, int W,
                                                        const int32_t* __restrict__ sites,
                                                        const uint32_t* __restrict__ X, const float* __restrict__ Z1,
                                                        const float* __restrict__ W1T, __half* __restrict__ Nh,
                                                        __half* __restrict__ Nl) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r0 = kNbrR * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r0 < rows; r0 += kNbrR * nw) {
    int k[kNbrR], b[kNbrR];
    bool x[kNbrR];
#pragma unroll
    for (int q = 0; q < kNbrR; ++q) {
      const int r = min(r0 + q, rows - 1);  // (a clamped duplicate row is recomputed, not stored)
      k[q] = sites[r / Bc];
      b[q] = b0 + r % Bc;
    }
#pragma unroll
    for (int q = 0; q < kNbrR; ++q) x[q] = (X[(size_t)b[q] * W + (k[q] >> 5)] >> (k[q] & 31)) & 1u;
    for (int c = 2 * lane; c < hp; c += 64) {
      float zv[kNbrR][2], wv[kNbrR][2];
#pragma unroll
      for (int q = 0; q < kNbrR; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const bool in = c + u < h;
          zv[q][u] = in ? Z1[(size_t)b[q] * h + c + u] : 0.f;
          wv[q][u] = in ? W1T[(size_t)k[q] * h + c + u] : 0.f;
        }
#pragma unroll
      for (int q = 0; q < kNbrR; ++q) {
        if (r0 + q >= rows) break;
        float g[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          g[u] = c + u < h ? fmaxf(zv[q][u] + (x[q] ? -wv[q][u] : wv[q][u]), 0.f) : (c + u == h ? 1.f : 0.f);
        uint32_t hi, lo;
        ptx::split_f16x2(g[0], g[1], hi, lo);
        const size_t o = ((size_t)(r0 + q) * hp + c) >> 1;
        reinterpret_cast<__half2*>(Nh)[o] = *reinterpret_cast<const __half2*>(&hi);
        reinterpret_cast<__half2*>(Nl)[o] = *reinterpret_cast<const __half2*>(&lo);
      }
    }
  }
}

// nb[t * B + b] = sum of the neighbour row's partials (fixed order)
__global__ void nbr_reduce_kernel(int rows, int Bc, int b0, int B, int parts, const double* __restrict__ part,
                                  double* __restrict__ nb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += part[(size_t)p * rows + r];
  nb[(size_t)(r / Bc) * B + b0 + r % Bc] = s;
}

// ===========================================================================
// Local energies (estimator.hpp:59-89), one CTA per sample:
//   d_k = log psi(x ^ e_k) - cached_b
//       = (nb_k - sum_{i >= k} lterm_i) / 2 + (lpf_b - cached_b)    k < Hd
//       = fterm_k / 2 + (lpf_b - cached_b)                           k >= Hd
//   shift = max(0, max_k d_k) if > 50 else 0;  l_b = H_xx - e^shift sum_k alpha_k e^(d_k - shift)
// The suffix sums are total - prefix, the prefixes of the first Hd terms come from one block
// scan (fp64).
// ===========================================================================
template <int T>
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if (T == 32) return v;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < T / 32; ++k) s += red[k];
  return s;
}
template <int T>
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  if (T == 32) return v;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
#pragma unroll
  for (int k = 1; k < T / 32; ++k) s = fmax(s, red[k]);
  return s;
}

// T threads per sample (32 for small models, 256 for large ones)
template <int T>
__global__ void __launch_bounds__(T) spec_local_kernel(int B, int n, int Hd, int S, int sH,
                                                       const int32_t* __restrict__ sites,
                                                       const double* __restrict__ alpha_s, int chunks,
                                                       const double* __restrict__ dpart,
                                                       const float* __restrict__ lterm,
                                                       const float* __restrict__ fterm,
                                                       const double* __restrict__ nb,
                                                       const double* __restrict__ lpf,
                                                       const double* __restrict__ cached, double* __restrict__ local,
                                                       uint32_t* __restrict__ flag) {
  __shared__ double red[T / 32];
  __shared__ double pre[kMaxHidden + 1];  // exclusive prefix of lterm over the head positions
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double v = 0.0;
  for (int c = tid; c < chunks; c += T) v += dpart[(size_t)c * B + b];
  const double diag = block_sum<T>(v, red);
  double acc = 0.0;
  if (S > 0) {
    const double corr = lpf[b] - cached[b];
    const float* lt = lterm + (size_t)b * n;
    const float* ft = fterm + (size_t)b * n;
    v = 0.0;
    for (int i = tid; i < n; i += T) v += (double)lt[i];
    const double tot = block_sum<T>(v, red);
    if (sH > 0) {  // block scan of lterm[0 .. Hd): E consecutive terms per thread (Hd <= 1024)
      const int E = (Hd + T - 1) / T, i0 = tid * E;
      double run = 0.0;
      for (int u = 0; u < E; ++u)
        if (i0 + u < Hd) run += (double)lt[i0 + u];
      double incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      double base = incl - run;
      if (T > 32) {
        __syncthreads();
        if (lane == 31) red[warp] = incl;
        __syncthreads();
        for (int k = 0; k < warp; ++k) base += red[k];
      }
      for (int u = 0; u < E && i0 + u < Hd; ++u) {
        pre[i0 + u] = base;
        base += (double)lt[i0 + u];
      }
      __syncthreads();
    }
    auto d_of = [&](int q) {
      const int k = sites[q];
      return q < sH ? 0.5 * (nb[(size_t)q * B + b] - (tot - pre[k])) + corr : 0.5 * (double)ft[k] + corr;
    };
    double mx = 0.0;  // (the reference's running maximum starts at 0)
    for (int q = tid; q < S; q += T) mx = fmax(mx, d_of(q));
    mx = block_max<T>(mx, red);
    const double shift = mx > 50.0 ? mx : 0.0;
    v = 0.0;
    for (int q = tid; q < S; q += T) v -= alpha_s[q] * exp(d_of(q) - shift);
    acc = block_sum<T>(v, red) * exp(shift);
  }
  if (tid == 0) {
    const double l = diag + acc;
    local[b] = l;
    if (!isfinite(l)) atomicOr(flag, 2u);  // (bit 1: non-finite local energy; bit 0: logit overflow)
  }
}

// ===========================================================================
// Host side
// ===========================================================================
struct SpecState {
  int n = 0, S = 0, sH = 0;
  int64_t np = 0, per_chunk = 1;
  int chunks = 1;
  bool dense = false;  // pairs are the complete row-major upper triangle
  double* alpha_s = nullptr;  // [S] alpha of the sites (alpha > 0, ascending)
  int32_t* sites = nullptr;   // [S]
  int32_t* site_of = nullptr; // [n] site index or -1
  double* beta = nullptr;     // [n]
  int32_t *pi = nullptr, *pj = nullptr;
  double* pv = nullptr;
  // batch scratch
  int cap_B = 0;
  float *Z1 = nullptr, *lterm = nullptr, *fterm = nullptr;
  double *lpf = nullptr, *dpart = nullptr, *nb = nullptr, *local = nullptr, *cached = nullptr;
  uint32_t* Tg = nullptr;  // bit-sliced spins of the sample groups (diagonal kernel)
  int cap_R = 0, cap_parts = 0;
  __half *Nh = nullptr, *Nl = nullptr;
  double* nbpart = nullptr;
  std::vector<double> alpha_host, beta_host;
  std::vector<int32_t> pi_host, pj_host;
  std::vector<double> pv_host;
};

static void validate_spec(int n, const double* alpha, const double* beta, const int32_t* pi, const int32_t* pj,
                          int64_t np) {  // HamiltonianSpec::validate (hamiltonian.cpp:36-54)
  if (np < 0) throw InvalidArgument("num_pairs must be >= 0");
  for (int i = 0; i < n; ++i)
    if (!(alpha[i] >= 0.0)) throw InvalidArgument("alpha must be non-negative");
  (void)beta;
  std::vector<uint64_t> keys((size_t)np);
  for (int64_t t = 0; t < np; ++t) {
    if (pi[t] < 0 || pj[t] >= n || pi[t] >= pj[t])
      throw InvalidArgument("pair indices must satisfy 0 <= i < j < n");
    keys[t] = ((uint64_t)(uint32_t)pi[t] << 32) | (uint32_t)pj[t];
  }
  std::vector<uint64_t> sorted = keys;
  std::sort(sorted.begin(), sorted.end());
  for (size_t t = 1; t < sorted.size(); ++t)
    if (sorted[t] == sorted[t - 1])
      throw InvalidArgument("duplicate pair (" + std::to_string((sorted[t] >> 32) + 1) + "," +
                            std::to_string((sorted[t] & 0xffffffffu) + 1) + ")");
}

void spec_free(Handle* H) {
  SpecState* s = H->spec;
  if (!s) return;
  sfree(s->alpha_s);
  sfree(s->sites);
  sfree(s->site_of);
  sfree(s->beta);
  sfree(s->pi);
  sfree(s->pj);
  sfree(s->pv);
  sfree(s->Z1);
  sfree(s->lterm);
  sfree(s->fterm);
  sfree(s->lpf);
  sfree(s->dpart);
  sfree(s->Tg);
  sfree(s->nb);
  sfree(s->local);
  sfree(s->cached);
  sfree(s->Nh);
  sfree(s->Nl);
  sfree(s->nbpart);
  delete s;
  H->spec = nullptr;
}

void spec_set(Handle* H, const double* alpha, const double* beta, const int32_t* pi, const int32_t* pj,
              const double* pv, int64_t np) {
  const int n = H->L.n;
  if (!alpha || !beta || (np > 0 && (!pi || !pj || !pv))) throw InvalidArgument("null spec array");
  validate_spec(n, alpha, beta, pi, pj, np);
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  spec_free(H);
  H->invalidate_graph();
  SpecState* s = new SpecState();
  H->spec = s;
  s->n = n;
  s->np = np;
  std::vector<int32_t> sites, site_of(n, -1);
  std::vector<double> as;
  for (int i = 0; i < n; ++i)
    if (alpha[i] > 0.0) {
      site_of[i] = (int32_t)sites.size();
      sites.push_back(i);
      as.push_back(alpha[i]);
    }
  s->S = (int)sites.size();
  s->sH = 0;
  while (s->sH < s->S && sites[s->sH] < H->L.Hd) ++s->sH;
  s->alpha_host.assign(alpha, alpha + n);
  s->beta_host.assign(beta, beta + n);
  s->pi_host.assign(pi, pi + np);
  s->pj_host.assign(pj, pj + np);
  s->pv_host.assign(pv, pv + np);
  auto up = [&](auto** d, const auto* src, size_t cnt) {
    salloc(d, std::max<size_t>(cnt, 1));
    if (cnt) VQMC_CUDA(cudaMemcpy(*d, src, cnt * sizeof(**d), cudaMemcpyHostToDevice));
  };
  up(&s->alpha_s, as.data(), as.size());
  up(&s->sites, sites.data(), sites.size());
  up(&s->site_of, site_of.data(), site_of.size());
  up(&s->beta, beta, (size_t)n);
  up(&s->pi, pi, (size_t)np);
  up(&s->pj, pj, (size_t)np);
  up(&s->pv, pv, (size_t)np);
  // complete row-major pair list (random_tim): the diagonal kernel reads only the values
  s->dense = n >= 2 && np == (int64_t)n * (n - 1) / 2;
  for (int64_t t = 0, i = 0, j = 1; s->dense && t < np; ++t) {
    if (pi[t] != i || pj[t] != j) s->dense = false;
    if (++j == n) {
      ++i;
      j = i + 1;
    }
  }
  if (s->dense) {  // chunks of row pairs (n / 2 tasks of n - 1 pairs): ~one task per warp, <= 1184 chunks
    const int64_t tasks = std::max(1, n / 2);
    s->per_chunk = std::max<int64_t>(8, (tasks + 1183) / 1184);
    s->chunks = (int)((tasks + s->per_chunk - 1) / s->per_chunk);
  } else {  // chunks of >= 8192 pairs, at most 256
    s->chunks = (int)std::min<int64_t>(256, std::max<int64_t>(1, (np + 8191) / 8192));
    s->per_chunk = std::max<int64_t>(1, (np + s->chunks - 1) / s->chunks);
  }
}

static void spec_ensure(Handle* H, int B) {
  SpecState* s = H->spec;
  const Layout& L = H->L;
  if (B > s->cap_B) {
    salloc(&s->dpart, (size_t)s->chunks * B);
    salloc(&s->Tg, (size_t)B * L.n);  // (groups of >= 1 sample: at most B groups)
    salloc(&s->local, (size_t)B);
    salloc(&s->cached, (size_t)B);
    salloc(&s->lpf, (size_t)B);
    if (s->S > 0) {
      salloc(&s->Z1, (size_t)B * L.h);
      salloc(&s->lterm, (size_t)B * L.n);
      salloc(&s->fterm, (size_t)B * L.n);
      salloc(&s->nb, (size_t)std::max(1, s->sH) * B);
    }
    s->cap_B = B;
  }
  if (s->sH > 0) {
    // neighbour rows per GEMM launch: whole samples' site sets, up to ~256 MB of operand pairs
    const int64_t budget = (int64_t)(256 << 20) / (4 * (int64_t)H->hp18);
    const int64_t want = std::min<int64_t>((int64_t)B * s->sH, std::max<int64_t>(s->sH, budget));
    const int parts = 3 * ((L.n + kTailBN - 1) / kTailBN) + 3;
    if (want > s->cap_R || parts > s->cap_parts) {
      const int R = (int)std::max<int64_t>(want, s->cap_R);
      salloc(&s->Nh, (size_t)R * H->hp18 + 128);
      salloc(&s->Nl, (size_t)R * H->hp18 + 128);
      salloc(&s->nbpart, (size_t)parts * R);
      s->cap_R = R;
      s->cap_parts = parts;
    }
  }
}

// local_energy_batch (estimator.hpp:43-90) of the configurations in H->X with the cached log psi
// in d_cached (device, [B]; nullptr: the model's own log psi of the configurations); local
// energies into d_local (device).  A non-finite local energy sets bit 1 of the handle's sticky
// flag (the step's Adam then skips the update and the host raises NumericError).
void launch_spec_local(Handle* H, int B, const double* d_cached, double* d_local) {
  SpecState* s = H->spec;
  if (!s) throw InvalidArgument("no Hamiltonian spec set on this handle (vqmc_gpu_set_spec)");
  spec_ensure(H, B);
  const Layout& L = H->L;
  {
    KScope ks(H, "spec_diag");
    // samples per CTA: 32, or fewer for small batches (more CTAs over the pair chunks)
    const int G = B >= 32 ? 32 : B >= 16 ? 16 : B >= 8 ? 8 : B >= 4 ? 4 : B >= 2 ? 2 : 1;
    const int groups = (B + G - 1) / G;
    spec_slice_kernel<<<dim3((L.W + 7) / 8, groups), 256, 0, H->stream>>>(B, L.n, L.W, G, H->X, s->Tg);
    SPEC_LAUNCH_CHECK();
    H->launches++;
    const size_t smem = (size_t)L.n * sizeof(uint32_t);
    const dim3 grid(groups, s->chunks);
    auto go = [&](auto kern) {
      ensure_smem_attr((const void*)kern, smem);
      kern<<<grid, 256, smem, H->stream>>>(B, L.n, s->Tg, s->beta, s->dense ? 1 : 0, s->np, s->per_chunk, s->pi,
                                           s->pj, s->pv, s->dpart);
    };
    switch (G) {
      case 32: go(spec_diag_kernel<32>); break;
      case 16: go(spec_diag_kernel<16>); break;
      case 8: go(spec_diag_kernel<8>); break;
      case 4: go(spec_diag_kernel<4>); break;
      case 2: go(spec_diag_kernel<2>); break;
      default: go(spec_diag_kernel<1>); break;
    }
    SPEC_LAUNCH_CHECK();
    H->launches++;
  }
  if (s->S > 0) {
    forward_plain(H, B, nullptr, s->lterm, s->fterm, s->Z1, s->lpf);
    if (!d_cached) d_cached = s->lpf;
    if (s->sH > 0) {
      const int Bc = std::max(1, std::min(B, s->cap_R / s->sH));
      for (int b0 = 0; b0 < B; b0 += Bc) {
        const int bc = std::min(Bc, B - b0), rows = bc * s->sH;
        {
          KScope ks(H, "tim_nbr_build");
          const int grid = (int)std::min<int64_t>(((int64_t)rows + 8 * kNbrR - 1) / (8 * kNbrR), 148 * 8);
          nbr_build_kernel<<<grid, 256, 0, H->stream>>>(rows, bc, b0, L.h, H->hp18, L.W, s->sites, H->X, s->Z1,
                                                         H->P + L.off_w1t, s->Nh, s->Nl);
          SPEC_LAUNCH_CHECK();
          H->launches++;
        }
        const int parts = launch_nbr_umma(H, rows, bc, b0, s->sites, s->Nh, s->Nl, s->nbpart);
        H->launches++;
        {
          KScope ks(H, "tim_nbr_reduce");
          nbr_reduce_kernel<<<(rows + 255) / 256, 256, 0, H->stream>>>(rows, bc, b0, B, parts, s->nbpart, s->nb);
          SPEC_LAUNCH_CHECK();
          H->launches++;
        }
      }
    }
  }
  {
    KScope ks(H, "spec_local");
    const double* dc = d_cached ? d_cached : s->lpf;
    if (L.n <= 256 && s->chunks <= 64)
      spec_local_kernel<32><<<B, 32, 0, H->stream>>>(B, L.n, L.Hd, s->S, s->sH, s->sites, s->alpha_s, s->chunks,
                                                     s->dpart, s->lterm, s->fterm, s->nb, s->lpf, dc, d_local,
                                                     H->d_flag);
    else
      spec_local_kernel<256><<<B, 256, 0, H->stream>>>(B, L.n, L.Hd, s->S, s->sH, s->sites, s->alpha_s, s->chunks,
                                                       s->dpart, s->lterm, s->fterm, s->nb, s->lpf, dc, d_local,
                                                       H->d_flag);
    SPEC_LAUNCH_CHECK();
    H->launches++;
  }
}

double* spec_local_buffer(Handle* H, int B) {
  spec_ensure(H, B);
  return H->spec->local;
}
double* spec_cached_buffer(Handle* H, int B) {
  spec_ensure(H, B);
  return H->spec->cached;
}

}  // namespace vqmc_b200
