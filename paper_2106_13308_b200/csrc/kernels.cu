// VQMC step kernels for sm_100a: energy, statistics / REINFORCE weights, the backward's elementwise
// passes and Adam (the GEMMs are tcgen05 kernels in gemm.cu, the head sampler is head.cu, the plain
// forward of given configurations and general-spec energies are spec.cu).
//
// Reference path (arxiv/paper_2106_13308, /root/reference/proj):
//   auto_sample            proj/src/sampler.cpp:35-59      -> head_v2_kernel (head.cu) + tail GEMM (gemm.cu)
//   made_forward           proj/src/models.cpp:51-62       -> z1_given_kernel + z2_given_umma (spec.cu, gemm.cu)
//   local_energy_batch     proj/include/vqmc/estimator.hpp:43-57 -> energy_kernel
//   energy_and_variance +
//   gradient_from_locals   estimator.hpp:94-119            -> stats_weights_kernel
//   weighted_grad_log_psi  proj/src/models.cpp:175-198     -> dg1/gw2 (gemm.cu), dz1/gw1 kernels
//   adam_step              proj/src/optimizer.cpp:21-35    -> adam_kernel
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "device_common.cuh"
#include "adam.cuh"
#include "internal.cuh"
#include "ptx.cuh"

namespace vqmc_b200 {

// log_psi = (head + sum of tail partials) / 2, one warp per sample (fixed reduction order).
__global__ void finalize_logpsi_kernel(int B, int tiles, const double* __restrict__ lp_head,
                                       const double* __restrict__ lp_part,
                                       double* __restrict__ log_psi) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  double s = 0.0;
  for (int t = lane; t < tiles; t += 32) s += lp_part[(size_t)t * B + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) log_psi[b] = 0.5 * (lp_head[b] + s);  // sampler.cpp:56 / models.cpp:122-124
}

// ===========================================================================
// Max-Cut local energy over bit-packed samples (estimator.hpp:53-57,
// hamiltonian.cpp:61-69 with beta_ij = -1/4): cut_b = sum_E x_i XOR x_j,
// l_b = (|E| - 2 cut_b) / 4, exact.  S samples per CTA share every edge load.
// ===========================================================================
template <int S>
__global__ void __launch_bounds__(256) energy_kernel(int B, int W, int64_t nE,
                                                     const int2* __restrict__ edges,
                                                     const uint32_t* __restrict__ X,
                                                     int32_t* __restrict__ cut,
                                                     double* __restrict__ local) {
  extern __shared__ uint32_t sbits[];  // [S][W]
  const int b0 = blockIdx.x * S;
  for (int t = threadIdx.x; t < S * W; t += blockDim.x) {
    const int s = t / W, w = t % W;
    sbits[t] = (b0 + s < B) ? X[(size_t)(b0 + s) * W + w] : 0u;
  }
  __syncthreads();
  int cnt[S];
#pragma unroll
  for (int s = 0; s < S; ++s) cnt[s] = 0;
  for (int64_t e = threadIdx.x; e < nE; e += blockDim.x) {
    const int2 ed = edges[e];
    const int wi = ed.x >> 5, si = ed.x & 31, wj = ed.y >> 5, sj = ed.y & 31;
#pragma unroll
    for (int s = 0; s < S; ++s)
      cnt[s] += ((sbits[s * W + wi] >> si) ^ (sbits[s * W + wj] >> sj)) & 1u;
  }
  __shared__ int red[S][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    int v = cnt[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) red[s][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < S) {
    const int s = threadIdx.x;
    int v = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[s][w];
    if (b0 + s < B) {
      cut[b0 + s] = v;
      local[b0 + s] = 0.25 * ((double)nE - 2.0 * (double)v);
    }
  }
}

// ===========================================================================
// Max-Cut cuts, bit-sliced over samples (the default path; maxcut_cut_kernel below).
// ===========================================================================
// 32x32 bit transpose across a warp with one funnel rotation + one LOP3 per stage (the bits
// that wrap around are masked away): lane r holds row r; returns column `lane`.
__device__ __forceinline__ uint32_t transpose32_rot(uint32_t v, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int j = 16 >> t;
    const bool hi = (lane & j) != 0;
    const uint32_t keep = hi ? ~masks[t] : masks[t];  // this lane's own bits
    const uint32_t o = __shfl_xor_sync(kFull, v, j);
    const uint32_t r = __funnelshift_l(o, o, hi ? 32 - j : j);  // rotl(o, j) or rotr(o, j)
    v = (v & keep) | (r & ~keep);
  }
  return v;
}

// 32 x 32 bit transpose of v[r] (row r, bit c = M[r][c]) in registers: afterwards v[c] bit r =
// M[r][c].  Five delta-swap stages of 16 register pairs; the 16- and 8-bit stages are byte
// permutes (one PRMT per output word).
__device__ __forceinline__ void transpose32_regs(uint32_t (&v)[32]) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t a = v[r], b = v[r + 16];
    v[r] = __byte_perm(a, b, 0x5410);
    v[r + 16] = __byte_perm(a, b, 0x7632);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    if (r & 8) continue;
    const uint32_t a = v[r], b = v[r + 8];
    v[r] = __byte_perm(a, b, 0x6240);
    v[r + 8] = __byte_perm(a, b, 0x7351);
  }
#pragma unroll
  for (int t = 2; t < 5; ++t) {
    const int j = 16 >> t;
    const uint32_t m = masks[t];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      if (r & j) continue;
      // swap the high-j bits of v[r] (columns >= j within each 2j block) with the low bits of v[r + j]
      const uint32_t x = ((v[r] >> j) ^ v[r + j]) & m;
      v[r + j] ^= x;
      v[r] ^= x << j;
    }
  }
}

// Carry-save adder: (hi, lo) = a + b + c bitwise (two LOP3s).
__device__ __forceinline__ void csa(uint32_t& hi, uint32_t& lo, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  hi = (a & b) | (u & c);
  lo = u ^ c;
}

// Max-Cut cut counts over bit-sliced samples (local_energy_batch's diagonal branch,
// estimator.hpp:53-57; diagonal_energy hamiltonian.cpp:61-69; cut_value :121-124).
//
// Edges arrive bank-ordered and packed (upload_edges): entry e = 4u | 4v << 16 (byte offsets),
// in batches of 32 with pairwise-distinct u mod 32 and pairwise-distinct v mod 32, interleaved so
// that a warp's 16-byte quad loads (lane l: entry l of four batches) hand each of its four lookup
// rounds T[u], T[v] one batch: conflict-free, 1/4 load instruction per entry.  A CTA keeps its edge chunk
// resident in shared memory and walks sample groups g = blockIdx.y, += gridDim.y (32 samples per
// group): the group's packed rows arrive by one bulk copy into T, every thread reads one word
// column into registers, and after a barrier writes it back transposed (in place: T[swz(node)] =
// that node's spin in all 32 samples).  One XOR per edge gives the 32-sample cut mask, and
// Harley-Seal carry-save counters (ones, twos, fours, eights + a ripple counter of sixteens) sum
// them at ~2 logic ops per edge (<= 63 entries per thread: 6 planes).  The planes are transposed back (lane s <- sample s)
// and popcounted.  Shared memory stays <= ~110 KB so two CTAs share an SM (one's copy and
// transpose overlap the other's edge pass).  Per-chunk counts are exact integers, summed in a
// fixed order by the statistics kernel.   Shared memory: T [32 W] | zero [32] | E [chunk entries].
constexpr int kCutThreads = 512;
__global__ void __launch_bounds__(kCutThreads, 2) maxcut_cut_kernel(int B, int W, int64_t nEp, int64_t per_chunk,
                                                                    const uint32_t* __restrict__ edges,
                                                                    const uint32_t* __restrict__ X,
                                                                    int32_t* __restrict__ cpart) {
  extern __shared__ __align__(16) uint32_t smem_words[];
  const int TW = 32 * W + 32;  // transposed spins + 32 zero words (the padding entries' targets)
  uint32_t* T = smem_words;
  uint32_t* E = smem_words + TW;
  __shared__ int scnt[32];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kCutThreads / 32;
  const int groups = (B + 31) / 32;
  const int64_t e0 = (int64_t)blockIdx.x * per_chunk, e1 = min(nEp, e0 + per_chunk);
  const int ne = (int)(e1 - e0);  // multiple of 128
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) ptx::mbar_init(&bar[k], 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) {
    scnt[tid] = 0;
    T[32 * W + tid] = 0u;
  }
  __syncthreads();
  if (tid == 0 && ne > 0) {
    ptx::mbar_expect_tx(&bar[1], 4u * (uint32_t)ne);
    ptx::bulk_g2s(E, edges + e0, 4u * (uint32_t)ne, &bar[1]);
  }
  bool edges_ready = false;
  int it = 0;
  for (int g = blockIdx.y; g < groups; g += gridDim.y, ++it) {
    const int s0 = 32 * g, rows = min(32, B - s0);
    if (rows == 32) {
      if (tid == 0) {
        ptx::fence_proxy_async_smem();  // (the previous group's generic transposed writes to T)
        ptx::mbar_expect_tx(&bar[0], 128u * (uint32_t)W);
        ptx::bulk_g2s(T, X + (size_t)s0 * W, 128u * (uint32_t)W, &bar[0]);
      }
      ptx::mbar_wait(&bar[0], it & 1);
    } else {  // ragged last group
      for (int t = tid; t < 32 * W; t += kCutThreads) T[t] = t < rows * W ? X[(size_t)s0 * W + t] : 0u;
      __syncthreads();
    }
    // in-place transpose, one 32 x 32 bit block per thread in registers (thread w takes word column w:
    // 32 conflict-free loads, 5 delta-swap stages, 8 16-byte stores).  T is swizzled so that those
    // stores are conflict-free: node i lives at word swz(i) = i ^ (((i >> 5) & 7) << 2); the edge
    // entries carry swizzled indices (upload_edges).
    uint32_t v[32];
    const int w = tid;
    if (w < W) {
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = T[r * W + w];
    }
    __syncthreads();
    if (w < W) {
      transpose32_regs(v);
#pragma unroll
      for (int k = 0; k < 8; ++k)  // nodes 32 w + 4 k .. + 3, one 16-byte store
        *reinterpret_cast<uint4*>(T + 32 * w + 4 * (k ^ (w & 7))) = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    }
    if (!edges_ready) {
      if (ne > 0) ptx::mbar_wait(&bar[1], 0);
      edges_ready = true;
    }
    __syncthreads();
    // 16 entries per thread per pass (quads tid + 512 k: one 16-byte load each), Harley-Seal
    // carry-save counting.  Entries are byte offsets into T; a quad past the chunk reads as zeros
    // (both lookups hit word 0: XOR = 0).
    const uint4* E4 = reinterpret_cast<const uint4*>(E);
    const char* Tb = reinterpret_cast<const char*>(T);
    auto cutmask = [&](uint32_t p) {  // samples in which this edge is cut
      return *reinterpret_cast<const uint32_t*>(Tb + (p & 0xFFFFu)) ^ *reinterpret_cast<const uint32_t*>(Tb + (p >> 16));
    };
    const int nq = ne >> 2;
    uint32_t ones = 0, twos = 0, fours = 0, eights = 0, c16 = 0, c32 = 0;  // <= 63 per thread (launcher)
    for (int qb = 0; qb < nq; qb += 4 * kCutThreads) {
      uint32_t c[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c[4 * k] = c[4 * k + 1] = c[4 * k + 2] = c[4 * k + 3] = 0u;
        if (qb + k * kCutThreads < nq) {  // (CTA-uniform: the last pass is usually partial)
          const int q = qb + k * kCutThreads + tid;
          const uint4 p = q < nq ? E4[q] : make_uint4(0u, 0u, 0u, 0u);
          c[4 * k] = cutmask(p.x);
          c[4 * k + 1] = cutmask(p.y);
          c[4 * k + 2] = cutmask(p.z);
          c[4 * k + 3] = cutmask(p.w);
        }
      }
      uint32_t tA, tB, fA, fB, eA, eB, sx;
      csa(tA, ones, ones, c[0], c[1]);
      csa(tB, ones, ones, c[2], c[3]);
      csa(fA, twos, twos, tA, tB);
      csa(tA, ones, ones, c[4], c[5]);
      csa(tB, ones, ones, c[6], c[7]);
      csa(fB, twos, twos, tA, tB);
      csa(eA, fours, fours, fA, fB);
      csa(tA, ones, ones, c[8], c[9]);
      csa(tB, ones, ones, c[10], c[11]);
      csa(fA, twos, twos, tA, tB);
      csa(tA, ones, ones, c[12], c[13]);
      csa(tB, ones, ones, c[14], c[15]);
      csa(fB, twos, twos, tA, tB);
      csa(eB, fours, fours, fA, fB);
      csa(sx, eights, eights, eA, eB);
      c32 ^= c16 & sx;  // ripple counter of sixteens (two planes)
      c16 ^= sx;
    }
    // per-sample counts: transpose each plane (lane s <- sample s), popc, weight
    const int cnt = __popc(transpose32_rot(ones, lane)) + (__popc(transpose32_rot(twos, lane)) << 1) +
                    (__popc(transpose32_rot(fours, lane)) << 2) + (__popc(transpose32_rot(eights, lane)) << 3) +
                    (__popc(transpose32_rot(c16, lane)) << 4) + (__popc(transpose32_rot(c32, lane)) << 5);
    atomicAdd(&scnt[lane], cnt);
    __syncthreads();  // counts complete; every edge lookup into T done (the next group may overwrite it)
    if (tid < 32) {
      if (tid < rows) cpart[(size_t)blockIdx.x * B + s0 + tid] = scnt[tid];
      scnt[tid] = 0;
    }
    // (the next iteration's barriers order these resets before its atomics)
  }
}

// ===========================================================================
// In-batch statistics and REINFORCE weights, fused with the wG1 operand of the gW2 GEMM.
// Every CTA computes, over the worker segments of `seg` rows in a fixed order: cut_b (the sum
// of the energy kernel's per-chunk partial counts), l_b = (|E| - 2 cut_b) / 4 (exact), the
// segment mean (estimator.hpp:115, the per-worker baseline) and w_b = 2 (l_b - mean) / seg
// (estimator.hpp:116-117), stored normalised as w' = w / wscale with wscale the power of two
// >= max |w| (exact), so the fp16-pair operand w' G1 cannot overflow (the backward epilogues
// multiply by wscale).  CTA 0 also writes cut, l, w', wscale and the segments' exact integer
// cut sums (pooled statistics are formed from these on the host, trainer.cpp:246-248).  Then
// the grid writes wG1 = fp16 pair of [w' G1 | w'] (skipped when G1 is null).
// ===========================================================================
__global__ void __launch_bounds__(1024) stats_weights_kernel(int segs, int seg, int chunks, int64_t nE,
                                                             const int32_t* __restrict__ cpart,
                                                             int32_t* __restrict__ cut, double* __restrict__ local,
                                                             float* __restrict__ w, float* __restrict__ wscale,
                                                             int64_t* __restrict__ istat, int h, int ld,
                                                             const float* __restrict__ G1, __half* __restrict__ wgh,
                                                             __half* __restrict__ wgl, float* __restrict__ rstat,
                                                             int nranks, int rank, const double* __restrict__ lin,
                                                             double* __restrict__ lstat) {
  extern __shared__ float sw[];  // [B] weights of the whole batch (per CTA)
  __shared__ double sd[32], sd2[32];
  __shared__ long long si[32], sq[32];
  __shared__ int sm[32];
  __shared__ float smax[32];
  __shared__ double smean;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int B = segs * seg;
  const bool lead = blockIdx.x == 0;
  ptx::pdl_trigger();
  ptx::pdl_wait();
  // the wG1 part's G1 values do not depend on the statistics: load them first (<= 4 per thread)
  constexpr int kPre = 4;
  const int64_t wtotal = G1 ? (int64_t)B * ld : 0;
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  float g1pre[kPre];
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + tid + u * wstride;
    g1pre[u] = 0.f;
    if (t < wtotal) {
      const int b = (int)(t / ld), k = (int)(t % ld);
      if (k < h) g1pre[u] = G1[(size_t)b * h + k];
    }
  }
  float wmax = 0.f;
  const bool one = seg <= (int)blockDim.x;  // one sample per thread and segment: l_b stays in a register
  double lb_keep = 0.0;
  for (int sgi = 0; sgi < segs; ++sgi) {
    const int base = sgi * seg;
    double s = 0.0, s2 = 0.0;
    long long cs = 0, cq = 0;
    int cm = 0;
    for (int b = tid; b < seg; b += blockDim.x) {
      int c = 0;
      double lb;
      if (lin) {  // general spec: fp64 local energies (estimator.hpp:43-90)
        lb = lin[base + b];
        s2 += lb * lb;
      } else {
#pragma unroll 4
        for (int k = 0; k < chunks; ++k) c += cpart[(size_t)k * B + base + b];
        lb = 0.25 * ((double)nE - 2.0 * (double)c);  // l_b = (|E| - 2 cut_b) / 4, exact
      }
      if (lead) {
        if (!lin) cut[base + b] = c;
        local[base + b] = lb;
      }
      s += lb;
      cs += c;
      cq += (long long)c * c;
      cm = max(cm, c);
      lb_keep = lb;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(kFull, s, o);
      s2 += __shfl_xor_sync(kFull, s2, o);
      cs += __shfl_xor_sync(kFull, cs, o);
      cq += __shfl_xor_sync(kFull, cq, o);
      cm = max(cm, __shfl_xor_sync(kFull, cm, o));
    }
    if (lane == 0) { sd[warp] = s; sd2[warp] = s2; si[warp] = cs; sq[warp] = cq; sm[warp] = cm; }
    __syncthreads();
    if (warp == 0) {  // (Max-Cut: the l_b are multiples of 1/4, so every fp64 sum here is exact)
      double t = lane < nw ? sd[lane] : 0.0, t2 = lane < nw ? sd2[lane] : 0.0;
      long long a = lane < nw ? si[lane] : 0, q = lane < nw ? sq[lane] : 0;
      int mx = lane < nw ? sm[lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(kFull, t, o);
        t2 += __shfl_xor_sync(kFull, t2, o);
        a += __shfl_xor_sync(kFull, a, o);
        q += __shfl_xor_sync(kFull, q, o);
        mx = max(mx, __shfl_xor_sync(kFull, mx, o));
      }
      if (lane == 0) smean = t / (double)seg;
      if (lead && lane == 0) {
        istat[3 * sgi + 0] = a;
        istat[3 * sgi + 1] = q;
        istat[3 * sgi + 2] = mx;
        if (lstat) {  // [0, 2): the rank's sums of l and l^2 (all-reduced across ranks); [2 + 2 s ...) per segment
          lstat[2 + 2 * sgi] = t;
          lstat[3 + 2 * sgi] = t2;
          lstat[0] = (sgi ? lstat[0] : 0.0) + t;
          lstat[1] = (sgi ? lstat[1] : 0.0) + t2;
        }
      }
    }
    __syncthreads();
    const double mean = smean;
    for (int b = tid; b < seg; b += blockDim.x) {
      double lb;
      if (one) {
        lb = lb_keep;
      } else if (lin) {
        lb = lin[base + b];
      } else {
        int c = 0;
#pragma unroll 4
        for (int k = 0; k < chunks; ++k) c += cpart[(size_t)k * B + base + b];
        lb = 0.25 * ((double)nE - 2.0 * (double)c);
      }
      const float wb = (float)(2.0 * (lb - mean) / (double)seg);
      sw[base + b] = wb;
      wmax = fmaxf(wmax, fabsf(wb));
    }
    __syncthreads();  // smean / partials are reused by the next segment
  }
  if (lead && tid == 0 && rstat) {
    // this rank's exact cut statistics as 16-bit fp32 limbs riding in the gradient all-reduce (sum):
    // [0, 3) cut sum, [3, 7) cut^2 sum, [7 + 2 r, 9 + 2 r) rank r's best cut (zero in other ranks'
    // slots).  Every limb sum over <= 256 ranks is < 2^24: exact in fp32 (dp.stat_limbs_decode).
    unsigned long long a = 0, q = 0, mx = 0;
    for (int sgi = 0; sgi < segs; ++sgi) {
      a += (unsigned long long)istat[3 * sgi];
      q += (unsigned long long)istat[3 * sgi + 1];
      mx = max(mx, (unsigned long long)istat[3 * sgi + 2]);
    }
    for (int k = 0; k < 3; ++k) rstat[k] = (float)((a >> (16 * k)) & 0xFFFFull);
    for (int k = 0; k < 4; ++k) rstat[3 + k] = (float)((q >> (16 * k)) & 0xFFFFull);
    for (int r = 0; r < nranks; ++r)
      for (int k = 0; k < 2; ++k) rstat[7 + 2 * r + k] = r == rank ? (float)((mx >> (16 * k)) & 0xFFFFull) : 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(kFull, wmax, o));
  if (lane == 0) smax[warp] = wmax;
  __syncthreads();
  float m = lane < nw ? smax[lane] : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  // wscale = 2^e >= m (1 when every weight is 0); w' = w * 2^-e exactly
  int e = 0;
  if (m > 0.f) frexpf(m, &e);  // m = f 2^e, f in [0.5, 1)
  const float sc = ldexpf(1.f, e), inv = ldexpf(1.f, -e);
  for (int b = tid; b < B; b += blockDim.x) {
    const float wn = sw[b] * inv;
    sw[b] = wn;
    if (lead) w[b] = wn;
  }
  if (lead && tid == 0) *wscale = sc;
  if (G1 == nullptr) return;
  __syncthreads();
  // wG1[b][k] = w'_b G1[b][k] (k < h), w'_b (k == h), 0 beyond; fp16 pair (gW2 B operand)
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + tid + u * wstride;
    if (t < wtotal) {
      const int b = (int)(t / ld), k = (int)(t % ld);
      const float x = k < h ? sw[b] * g1pre[u] : (k == h ? sw[b] : 0.f);
      ptx::split_f16(x, wgh[t], wgl[t]);
    }
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + tid + kPre * wstride; t < wtotal; t += wstride) {
    const int b = (int)(t / ld), k = (int)(t % ld);
    const float x = k < h ? sw[b] * G1[(size_t)b * h + k] : (k == h ? sw[b] : 0.f);
    ptx::split_f16(x, wgh[t], wgl[t]);
  }
}

// ===========================================================================
// Backward (models.cpp:175-198), with the REINFORCE row weights folded in:
//   E    = D . W2m            (split-K over n)        dg1 = w (.) E
//   dz1  = w_b E_bk [z1_bk > 0]                       ([G1 > 0] == [z1 > 0])
//   gW2  = (D^T (w (.) G1)) (.) M2,  gb2 = D^T w      (one GEMM, N = h + 1)
//   gW1T = (X^T dz1) (.) M1^T,       gb1 = 1^T dz1    (one GEMM, M = Hd + 1)
// ===========================================================================
namespace bwcfg {
constexpr int BK = 16, TM = 8, TN = 8;
constexpr int QM = 64, QN = 64;  // gW1
}  // namespace bwcfg

// dz1' = w'_b E_bk [z1_bk > 0] as a bf16 pair (gW1 operand; gw1_finalize multiplies by wscale).
__global__ void dz1_kernel(int B, int h, int hp, int splits, const float* __restrict__ Epart,
                           const float* __restrict__ w, const float* __restrict__ G1,
                           __nv_bfloat16* __restrict__ dz1bh, __nv_bfloat16* __restrict__ dz1bl) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  // 4 consecutive k per thread (h % 4 == 0: 16-byte loads of every partial; else scalar)
  const size_t total = (size_t)B * h;
  const size_t t4 = 4 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (t4 >= total) return;
  if ((h & 3) == 0) {
    const int b = (int)(t4 / h), k = (int)(t4 % h);
    const float4 g = *reinterpret_cast<const float4*>(G1 + t4);
    const float wb = w[b];
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int z = 0; z < splits; ++z) {  // (unrolled: the partials' loads in flight together, same order of adds)
      const float4 p = *reinterpret_cast<const float4*>(Epart + (size_t)z * total + t4);
      s.x += p.x;
      s.y += p.y;
      s.z += p.z;
      s.w += p.w;
    }
    const float d[4] = {g.x > 0.f ? s.x * wb : 0.f, g.y > 0.f ? s.y * wb : 0.f, g.z > 0.f ? s.z * wb : 0.f,
                        g.w > 0.f ? s.w * wb : 0.f};  // relu'(z1) = [z1 > 0] (models.cpp:181)
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ptx::split_bf16(d[u], hi[u], lo[u]);
    *reinterpret_cast<uint2*>(dz1bh + (size_t)b * hp + k) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(dz1bl + (size_t)b * hp + k) = *reinterpret_cast<const uint2*>(lo);
    return;
  }
  for (size_t t = t4; t < t4 + 4 && t < total; ++t) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += Epart[(size_t)z * total + t];
    const int b = (int)(t / h), k = (int)(t % h);
    const float d = G1[t] > 0.f ? s * w[b] : 0.f;
    ptx::split_bf16(d, dz1bh[(size_t)b * hp + k], dz1bl[(size_t)b * hp + k]);
  }
}

// gW1T = (sum of partials) (.) M1^T, gb1 = the ones row (j == Hd).
__global__ void gw1_finalize_kernel(int h, int Hd, int splits, const float* __restrict__ part,
                                    const int32_t* __restrict__ deg, const float* __restrict__ wscale,
                                    float* __restrict__ gW1T, float* __restrict__ gb1) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int total = (Hd + 1) * h;
  const int t4 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);  // 4 consecutive k (h % 4 == 0) or scalar
  if (t4 >= total) return;
  const float sc = *wscale;
  const int n4 = (h & 3) == 0 ? 4 : 1;
  for (int t = t4; t < t4 + 4 && t < total; t += n4) {
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    if (n4 == 4) {
#pragma unroll 4
      for (int z = 0; z < splits; ++z) {
        const float4 p = *reinterpret_cast<const float4*>(part + (size_t)z * total + t);
        s[0] += p.x;
        s[1] += p.y;
        s[2] += p.z;
        s[3] += p.w;
      }
    } else {
      for (int z = 0; z < splits; ++z) s[0] += part[(size_t)z * total + t];
    }
    for (int u = 0; u < n4; ++u) {
      const int j = (t + u) / h, k = (t + u) % h;
      const float v = s[u] * sc;
      if (j < Hd) gW1T[(size_t)j * h + k] = (j + 1 <= deg[k]) ? v : 0.f;  // M1(k, j)
      else gb1[k] = v;
    }
  }
}

// The end of every Adam block: the block's partial of
// ||g||^2 into gpart[block_base + block]; the last of total_blocks blocks (shared done counter)
// sums them in a fixed order, resets the counter and advances the device step counters.
__device__ __forceinline__ void adam_block_finish(double sq, const StepParams* sp, double* __restrict__ gpart,
                                                  int block_base, int total_blocks, unsigned* __restrict__ done,
                                                  double* __restrict__ gnorm2) {
  __shared__ double red[8];
  __shared__ bool last;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(kFull, sq, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    gpart[block_base + blockIdx.x] = s;
    unsigned prev;  // acq_rel: publishes this block's partial, and (last block) acquires everyone's
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done) : "memory");
    last = prev == (unsigned)total_blocks - 1;
  }
  __syncthreads();
  if (!last) return;
  {  // fixed-order final sum by the last block: strided thread sums, then a fixed shuffle tree
    __threadfence();  // (orders the other threads' reads after thread 0's acquire)
    double s = 0.0;
#pragma unroll 4
    for (int i = threadIdx.x; i < total_blocks; i += blockDim.x) s += __ldcg(gpart + i);  // (L2: other blocks' partials)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    *gnorm2 = s;
    *done = 0u;
    // advance the device step counters for the next step (every other block has read them):
    // Philox call + 1, Adam t + 1 and its bias corrections (optimizer.cpp:28-29)
    StepParams* w = const_cast<StepParams*>(sp);
    w->call += 1;
    w->t += 1;
    w->bc1 = w->nbc1;  // (formed for t + 1 by the first Adam block: adam_next_bias)
    w->bc2 = w->nbc2;
    w->ibc1 = w->nibc1;
    w->ibc2 = w->nibc2;
  }
}

// Bias corrections of step t (optimizer.cpp:28-29) and their reciprocals.
__device__ __forceinline__ void adam_bias(float b1, float b2, int64_t t, float& bc1, float& bc2, float& ibc1,
                                          float& ibc2) {
  bc1 = (float)(1.0 - pow((double)b1, (double)t));
  bc2 = (float)(1.0 - pow((double)b2, (double)t));
  ibc1 = 1.f / bc1;
  ibc2 = 1.f / bc2;
}
// Thread 0 of the first Adam block: the next step's bias corrections (two fp64 pows) while the
// other blocks run, so the last block only copies them.
__device__ __forceinline__ void adam_next_bias(const StepParams* sp, int block_base) {
  if (block_base == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    StepParams* w = const_cast<StepParams*>(sp);
    adam_bias(w->b1, w->b2, w->t + 1, w->nbc1, w->nbc2, w->nibc1, w->nibc2);
  }
}

// ===========================================================================
// Adam over the live parameter buffer (optimizer.cpp:21-35), fp32 master
// weights, gradient scaled by 1/L (allreduce_mean's division, trainer.cpp:334).
// Also the squared-norm partials of the reduced gradient (trainer.cpp:253).
// ===========================================================================
// Adam over the live parameter buffer (optimizer.cpp:21-35), fp32 master weights, gradient
// scaled by 1/L (allreduce_mean's division, trainer.cpp:334), fused with everything that
// derives from the updated parameters: the squared norm of the reduced gradient (last-block
// reduction, fixed order; trainer.cpp:253), the fp16 pair of W2 for the GEMMs and the head
// sampler's padded / completion-ordered copies of the head blocks.
// Adam over the element range [lo, hi) of the live buffer.  The training step runs it as up to
// two launches (the [W2 | b2] range right after its gradient and the W1 GEMM's last read of W2,
// concurrently with the rest of the backward; then the [W1T | b1] range): every launch writes
// its per-block ||g||^2 partials at gpart[block_base + block], and the last block of ALL launches
// (a shared counter up to total_blocks) sums them in block order and advances the step counters.
__global__ void __launch_bounds__(256, 4) adam_kernel(int64_t lo, int64_t hi, float scale,
                                                   const StepParams* __restrict__ sp, float* __restrict__ P,
                                                   const float* __restrict__ G, float* __restrict__ M,
                                                   float* __restrict__ V, double* __restrict__ gpart,
                                                   int block_base, int total_blocks, unsigned* __restrict__ done,
                                                   double* __restrict__ gnorm2, AdamOut o) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  AdamHyper hp;
  hp.load(sp);
  adam_next_bias(sp, block_base);
  float sqf = 0.f;  // fp32 partial of ||g||^2 per element group, summed into fp64 per thread
  double sq = 0.0;
  auto upd = [&](float g, float& m, float& v, float& p) {
    g *= scale;
    sqf = fmaf(g, g, sqf);
    hp.update(g, m, v, p);
  };
  // float4 groups inside [lo, hi); scalar heads / tails
  const bool skip = o.flag != nullptr && *(volatile const uint32_t*)o.flag != 0u;  // failed step: no update
  const int64_t q_lo = (lo + 3) / 4, q_hi = skip ? q_lo : hi / 4;
  const int64_t nq = q_hi > q_lo ? q_hi - q_lo : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  G += 4 * q_lo;
  M += 4 * q_lo;
  V += 4 * q_lo;
  P += 4 * q_lo;
  const int64_t t_off = 4 * q_lo;  // element index of the shifted base
  const int64_t w2_bulk0 = (int64_t)o.Hd * o.h, w2_end = o.off_b2 - o.off_w2;  // W2 rows >= Hd
  // one float4 group per thread per iteration, the next group's loads issued before this one's math
  // (software pipelining: the loads stay in flight through the update arithmetic)
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float4 g4, m4, v4, p4;
  if (q < nq) {
    g4 = reinterpret_cast<const float4*>(G)[q];
    m4 = reinterpret_cast<float4*>(M)[q];
    v4 = reinterpret_cast<float4*>(V)[q];
    p4 = reinterpret_cast<float4*>(P)[q];
  }
  for (; q < nq; q += stride) {
    const int64_t qn = q + stride;
    float4 gn, mn, vn, pn;
    if (qn < nq) {
      gn = reinterpret_cast<const float4*>(G)[qn];
      mn = reinterpret_cast<float4*>(M)[qn];
      vn = reinterpret_cast<float4*>(V)[qn];
      pn = reinterpret_cast<float4*>(P)[qn];
    }
    upd(g4.x, m4.x, v4.x, p4.x);
    upd(g4.y, m4.y, v4.y, p4.y);
    upd(g4.z, m4.z, v4.z, p4.z);
    upd(g4.w, m4.w, v4.w, p4.w);
    reinterpret_cast<float4*>(M)[q] = m4;
    reinterpret_cast<float4*>(V)[q] = v4;
    reinterpret_cast<float4*>(P)[q] = p4;
    const int64_t t = t_off + 4 * q;
    const int64_t w = t - o.off_w2;
    if (o.vec_w2 && w >= w2_bulk0 && w < w2_end) {
      // bulk of W2 (rows >= Hd): 4 consecutive entries of one row -> 8-byte stores of both halves
      unsigned i, k;
      w2_row(o, (unsigned)w, i, k);
      uint2 hi, lo;
      ptx::split_f16x2(p4.x, p4.y, hi.x, lo.x);
      ptx::split_f16x2(p4.z, p4.w, hi.y, lo.y);
      *reinterpret_cast<uint2*>(o.W2h + (size_t)i * o.hp18 + k) = hi;
      *reinterpret_cast<uint2*>(o.W2l + (size_t)i * o.hp18 + k) = lo;
    } else {
      adam_side_writes(o, t, p4.x);
      adam_side_writes(o, t + 1, p4.y);
      adam_side_writes(o, t + 2, p4.z);
      adam_side_writes(o, t + 3, p4.w);
    }
    sq += (double)sqf;  // (4 fp32 terms per partial: ||g||^2 keeps ~fp32-grade relative error)
    sqf = 0.f;
    g4 = gn;
    m4 = mn;
    v4 = vn;
    p4 = pn;
  }
  G -= t_off;
  M -= t_off;
  V -= t_off;
  P -= t_off;
  const int64_t e_head = nq > 0 ? 4 * q_lo : hi;  // scalar elements: [lo, 4 q_lo) and [4 q_hi, hi)
  const int64_t n_head = skip ? 0 : e_head - lo, n_tail = nq > 0 ? hi - 4 * q_hi : 0;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n_head + n_tail; x += stride) {
    const int64_t t = x < n_head ? lo + x : 4 * q_hi + (x - n_head);
    float g = G[t], m = M[t], v = V[t], p = P[t];
    upd(g, m, v, p);
    M[t] = m;
    V[t] = v;
    P[t] = p;
    adam_side_writes(o, t, p);
  }
  sq += (double)sqf;
  adam_block_finish(sq, sp, gpart, block_base, total_blocks, done, gnorm2);
}

__global__ void sum_partials_kernel(int cnt, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    *out = t;
  }
}

// ===========================================================================
// Launchers
// ===========================================================================
#define LAUNCH_CHECK() VQMC_CUDA(cudaGetLastError())

void ensure_smem_attr(const void* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  VQMC_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kern, dev}];
  if (have >= bytes) return;
  VQMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
}

void record_event_on(Handle* H, cudaEvent_t ev, cudaStream_t stream) {
  if (H->capturing) VQMC_CUDA(cudaEventRecordWithFlags(ev, stream, cudaEventRecordExternal));
  else VQMC_CUDA(cudaEventRecord(ev, stream));
}
void record_event(Handle* H, cudaEvent_t ev) { record_event_on(H, ev, H->stream); }

KScope::KScope(Handle* h, const char* name, cudaStream_t stream) : H(h), slot(-1), s(stream ? stream : h->stream) {
  if (!H->ktimer || H->kt_count >= Handle::kKtPool) return;
  slot = H->kt_count++;
  H->kt_name[slot] = name;
  record_event_on(H, H->kt_start[slot], s);
}
KScope::~KScope() {
  if (slot >= 0) record_event_on(H, H->kt_end[slot], s);
}

// Derived device copies of the parameters (after set_params): the head sampler's staged
// head blocks and the fp16 pair of W2 (Adam refreshes both itself).
void launch_params_refresh(Handle* H) {
  launch_head_pack(H);
  launch_split_w2(H);
}

void launch_z2(Handle* H, int B, int col0, const double* uni, RngSpec rng, bool given, double* cond,
               bool want_lp) {
  (void)col0;
  (void)cond;
  if (given) throw std::logic_error("launch_z2: given configurations go through forward_plain (spec.cu)");
  launch_tail_umma(H, B, uni, rng, want_lp);
}

void launch_finalize_logpsi(Handle* H, int B, int tiles) {
  KScope ks(H, "finalize_logpsi");
  finalize_logpsi_kernel<<<(B + 7) / 8, 256, 0, H->stream>>>(B, tiles, H->lp_head, H->lp_part, H->log_psi);
  LAUNCH_CHECK();
  H->launches++;
}

void launch_energy(Handle* H, int B) {
  if (H->dense_energy) {  // tensor-core quadratic form (energy_dense.cu)
    launch_energy_dense(H, B);
    return;
  }
  const int W = H->L.W;
  const size_t tw = (size_t)(32 * W + 32) * sizeof(uint32_t);
  const size_t cap = 110 * 1024;  // two CTAs per SM
  if (H->d_edges_bank && W <= kCutThreads && tw + 16 * 1024 <= cap) {  // bit-sliced path (n <= 12,288)
    const int groups = (B + 31) / 32;
    const int64_t nEp = H->num_edges_bank;
    // edge chunks: fit the remaining shared memory; small batches split further (more CTAs, up to
    // two per SM) while a chunk keeps >= 2 passes' worth of entries; groups are spread over the CTAs
    const int64_t per_max = std::min<int64_t>(63 * kCutThreads, (int64_t)((cap - tw) / 4)) & ~int64_t(127);
    int64_t chunks = std::max<int64_t>(1, (nEp + per_max - 1) / per_max);
    // small batches: at most 4 edge chunks (each chunk's CTA redoes its group's bit transposes;
    // measured at B = 1024, N = 10k: 4 chunks 11.1 us, 8 chunks 13.2 us, 1 chunk 13.2 us)
    static const int64_t max_chunks = [] {
      const char* e = std::getenv("VQMC_CUT_MAXCHUNKS");
      return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)4;
    }();
    while (chunks * groups * 2 <= 2 * 148 && nEp / (2 * chunks) >= 2 * kCutThreads && 2 * chunks <= max_chunks)
      chunks *= 2;
    int64_t per = std::max<int64_t>(128, ((nEp + chunks - 1) / chunks + 127) & ~int64_t(127));
    chunks = std::max<int64_t>(1, (nEp + per - 1) / per);
    const int ctas_y = (int)std::min<int64_t>(groups, std::max<int64_t>(1, (2 * 148) / chunks));
    const size_t smem = tw + (size_t)per * 4;
    ensure_smem_attr((const void*)maxcut_cut_kernel, cap);
    H->ensure_cpart((int)chunks * B);
    H->cut_chunks = (int)chunks;
    KScope ks(H, "maxcut_energy");
    launch_k(H, maxcut_cut_kernel, dim3((unsigned)chunks, (unsigned)ctas_y), dim3(kCutThreads), smem, B, W, nEp, per,
             (const uint32_t*)H->d_edges_bank, (const uint32_t*)H->X, H->cpart);
    LAUNCH_CHECK();
    H->launches++;
    return;
  }
  constexpr int S = 4;
  const size_t smem = (size_t)S * W * sizeof(uint32_t);
  ensure_smem_attr((const void*)energy_kernel<S>, smem);
  H->ensure_cpart(B);
  H->cut_chunks = 1;
  KScope ks(H, "maxcut_energy");
  energy_kernel<S><<<(B + S - 1) / S, 256, smem, H->stream>>>(B, W, H->num_edges, H->d_edges, H->X,
                                                              H->cpart, H->local);
  LAUNCH_CHECK();
  H->launches++;
}

__global__ void cuts_reduce_kernel(int B, int chunks, const int32_t* __restrict__ cpart, int32_t* __restrict__ cut) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int c = 0;
  for (int k = 0; k < chunks; ++k) c += cpart[(size_t)k * B + b];
  cut[b] = c;
}

void launch_cuts_reduce(Handle* H, int B) {
  cuts_reduce_kernel<<<(B + 255) / 256, 256, 0, H->stream>>>(B, H->cut_chunks, H->cpart, H->cut);
  LAUNCH_CHECK();
  H->launches++;
}

void launch_weights_from_locals(Handle* H, int B, int seg, bool with_wg1, const double* lin, double* lstat) {
  const Layout& L = H->L;
  const size_t smem = (size_t)B * sizeof(float);
  ensure_smem_attr((const void*)stats_weights_kernel, smem);
  const int64_t total = (int64_t)B * H->hp18;
  const int grid = with_wg1 ? (int)std::max<int64_t>(1, std::min<int64_t>(148, (total + 4095) / 4096)) : 1;
  KScope ks(H, with_wg1 ? "stats_weights_wg1" : "stats_weights");
  launch_k(H, stats_weights_kernel, dim3(grid), dim3(1024), smem, B / seg, seg, H->cut_chunks, H->num_edges,
           (const int32_t*)H->cpart, H->cut, H->local, H->w, H->d_wscale, H->d_istat, L.h, (int)H->hp18,
           (const float*)(with_wg1 ? H->G1 : nullptr), H->wG1h, H->wG1l,
           (float*)(with_wg1 && H->nccl_comm && !lin ? H->G + L.total : nullptr), H->nranks, H->rank, lin, lstat);
  LAUNCH_CHECK();
  H->launches++;
}

void launch_backward(Handle* H, int B, bool wg1_done) {
  launch_gw2_umma(H, B, wg1_done);  // gW2 (.) M2 and gb2
  launch_backward_tail(H, B);
}

// dg1 -> dz1 -> gW1: the W1 / b1 part of the gradient (independent of gW2)
void launch_backward_tail(Handle* H, int B) {
  launch_dg1_umma(H, B);  // E = D . W2m (split-K partials): the step's last read of the W2 pairs
  launch_backward_after_dg1(H, B);
}

// dz1 -> gW1 (+ finalize)
void launch_backward_after_dg1(Handle* H, int B, cudaEvent_t after_dz1) {
  using namespace bwcfg;
  const Layout& L = H->L;
  {
    KScope ks(H, "bw_dz1");
    const size_t total = ((size_t)B * L.h + 3) / 4;  // (4 entries per thread)
    launch_k(H, dz1_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, B, L.h, H->hp8, H->splits,
             (const float*)H->Epart, (const float*)H->w, (const float*)H->G1, H->dz1bh, H->dz1bl);
    LAUNCH_CHECK();
    H->launches++;
  }
  if (after_dz1) VQMC_CUDA(cudaEventRecord(after_dz1, H->stream));
  {
    int splits = 1;
    launch_gw1_umma(H, B, splits);  // gW1 (tcgen05): direct epilogue, or split-K partials
    if (splits == 1) return;
    KScope ks(H, "bw_gw1_finalize");
    const int total = ((L.Hd + 1) * L.h + 3) / 4;  // (4 entries per thread)
    launch_k(H, gw1_finalize_kernel, dim3((total + 255) / 256), dim3(256), 0, L.h, L.Hd, splits,
             (const float*)H->gw1_part, (const int32_t*)H->d_deg, (const float*)H->d_wscale, H->G + L.off_w1t,
             H->G + L.off_b1);
    LAUNCH_CHECK();
    H->launches++;
  }
}

__global__ void set_step_kernel(StepParams* sp, uint64_t call, int64_t t, float lr, float b1, float b2,
                                float eps) {
  sp->call = call;
  sp->t = t;
  sp->lr = lr;
  sp->b1 = b1;
  sp->b2 = b2;
  sp->eps = eps;
  adam_bias(b1, b2, t, sp->bc1, sp->bc2, sp->ibc1, sp->ibc2);
  adam_bias(b1, b2, t + 1, sp->nbc1, sp->nbc2, sp->nibc1, sp->nibc2);
}

void launch_set_step(Handle* H, uint64_t call, int64_t t, double lr, double b1, double b2, double eps) {
  set_step_kernel<<<1, 1, 0, H->stream>>>(H->d_step, call, t, (float)lr, (float)b1, (float)b2, (float)eps);
  LAUNCH_CHECK();
  H->launches++;
}

static AdamOut adam_out(const Handle* H, bool gated) {
  const Layout& L = H->L;
  const bool vec = (L.h % 4) == 0 && (L.off_w2 % 4) == 0;
  return AdamOut{L.h, H->hp18, L.Hd, H->head_hpk, H->head_Hdp, 1.f / (float)L.h, H->head_fast, vec, L.off_b1,
                 L.off_w2, L.off_b2,
                 H->d_comp_pos, H->W1Tp, H->W2cp, H->W2h, H->W2l,
                 gated ? H->d_flag : nullptr, H->head_v4, H->h4};
}

void launch_adam(Handle* H, float grad_scale, bool gated) {  // the whole live buffer in one launch
  KScope ks(H, "adam");
  const int nb = std::min(H->gpart_n, 148 * 4);  // (4 resident 256-thread blocks per SM)
  launch_k(H, adam_kernel, dim3(nb), dim3(256), 0, (int64_t)0, H->L.total, grad_scale,
           (const StepParams*)H->d_step, H->P, (const float*)H->G, H->Mo, H->Vo, H->d_gpart, 0, nb, H->d_done,
           H->d_scal, adam_out(H, gated));
  LAUNCH_CHECK();
  H->launches++;
}

// Adam split at off_w2: part 0 = [off_w2, total) ([W2 | b2]: ~99% of the parameters) with
// blocks0 blocks on `stream0`, part 1 = [0, off_w2) ([W1T | b1]) on the handle's stream.
void launch_adam_part(Handle* H, float grad_scale, int part, cudaStream_t stream) {
  const Layout& L = H->L;
  // part 0 runs beside dz1 -> gW1: 4 blocks on each of the SMs gW2 used (4 x 256 threads fill an SM)
  const int blocks0 = std::min(H->gpart_n / 2, 4 * std::max(2, H->adam_w2_sms));
  // part 1 ([W1T | b1], ~1% of the parameters) on 148 blocks: one float4 group per thread (its time
  // is mostly load latency and the last block's final sum: 17.6 -> 15.3 us vs 74 blocks)
  const int blocks1 = std::min(H->gpart_n - blocks0, H->gpart_n / 8);
  const int64_t lo = part == 0 ? L.off_w2 : 0, hi = part == 0 ? L.total : L.off_w2;
  const int nb = part == 0 ? blocks0 : blocks1;
  KScope ks(H, part == 0 ? "adam_w2" : "adam_w1", stream);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  if (H->pdl) {  // (adam_kernel waits before touching global memory)
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  VQMC_CUDA(cudaLaunchKernelEx(&cfg, adam_kernel, lo, hi, grad_scale, (const StepParams*)H->d_step, H->P,
                               (const float*)H->G, H->Mo, H->Vo, H->d_gpart, part == 0 ? 0 : blocks0, blocks0 + blocks1,
                               H->d_done, H->d_scal, adam_out(H, true)));
  LAUNCH_CHECK();
  H->launches++;
}

}  // namespace vqmc_b200

// ===========================================================================
// Energy-kernel throughput hook (bench / profiles): cut values of B device-resident random spin
// rows through the production launcher (edge-list or dense path, as the handle dispatches), timed
// with CUDA events on the handle's stream over `iters` launches after one warm-up.  The batch
// lives in its own buffer (the handle's batch buffers are not grown to B).
// ===========================================================================
namespace vqmc_b200 {
__global__ void random_bits_kernel(int64_t words, int n, int W, uint64_t seed, uint32_t* __restrict__ X) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < words; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)t * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const int w = (int)(t % W);
    const int valid = n - 32 * w;  // bits of this word inside the row
    uint32_t v = (uint32_t)z;
    if (valid < 32) v &= (1u << valid) - 1u;
    X[t] = v;
  }
}
}  // namespace vqmc_b200

extern "C" int vqmc_test_energy_rate(vqmc_gpu_t* g, int B, int iters, float* ms_per_launch, int* chunks_out) {
  using namespace vqmc_b200;
  Handle* H = reinterpret_cast<Handle*>(g);
  uint32_t* X = nullptr;
  uint32_t* saved = H->X;
  int saved_cap = H->cap_B;
  try {
    const int64_t words = (int64_t)B * H->L.W;
    VQMC_CUDA(cudaMalloc((void**)&X, words * sizeof(uint32_t)));
    random_bits_kernel<<<148 * 8, 256, 0, H->stream>>>(words, H->L.n, H->L.W, 12345, X);
    VQMC_CUDA(cudaGetLastError());
    H->invalidate_graph();
    H->X = X;
    H->cap_B = std::max(H->cap_B, B);  // (only the energy path runs against this buffer)
    cudaEvent_t e0, e1;
    VQMC_CUDA(cudaEventCreate(&e0));
    VQMC_CUDA(cudaEventCreate(&e1));
    launch_energy(H, B);  // warm-up (sizes cpart)
    VQMC_CUDA(cudaEventRecord(e0, H->stream));
    for (int i = 0; i < iters; ++i) launch_energy(H, B);
    VQMC_CUDA(cudaEventRecord(e1, H->stream));
    VQMC_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    VQMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_launch = ms / std::max(1, iters);
    *chunks_out = H->cut_chunks;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  } catch (const std::exception& ex) {
    H->X = saved;
    H->cap_B = saved_cap;
    if (X) cudaFree(X);
    set_error(ex.what());
    return status_of(ex);
  }
  H->X = saved;
  H->cap_B = saved_cap;
  cudaFree(X);
  return VQMC_OK;
}

// ===========================================================================
// Forward / TIM local-energy throughput hook (profiles): B device-resident random configurations
// in the handle's batch buffers; mode 0 = the plain forward (log_psi_batch: z1_given + the tcgen05
// given-bits GEMM + finalize), mode 1 = local_energy_batch of the handle's spec (diagonal, base
// forward, neighbour GEMMs, combine).  Timed with CUDA events over `iters` calls after one warm-up;
// then one pass with per-kernel events (names_out: cap slots of 32 chars).
// ===========================================================================
extern "C" int vqmc_test_forward_rate(vqmc_gpu_t* g, int B, int iters, int mode, float* ms_per_call, char* names_out,
                                      float* kms_out, int cap, int* count) {
  using namespace vqmc_b200;
  Handle* H = reinterpret_cast<Handle*>(g);
  try {
    if (mode == 1 && !H->spec) throw InvalidArgument("mode 1 needs a spec (vqmc_gpu_set_spec)");
    H->ensure_batch(B);
    const int64_t words = (int64_t)B * H->L.W;
    random_bits_kernel<<<148 * 8, 256, 0, H->stream>>>(words, H->L.n, H->L.W, 12345, H->X);
    VQMC_CUDA(cudaGetLastError());
    auto call = [&] {
      if (mode == 0) forward_plain(H, B, nullptr, nullptr, nullptr, nullptr, H->log_psi);
      else launch_spec_local(H, B, nullptr, spec_local_buffer(H, B));
    };
    cudaEvent_t e0, e1;
    VQMC_CUDA(cudaEventCreate(&e0));
    VQMC_CUDA(cudaEventCreate(&e1));
    call();  // warm-up (allocations, smem attributes)
    VQMC_CUDA(cudaEventRecord(e0, H->stream));
    for (int i = 0; i < iters; ++i) call();
    VQMC_CUDA(cudaEventRecord(e1, H->stream));
    VQMC_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    VQMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_call = ms / std::max(1, iters);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const int kt = H->ktimer;
    H->ktimer = 1;
    H->kt_count = 0;
    call();
    H->ktimer = kt;
    VQMC_CUDA(cudaStreamSynchronize(H->stream));
    const int c = std::min(cap, H->kt_count);
    for (int i = 0; i < c; ++i) {
      VQMC_CUDA(cudaEventElapsedTime(&kms_out[i], H->kt_start[i], H->kt_end[i]));
      std::strncpy(names_out + 32 * i, H->kt_name[i], 31);
      names_out[32 * i + 31] = 0;
    }
    *count = c;
    uint32_t flag = 0;
    VQMC_CUDA(cudaMemcpy(&flag, H->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag) {
      VQMC_CUDA(cudaMemset(H->d_flag, 0, sizeof(flag)));
      throw NumericError("non-finite value in the timed forward");
    }
  } catch (const std::exception& ex) {
    set_error(ex.what());
    return status_of(ex);
  }
  return VQMC_OK;
}
