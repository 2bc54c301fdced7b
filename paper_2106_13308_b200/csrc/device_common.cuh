// Device helpers shared by the VQMC kernels: Philox uniforms, the clamped
// Bernoulli conditional of the MADE output, and a SIMT fp32 GEMM main loop.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"
#include "ptx.cuh"

namespace vqmc_b200 {

constexpr unsigned kFull = 0xffffffffu;

// Philox4x32-10 (production-mode uniforms; restated in oracle/vqmc_oracle.cpp).
// key = mix_seed(seed, stream); counter = (bit >> 2, sample, call_lo, call_hi); output word
// j = bit & 3 gives u = (r_j + 1/2) * 2^-32 (32-bit resolution, never 0 or 1).
__device__ __forceinline__ void philox4_k(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                          uint32_t c3, uint32_t (&r)[4]) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  r[0] = c0;
  r[1] = c1;
  r[2] = c2;
  r[3] = c3;
}
__device__ __forceinline__ void philox4(uint64_t key, uint32_t quad, uint32_t sample, uint64_t call,
                                        uint32_t (&r)[4]) {
  philox4_k((uint32_t)key, (uint32_t)(key >> 32), quad, sample, (uint32_t)call, (uint32_t)(call >> 32), r);
}
__device__ __forceinline__ double u32_to_uniform(uint32_t r) { return ((double)r + 0.5) * 0x1.0p-32; }

// mix_seed (proj/include/vqmc/common.hpp:56-61) on the device.
__device__ __forceinline__ uint64_t mix_seed_dev(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Production-mode uniform of (row b, bit i): the batch is `segments` workers of
// `seg` rows; worker s draws from stream (stream0 + s) with sample index b - s*seg.
struct RngSpec {
  uint64_t seed, stream0, call;
  int seg;
  const StepParams* sp;  // when set, the call counter is read from device memory (graph replays)
  __device__ __forceinline__ uint64_t c() const { return sp ? sp->call : call; }
  // raw outputs for bits (i & ~3) .. (i | 3) of row b
  __device__ __forceinline__ void quad(int b, int i, uint32_t (&r)[4]) const {
    const int s = b / seg;
    philox4(mix_seed_dev(seed, stream0 + (uint64_t)s), (uint32_t)(i >> 2), (uint32_t)(b - s * seg), c(), r);
  }
  __device__ __forceinline__ double operator()(int b, int i) const {
    uint32_t r[4];
    quad(b, i, r);
    return u32_to_uniform(r[i & 3]);
  }
};

__device__ __forceinline__ float softplusf(float y) {
  return fmaxf(y, 0.f) + log1pf(expf(-fabsf(y)));
}

// One output unit of the MADE given its logit z (proj/src/models.cpp:59-60,
// 64-70, 163-171 and proj/src/sampler.cpp:50-53):
//   p_raw = sigmoid(z); p = clamp(p_raw, 1e-7, 1 - 1e-7)
//   draw:  x = [u < p]                      (fp64 compare, like the reference)
//   logt = x ? log p : log(1 - p)           (computed stably from z)
//   D    = 0.5 (x - p_raw), zeroed where the clamp is active (made_dz2)
struct Unit {
  float D;
  float logt;
  double p;
};

__device__ __forceinline__ double clamped_p(float z) {
  if (z >= kLogitHi) return 1.0 - kProbEps;
  if (z <= -kLogitHi) return kProbEps;
  return (double)(1.f / (1.f + __expf(-z)));
}

// Shared transcendental work of one output unit: e = exp(-|z|), r = 1 / (1 + e),
// log1p(e): sigmoid, its complement and both softplus values follow without cancellation.
struct UnitPre {
  float praw, qraw, sp_pos, sp_neg;  // p_raw, 1 - p_raw, softplus(z) = -log(1-p), softplus(-z) = -log p
  bool hi, lo;                       // clamp active at 1 - eps / at eps
  __device__ __forceinline__ double p() const {
    return hi ? 1.0 - kProbEps : (lo ? kProbEps : (double)praw);
  }
};
__device__ __forceinline__ UnitPre unit_pre(float z) {
  UnitPre o;
  o.hi = z >= kLogitHi;
  o.lo = z <= -kLogitHi;
  const float e = __expf(-fabsf(z));
  const float r = __frcp_rn(1.f + e);
  const float L = log1pf(e);  // accurate: the log-probs sum n of these terms
  o.praw = z >= 0.f ? r : e * r;
  o.qraw = z >= 0.f ? e * r : r;
  o.sp_pos = fmaxf(z, 0.f) + L;
  o.sp_neg = fmaxf(-z, 0.f) + L;
  return o;
}
// Same without the softplus terms (callers that do not accumulate the log-probability).
__device__ __forceinline__ UnitPre unit_pre_nolog(float z) {
  UnitPre o;
  o.hi = z >= kLogitHi;
  o.lo = z <= -kLogitHi;
  const float e = __expf(-fabsf(z));
  const float r = __frcp_rn(1.f + e);
  o.praw = z >= 0.f ? r : e * r;
  o.qraw = z >= 0.f ? e * r : r;
  o.sp_pos = 0.f;
  o.sp_neg = 0.f;
  return o;
}
__device__ __forceinline__ Unit unit_post(const UnitPre& q, int x) {
  Unit o;
  if (q.hi || q.lo) {
    const float lsmall = -16.11809565095832f, lbig = -1.00000005e-7f;  // log(1e-7), log1p(-1e-7)
    o.D = 0.f;
    o.logt = (q.hi == (x != 0)) ? lbig : lsmall;
  } else {
    o.logt = x ? -q.sp_neg : -q.sp_pos;
    o.D = x ? 0.5f * q.qraw : -0.5f * q.praw;
  }
  o.p = q.p();
  return o;
}
__device__ __forceinline__ Unit unit_terms(float z, int x) { return unit_post(unit_pre(z), x); }

// ---------------------------------------------------------------------------
// SIMT fp32 GEMM main loop: acc[TM][TN] += sum_k A(m, k) * B(n, k) over the
// tile (m0, n0) and k in [kb, ke).  Loaders are functors returning 0 outside
// the problem; `kMMajor` says whether consecutive m (or n) are contiguous so
// the tile loads coalesce.  Thread (tx, ty): rows ty + (BM/TM) * r, columns
// tx*4 + (BN/2) * q + j (two float4 groups for coalesced epilogue stores).
// ---------------------------------------------------------------------------
template <int BM, int BN, int BK, int TM, int TN>
struct SimtTile {
  static constexpr int NTX = BN / TN, NTY = BM / TM, NT = NTX * NTY;
  static_assert(TN == 8, "epilogue column map assumes TN == 8");
  static_assert(NTX * 4 * 2 == BN, "column map");
  __device__ static int row(int ty, int r) { return ty + NTY * r; }
  __device__ static int col(int tx, int c) { return tx * 4 + (BN / 2) * (c >> 2) + (c & 3); }
};

template <int BM, int BN, int BK, int TM, int TN, class LA, class LB>
__device__ __forceinline__ void simt_mainloop(float (&acc)[TM][TN], int m0, int n0, int kb, int ke,
                                              const LA& la, const LB& lb, float* smem) {
  using T = SimtTile<BM, BN, BK, TM, TN>;
  float* As = smem;            // [BK][BM]
  float* Bs = smem + BK * BM;  // [BK][BN]
  const int tid = threadIdx.x;
  const int tx = tid % T::NTX, ty = tid / T::NTX;
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = 0.f;
  constexpr int AE = (BM * BK + T::NT - 1) / T::NT;
  constexpr int BE = (BN * BK + T::NT - 1) / T::NT;
  float ra[AE], rb[BE];
  auto gload = [&](int k0) {
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      const int idx = tid + e * T::NT;
      int m, k;
      if (LA::kMMajor) { m = idx % BM; k = idx / BM; } else { k = idx % BK; m = idx / BK; }
      ra[e] = (idx < BM * BK && k0 + k < ke) ? la(m0 + m, k0 + k) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < BE; ++e) {
      const int idx = tid + e * T::NT;
      int n, k;
      if (LB::kMMajor) { n = idx % BN; k = idx / BN; } else { k = idx % BK; n = idx / BK; }
      rb[e] = (idx < BN * BK && k0 + k < ke) ? lb(n0 + n, k0 + k) : 0.f;
    }
  };
  auto sstore = [&]() {
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      const int idx = tid + e * T::NT;
      if (idx < BM * BK) {
        int m, k;
        if (LA::kMMajor) { m = idx % BM; k = idx / BM; } else { k = idx % BK; m = idx / BK; }
        As[k * BM + m] = ra[e];
      }
    }
#pragma unroll
    for (int e = 0; e < BE; ++e) {
      const int idx = tid + e * T::NT;
      if (idx < BN * BK) {
        int n, k;
        if (LB::kMMajor) { n = idx % BN; k = idx / BN; } else { k = idx % BK; n = idx / BK; }
        Bs[k * BN + n] = rb[e];
      }
    }
  };
  if (kb >= ke) return;
  gload(kb);
  for (int k0 = kb; k0 < ke; k0 += BK) {
    __syncthreads();
    sstore();
    __syncthreads();
    if (k0 + BK < ke) gload(k0 + BK);  // register prefetch of the next tile
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int r = 0; r < TM; ++r) a[r] = As[k * BM + T::row(ty, r)];
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k * BN + tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k * BN + BN / 2 + tx * 4]);
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
  }
}

}  // namespace vqmc_b200
