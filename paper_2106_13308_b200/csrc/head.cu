// Head sampler v2 (sm_100a): the strictly sequential bits 0 .. Hd-1 of the MADE
// ancestral sampler (proj/src/sampler.cpp:47-55 restricted to the bits whose
// conditionals still depend on earlier draws; Hd = max degree).
//
// Layout: one CTA = `nw` consumer warps (one sample each) + 1 producer warp.
// Per sampled bit i a warp applies two rank-1 updates held in registers
// (lane l owns hidden units and head outputs l + 32 m):
//     z1 += x_i * W1m[:, i]                      (all hidden units)
//     z2_head += relu(z1_k) * W2m[:, k]          (k = units completed by bit i)
// so bit i's logit is complete when it is drawn.  The rows W1m[:, i] and
// W2m[:, k] do not depend on the samples: the producer warp streams them for
// groups of G bits into a ring of shared-memory slots with cp.async.bulk (TMA)
// completing on mbarriers, shared by all warps of the CTA.
//
// The draw is x_i = [u < clamp(sigmoid(z))] evaluated as [logit(u) < z] with the
// clamp folded into the threshold (u < 1e-7 -> always 1, u >= 1 - 1e-7 -> always 0),
// so the serial chain per bit is: compare -> shfl x -> fma -> relu -> shfl g -> fma.
// The per-bit output terms (D, log-prob, conditionals) are computed 32 bits at a
// time, one bit per lane, off the chain.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "head4.cuh"
#include "ptx.cuh"

namespace vqmc_b200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Same with a suspend-time hint: the waiting thread sleeps instead of re-polling (producer warps
// share an SM sub-partition with a consumer warp, so their polling would steal its issue slots).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct HeadGeom {
  int G;       // bits per slot
  int R;       // slots in the ring
  int hp;      // padded W1 row length (floats, multiple of 4)
  int Hdp;     // padded W2 row length
  int cmax;    // max completions in one group of G bits
  int ngroups;
  int slot_floats;
  int ring_off;  // v3: byte offset of the row ring (after the mbarriers)
  size_t smem;
};

// logit threshold of a uniform: x = [u < clamp(sigmoid(z), eps, 1-eps)] == [thr < z]
__device__ __forceinline__ float logit_threshold(double u) {
  if (u < kProbEps) return -INFINITY;
  if (u >= 1.0 - kProbEps) return INFINITY;
  return (float)(log(u) - log1p(-u));
}

template <int KPL, bool FAST, bool GIVEN>
__global__ void __launch_bounds__(32 * 9) head_v2_kernel(
    int B, int n, int h, int Hd, int W, HeadGeom geo, const float* __restrict__ W1Tp,
    const float* __restrict__ W2cp, const float* __restrict__ b1, const float* __restrict__ b2,
    const int* __restrict__ comp_k, const int* __restrict__ comp_off, const double* __restrict__ uni,
    RngSpec rng, int w1skip, uint32_t* __restrict__ X, float* __restrict__ G1,
    __half* __restrict__ G1h, __half* __restrict__ G1l, int hp, __half* __restrict__ Dh,
    __half* __restrict__ Dl, int np, __nv_bfloat16* __restrict__ Xf, int hd1p, double* __restrict__ lp_head,
    double* __restrict__ cond) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int G = geo.G;  // power of two
  const int nw = blockDim.x / 32 - 1;  // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + geo.R;
  int* s_off = reinterpret_cast<int*>(empty + geo.R);           // [Hd + 1]
  int* s_ck = s_off + (Hd + 1);                                  // [h]
  float* ring = reinterpret_cast<float*>(smem_raw + ((16 * geo.R + 4 * (Hd + 1 + h) + 127) / 128) * 128);
  for (int t = threadIdx.x; t <= Hd; t += blockDim.x) s_off[t] = comp_off[t];
  for (int t = threadIdx.x; t < h; t += blockDim.x) s_ck[t] = comp_k[t];
  if (threadIdx.x == 0) {
    for (int r = 0; r < geo.R; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == nw) {  // ---------------- producer warp ----------------
    if (lane == 0) {
      int slot = 0, use = 0;
      for (int g = 0; g < geo.ngroups; ++g) {
        if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
        const int i0 = g * G, i1 = min(Hd, i0 + G);
        const int c0 = s_off[i0], c1 = s_off[i1];
        const uint32_t b_w1 = (uint32_t)(i1 - i0) * geo.hp * 4u;
        const uint32_t b_w2 = (uint32_t)(c1 - c0) * geo.Hdp * 4u;
        float* dst = ring + (size_t)slot * geo.slot_floats;
        mbar_expect_tx(&full[slot], b_w1 + b_w2);
        bulk_g2s(dst, W1Tp + (size_t)i0 * geo.hp, b_w1, &full[slot]);
        if (b_w2) bulk_g2s(dst + G * geo.hp, W2cp + (size_t)c0 * geo.Hdp, b_w2, &full[slot]);
        if (++slot == geo.R) {
          slot = 0;
          ++use;
        }
      }
    }
    return;
  }

  // ---------------- consumer warps: one sample each ----------------
  // The word loop is unrolled so every register index is static; G divides 32, so a
  // ring slot never straddles two words.  FAST: bit i completes exactly hidden unit i
  // (cyclic degrees with h <= n - 1, models.cpp:91), so the completed unit's register
  // is z1[m] on lane l and only the words >= m can still change.
  const int b = blockIdx.x * nw + warp;
  const bool active = b < B;
  float z1[KPL], z2[KPL];
#pragma unroll
  for (int m = 0; m < KPL; ++m) {
    const int k = lane + 32 * m;
    z1[m] = k < h ? b1[k] : 0.f;
    z2[m] = k < Hd ? b2[k] : 0.f;
  }
  double lp = 0.0;
  const size_t rowD = (size_t)b * np, rowC = (size_t)b * n;
  auto store_g1 = [&](int k, float g) {
    G1[(size_t)b * h + k] = g;
    ptx::split_f16(g, G1h[(size_t)b * hp + k], G1l[(size_t)b * hp + k]);
  };
  auto word_input = [&](int m, float& thr, int& xin) {
    const int ib = 32 * m + lane;
    thr = 0.f;
    xin = 0;
    if (active && ib < Hd) {
      if (GIVEN) xin = (X[(size_t)b * W + m] >> lane) & 1;
      else thr = logit_threshold(uni ? uni[(size_t)ib * B + b] : rng(b, ib));
    }
  };
  float thr_next;
  int xin_next;
  word_input(0, thr_next, xin_next);
  const float* w1s = ring;
  const float* w2s = ring;
  int cbase = 0;
  int slot = 0, use = 0;
#pragma unroll
  for (int m = 0; m < KPL; ++m) {
    if (32 * m < Hd) {
      const float thr = thr_next;
      const int xin = xin_next;
      if (32 * (m + 1) < Hd) word_input(m + 1, thr_next, xin_next);  // overlaps this word
      float zmine = 0.f, gmine = 0.f;
      int xmine = 0;
      const int lend = min(32, Hd - 32 * m);
      constexpr int RS = 32 * KPL;  // FAST: row stride of the staged W1 / W2 rows (compile time)
      const float* wr1 = w1s;
      const float* wr2 = w2s;
      for (int l = 0; l < lend; ++l) {
        const int i = 32 * m + l;
        if ((i & (G - 1)) == 0) {
          mbar_wait(&full[slot], use & 1);
          w1s = ring + (size_t)slot * geo.slot_floats;
          w2s = w1s + G * geo.hp;
          wr1 = w1s;
          wr2 = w2s;
          cbase = s_off[i];
        }
        const float z = z2[m];
        int x = GIVEN ? xin : (thr < z ? 1 : 0);
        if (lane == l) {
          zmine = z;
          xmine = x;
        }
        // rows are zero-padded to 32 * KPL floats: no bounds predicates below
        const float xf = (float)__shfl_sync(kFull, x, l);
        if (FAST) {
#pragma unroll
          for (int mm = 0; mm < KPL; ++mm)
            if (mm >= m) z1[mm] = fmaf(xf, wr1[lane + 32 * mm], z1[mm]);
          const float gk = __shfl_sync(kFull, fmaxf(z1[m], 0.f), l);
          if (lane == l) gmine = gk;  // hidden unit i = 32 m + l; stored at the end of the word
#pragma unroll
          for (int mm = 0; mm < KPL; ++mm)
            if (mm >= m) z2[mm] = fmaf(wr2[lane + 32 * mm], gk, z2[mm]);
          wr1 += RS;
          wr2 += RS;
        } else {
          const float* wr = w1s + (i & (G - 1)) * geo.hp;
#pragma unroll
          for (int mm = 0; mm < KPL; ++mm)
            if (!w1skip || mm >= m) z1[mm] = fmaf(xf, wr[lane + 32 * mm], z1[mm]);
          for (int c = s_off[i]; c < s_off[i + 1]; ++c) {
            const int k = s_ck[c];
            const int ks = k >> 5, kl = k & 31;
            float v = 0.f;
#pragma unroll
            for (int mm = 0; mm < KPL; ++mm) v = (mm == ks) ? z1[mm] : v;
            const float gk = __shfl_sync(kFull, fmaxf(v, 0.f), kl);
            if (active && lane == kl) store_g1(k, gk);
            const float* wr2g = w2s + (c - cbase) * geo.Hdp;
#pragma unroll
            for (int mm = 0; mm < KPL; ++mm)
              if (mm >= m && 32 * mm < geo.Hdp) z2[mm] = fmaf(wr2g[lane + 32 * mm], gk, z2[mm]);
          }
        }
        if (((i + 1) & (G - 1)) == 0 || i == Hd - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          if (++slot == geo.R) {
            slot = 0;
            ++use;
          }
        }
      }
      if (FAST && active && 32 * m + lane < Hd) store_g1(32 * m + lane, gmine);
      // word complete: per-lane output terms and bit packing (off the serial chain)
      const int ib = 32 * m + lane;
      const bool mine = active && ib < Hd;
      if (mine) {
        const Unit u = unit_terms(zmine, xmine);
        ptx::split_f16(u.D, Dh[rowD + ib], Dl[rowD + ib]);
        lp += (double)u.logt;
        if (cond) cond[rowC + ib] = u.p;
        Xf[(size_t)b * hd1p + ib] = __float2bfloat16_rn((float)xmine);
      }
      const uint32_t word = __ballot_sync(kFull, mine && xmine);
      if (!GIVEN && active && lane == 0) X[(size_t)b * W + m] = word;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lp += __shfl_xor_sync(kFull, lp, o);
  if (active && lane == 0) {
    lp_head[b] = lp;
    Xf[(size_t)b * hd1p + Hd] = __float2bfloat16_rn(1.f);  // ones column: gb1 = 1^T dz1
  }
}

// ===========================================================================
// Head sampler v3: the "fast" MADE structure (bit i completes exactly hidden unit i:
// the reference's cyclic degrees deg_k = k + 1 when h <= n - 1, models.cpp:91), two
// samples per warp.
//
// Lane l owns units / outputs 32 m + l (word slot m).  While word m is sampled, only slots
// >= m still change, so the registers hold RELATIVE slots t = slot - m (shifted down by one
// after every word) and the staged rows of the bits of word m are stored in the same
// relative, lane-interleaved order: row i (word m = i / 32) keeps unit 32 (m + t) + l at
// position 128 (t >> 2) + 4 l + (t & 3), so one LDS.128 gives a lane four consecutive
// relative slots and the rows shrink word by word (triangular staging).  The code of a bit
// is therefore the same for every word (a compact loop, no per-word unrolling).
//
// Bit i = 32 m + l is owned by lane l: it has the logit z2[0] and z1[0] of unit i (and the
// diagonal weight W1T[i][i] in its own float4), so it computes x_i and g_i = relu(z1_i +
// x_i W1T[i][i]) without communication and sends both in ONE shuffle (x in the sign bit of
// g >= 0).  Every lane then applies the two rank-1 updates.  Serial chain per bit: compare,
// select, max, select, shuffle, fma.  The rows of bit i + 1 are loaded while bit i is
// processed (ping-pong registers); the two samples share every shared-memory load.
// ===========================================================================
__host__ __device__ __forceinline__ int head_rel_pos(int t, int l) { return 128 * (t >> 2) + 4 * l + (t & 3); }
// staged floats of a row of word m (KPL word slots per lane)
__host__ __device__ __forceinline__ int head_row_floats(int KPL, int m) { return 128 * ((KPL - m + 3) >> 2); }

// Per-lane input of word m (this lane's bit 32 m + lane): the logit threshold of its uniform.
// Production draws: u = (r + 1/2) 2^-32 from a 32-bit Philox word r, so logit(u) =
// log((r + 1/2) / (~r + 1/2)) in fp32 (the ratio is exact up to fp32 rounding: the threshold
// is within ~2e-7 of the fp64 value, far inside the 1e-5 flip tolerance), with the
// clamp folded in: u < 1e-7 <=> r <= 428, u >= 1 - 1e-7 <=> ~r <= 428.  Parity mode (given
// fp64 uniforms) keeps the fp64 threshold.
__device__ __forceinline__ float head_threshold(const double* __restrict__ uni, RngSpec rng, int B, int b, int ib) {
  if (uni) return logit_threshold(uni[(size_t)ib * B + b]);
  uint32_t r4[4];
  rng.quad(b, ib, r4);
  const uint32_t r = r4[ib & 3], nr = ~r;
  if (r <= 428u) return -INFINITY;
  if (nr <= 428u) return INFINITY;
  return logf(((float)r + 0.5f) / ((float)nr + 0.5f));  // one log of the ratio: ~1e-7 absolute
}

// Logit thresholds of the head bits, thr[b][i] for i < Hd8 (bits >= Hd: +inf, they draw 0).
// Given configurations (made_forward) become -inf / +inf, so the head draws exactly those bits.
// One thread per (sample, 4 consecutive bits): one Philox call serves all four.
__global__ void head_thresholds_kernel(int B, int Hd, int Hd8, int W, const double* __restrict__ uni, RngSpec rng,
                                       const uint32_t* __restrict__ X, int given, float* __restrict__ thr) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int q4 = Hd8 >> 2;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * q4) return;
  const int b = (int)(t / q4), i0 = 4 * (int)(t % q4);
  float out[4];
  if (given) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k;
      out[k] = (i < Hd && ((X[(size_t)b * W + (i >> 5)] >> (i & 31)) & 1)) ? -INFINITY : INFINITY;
    }
  } else if (uni) {
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = i0 + k < Hd ? logit_threshold(uni[(size_t)(i0 + k) * B + b]) : INFINITY;
  } else {
    uint32_t r4[4];
    rng.quad(b, i0, r4);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t r = r4[k], nr = ~r;
      float v = r <= 428u ? -INFINITY : (nr <= 428u ? INFINITY : logf(((float)r + 0.5f) / ((float)nr + 0.5f)));
      out[k] = i0 + k < Hd ? v : INFINITY;
    }
  }
  *reinterpret_cast<float4*>(thr + (size_t)b * Hd8 + i0) = make_float4(out[0], out[1], out[2], out[3]);
}

// Outputs of one completed bit (sample b, bit ib; off the serial chain).
__device__ __forceinline__ double head_emit(int b, int ib, float z, float z1, int x, int n, int h, int hp, int np,
                                         int hd1p, float* __restrict__ G1, __half* __restrict__ G1h,
                                         __half* __restrict__ G1l, __half* __restrict__ Dh, __half* __restrict__ Dl,
                                         __nv_bfloat16* __restrict__ Xf, double* __restrict__ cond) {
  const float g = fmaxf(z1, 0.f);
  G1[(size_t)b * h + ib] = g;
  ptx::split_f16(g, G1h[(size_t)b * hp + ib], G1l[(size_t)b * hp + ib]);
  const Unit u = unit_terms(z, x);
  ptx::split_f16(u.D, Dh[(size_t)b * np + ib], Dl[(size_t)b * np + ib]);
  if (cond) cond[(size_t)b * n + ib] = u.p;
  Xf[(size_t)b * hd1p + ib] = __float2bfloat16_rn((float)x);
  return (double)u.logt;
}

struct HeadV3Args {
  int B, n, h, W;
  HeadGeom geo;
  const float* W1Tq;
  const float* W2cq;
  const float* b1;
  const float* b2;
  const double* uni;
  RngSpec rng;
  uint32_t* X;
  float* G1;
  __half* G1h;
  __half* G1l;
  int hp;
  __half* Dh;
  __half* Dl;
  int np;
  __nv_bfloat16* Xf;
  int hd1p;
  double* lp_head;
  double* cond;
  const float* thr;  // [B][Hd8] logit thresholds (head_thresholds_kernel)
};

constexpr int kHeadS = 2;  // samples per consumer warp (they share every shared-memory row load)

// Consumer state of one warp (kHeadS samples): relative slots and the ping-pong row buffers.
template <int KG>
struct HeadV3State {
  static constexpr int KPL = 4 * KG;
  float z1[kHeadS][KPL], z2[kHeadS][KPL];
  float4 wa1[KG], wa2[KG], wb1[KG], wb2[KG];
  float thr[kHeadS];       // this lane's logit threshold of the current word (given bits: -inf / +inf)
  float thr_next[kHeadS];  // the next word's (prefetched)
  float vp[kHeadS];   // shuffled (x, g) of the pending bit
  float dg;           // this lane's diagonal weight W1T[i][i] of the current bit (row of bit i, slot 0)
#ifdef VQMC_HEAD_PROF
  long long wait_cycles = 0;
#endif
  int slot, use;
  const float* rows;
};

// Rank-1 updates of one bit (shuffled value v: x in the sign bit, g = |v|) to relative slots
// [T0, T1) with that bit's rows (w1, w2).
template <int KG, int T0, int T1>
__device__ __forceinline__ void head_v3_update(HeadV3State<KG>& S, const float (&v)[kHeadS], const float4 (&w1)[KG],
                                               const float4 (&w2)[KG]) {
#pragma unroll
  for (int a = 0; a < kHeadS; ++a) {
    const float xf = (__float_as_uint(v[a]) >> 31) ? 1.f : 0.f;
    const float ga = fabsf(v[a]);
#pragma unroll
    for (int t = T0; t < T1; ++t) {
      const float4& r1 = w1[t >> 2];
      const float4& r2 = w2[t >> 2];
      const float c1 = (t & 3) == 0 ? r1.x : (t & 3) == 1 ? r1.y : (t & 3) == 2 ? r1.z : r1.w;
      const float c2 = (t & 3) == 0 ? r2.x : (t & 3) == 1 ? r2.y : (t & 3) == 2 ? r2.z : r2.w;
      S.z1[a][t] = fmaf(xf, c1, S.z1[a][t]);
      S.z2[a][t] = fmaf(ga, c2, S.z2[a][t]);
    }
  }
}

// Ring geometry in registers (the bit loop must not reload kernel parameters).
struct HeadRing {
  uint64_t* full;
  uint64_t* empty;
  float* ring;
  int G, R, slot_floats, Hd;
  int Hd8;  // bits rounded up to the 8-bit slot (staged rows padded with zero rows)
};

// Eight bits i0 .. i0 + 7 = one ring slot (G == 8, i0 slot-aligned), unrolled: static row
// buffers, static shuffle lanes l0 + k, and a single slot handover after the eighth bit.
template <int KG, int NQ, bool GIVEN, int K>
__device__ __forceinline__ void head_v3_bit8(HeadV3State<KG>& S, const HeadRing& Rg, int lane, int i0, int l0,
                                             float4 (&P1)[KG], float4 (&P2)[KG], const float4 (&C1)[KG],
                                             const float4 (&C2)[KG]) {
  constexpr int RS = 128 * KG;
  head_v3_update<KG, 0, 1>(S, S.vp, P1, P2);  // slot 0 of bit i - 1: on the serial chain
  float v[kHeadS];
#pragma unroll
  for (int a = 0; a < kHeadS; ++a) {
    const bool x = S.thr[a] < S.z2[a][0];
    const float z1u = x ? S.z1[a][0] + S.dg : S.z1[a][0];  // + x_i W1T[i][i] (prefetched diagonal)
    const float g = fmaxf(z1u, 0.f);
    v[a] = x ? -g : g;
    v[a] = __shfl_sync(kFull, v[a], l0 + K);
  }
  // rows of bit i + 1 (slot handover after the eighth bit); its diagonal weight is fetched now,
  // ahead of the bulk update, so the next bit's serial chain does not wait on shared memory
  const float* r1 = nullptr;
  if (K < 7) {
    r1 = S.rows + (K + 1) * RS + 4 * lane;
  } else if (i0 + 8 < Rg.Hd8) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&Rg.empty[S.slot]);  // rows of this slot are all in registers
    if (++S.slot == Rg.R) {
      S.slot = 0;
      ++S.use;
    }
    mbar_wait(&Rg.full[S.slot], S.use & 1);
    S.rows = Rg.ring + (size_t)S.slot * Rg.slot_floats;
    r1 = S.rows + 4 * lane;
  }
  if (r1) S.dg = r1[0];
  head_v3_update<KG, 1, 4 * NQ>(S, S.vp, P1, P2);  // the rest of bit i - 1
#pragma unroll
  for (int a = 0; a < kHeadS; ++a) S.vp[a] = v[a];
  if (r1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      P1[q] = *reinterpret_cast<const float4*>(r1 + 128 * q);
      P2[q] = *reinterpret_cast<const float4*>(r1 + 8 * RS + 128 * q);
    }
  }
}

template <int KG, int NQ, bool GIVEN>
__device__ __forceinline__ void head_v3_group8(HeadV3State<KG>& S, const HeadRing& Rg, int lane, int i0, int l0) {
  head_v3_bit8<KG, NQ, GIVEN, 0>(S, Rg, lane, i0, l0, S.wb1, S.wb2, S.wa1, S.wa2);
  head_v3_bit8<KG, NQ, GIVEN, 1>(S, Rg, lane, i0, l0, S.wa1, S.wa2, S.wb1, S.wb2);
  head_v3_bit8<KG, NQ, GIVEN, 2>(S, Rg, lane, i0, l0, S.wb1, S.wb2, S.wa1, S.wa2);
  head_v3_bit8<KG, NQ, GIVEN, 3>(S, Rg, lane, i0, l0, S.wa1, S.wa2, S.wb1, S.wb2);
  head_v3_bit8<KG, NQ, GIVEN, 4>(S, Rg, lane, i0, l0, S.wb1, S.wb2, S.wa1, S.wa2);
  head_v3_bit8<KG, NQ, GIVEN, 5>(S, Rg, lane, i0, l0, S.wa1, S.wa2, S.wb1, S.wb2);
  head_v3_bit8<KG, NQ, GIVEN, 6>(S, Rg, lane, i0, l0, S.wb1, S.wb2, S.wa1, S.wa2);
  head_v3_bit8<KG, NQ, GIVEN, 7>(S, Rg, lane, i0, l0, S.wa1, S.wa2, S.wb1, S.wb2);
}

// Side channels of a head CTA (besides the row ring):
//   thr (global)       logit thresholds [B][Hd8] from head_thresholds_kernel (consumers prefetch a word ahead)
//   zb[p][s][2][32]    final (z2, z1) of this lane's bit of word m, p = m & 1 (consumers -> emit warps)
struct HeadSide {
  uint64_t* zdone;      // [2]: all consumers wrote zb[p] (count nw)
  uint64_t* zfree;      // [2]: the emit warps consumed zb[p] (count kHeadEmitWarps)
  const float* thr;     // global [B][Hd8]
  float* zb;            // [2][8][2][32]
  int Hd8, b0;          // threshold row stride; first sample of the CTA
};
constexpr int kHeadEmitWarps = 2;

// Words [m0, m1), all with NQ live groups of relative slots (NQ = KG - m0 / 4).
template <int KG, int NQ, bool GIVEN>
__device__ __forceinline__ void head_v3_words(HeadV3State<KG>& S, const HeadRing& Rg, const HeadSide& Sd, int lane,
                                              int warp, int m0, int m1) {
  constexpr int KPL = 4 * KG;
  const int Hd = Rg.Hd;
  const int nwords = (Sd.Hd8 + 31) >> 5;
#pragma unroll 1
  for (int m = m0; m < m1; ++m) {
#pragma unroll
    for (int a = 0; a < kHeadS; ++a) {
      S.thr[a] = S.thr_next[a];
      S.vp[a] = 0.f;  // nothing pending at a word start
      // next word's thresholds (global, coalesced; hidden behind this word)
      const int ib = 32 * (m + 1) + lane;
      if (m + 1 < nwords && ib < Sd.Hd8) S.thr_next[a] = Sd.thr[(size_t)(Sd.b0 + kHeadS * warp + a) * Sd.Hd8 + ib];
    }
    const int lend = min(32, Rg.Hd8 - 32 * m);
    const int i0 = 32 * m;
    // ring slots of 8 bits, unrolled (the bit count is padded to a multiple of 8 with dummy bits:
    // zero rows, threshold +inf, so they draw 0 and change nothing)
#pragma unroll 1
    for (int l = 0; l < lend; l += 8) head_v3_group8<KG, NQ, GIVEN>(S, Rg, lane, i0 + l, l);
    // flush the last bit's update (an 8-bit group ends with its rows in wb)
    head_v3_update<KG, 0, 4 * NQ>(S, S.vp, S.wb1, S.wb2);
    // word complete: this lane's bit 32 m + lane.  Later bits only add masked (exactly zero)
    // terms to slot 0, so z2[0] is the final logit and z1[0] the final pre-activation: hand
    // them to the emit warp (double-buffered by word parity).
    const int p = m & 1;
    if (m >= 2) mbar_wait(&Sd.zfree[p], ((m >> 1) - 1) & 1);
#pragma unroll
    for (int a = 0; a < kHeadS; ++a) {
      const int sidx = kHeadS * warp + a;
      float* zrow = Sd.zb + ((size_t)(p * 8 + sidx) * 2) * 32;
      zrow[lane] = S.z2[a][0];
      zrow[32 + lane] = S.z1[a][0];
#pragma unroll
      for (int t = 0; t + 1 < KPL; ++t) {  // shift the relative slots: slot m is complete
        S.z1[a][t] = S.z1[a][t + 1];
        S.z2[a][t] = S.z2[a][t + 1];
      }
      S.z1[a][KPL - 1] = 0.f;
      S.z2[a][KPL - 1] = 0.f;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&Sd.zdone[p]);
  }
}

template <int KG, int P, bool GIVEN>
__device__ __forceinline__ void head_v3_phases(HeadV3State<KG>& S, const HeadRing& Rg, const HeadSide& Sd, int lane,
                                               int warp, int nwords) {
  if constexpr (P < KG) {
    const int m0 = 4 * P, m1 = min(nwords, 4 * P + 4);
    if (m0 < m1) head_v3_words<KG, KG - P, GIVEN>(S, Rg, Sd, lane, warp, m0, m1);
    head_v3_phases<KG, P + 1, GIVEN>(S, Rg, Sd, lane, warp, nwords);
  }
}

// CTA layout: warps [0, nw) consumers (two samples each), warp nw the row producer (TMA),
// warps nw + 1 .. nw + kHeadEmitWarps the emit warps (per completed word: G1 and its fp16
// pair, D pair, spins, log-probability, packed X words).  The consumers only run the serial
// chain and the rank-1 updates; thresholds come precomputed (head_thresholds_kernel).
template <int KG, bool GIVEN>
__global__ void __launch_bounds__(32 * (8 / kHeadS + 1 + kHeadEmitWarps)) head_v3_kernel(const __grid_constant__ HeadV3Args A) {
  constexpr int KPL = 4 * KG;  // word slots per lane
  constexpr int RS = 128 * KG; // staged row stride (floats), both matrices
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int Hd = A.h;          // fast structure: Hd == h
  const int G = A.geo.G;       // bits per ring slot (= 8)
  const int nw = blockDim.x / 32 - 1 - kHeadEmitWarps;
  const int nwords = (Hd + 31) >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + A.geo.R;
  HeadSide Sd;
  Sd.zdone = empty + A.geo.R;
  Sd.zfree = Sd.zdone + 2;
  Sd.Hd8 = (Hd + 7) & ~7;
  Sd.thr = A.thr;
  Sd.b0 = kHeadS * nw * blockIdx.x;  // first sample of this CTA
  float* ring = reinterpret_cast<float*>(smem_raw + A.geo.ring_off);
  Sd.zb = ring + (size_t)A.geo.R * A.geo.slot_floats;
  if (threadIdx.x == 0) {
    for (int r = 0; r < A.geo.R; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], nw);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&Sd.zdone[p], nw);
      mbar_init(&Sd.zfree[p], kHeadEmitWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  ptx::pdl_trigger();
  ptx::pdl_wait();  // thresholds (previous kernel) complete
  const int cta_b0 = Sd.b0;

  if (warp == nw) {  // ---------------- producer warp ----------------
    if (lane == 0) {
      int slot = 0, use = 0;
      for (int g = 0; g < A.geo.ngroups; ++g) {
        if (use > 0) mbar_wait_sleep(&empty[slot], (use - 1) & 1);
        const int i0 = g * G, i1 = i0 + G;  // rows are padded to a multiple of G = 8 (zero rows)
        // every row of the slot belongs to word i0 / 32 (G divides 32): copy its staged length only
        const uint32_t rb = (uint32_t)head_row_floats(KPL, i0 >> 5) * 4u;
        float* dst = ring + (size_t)slot * A.geo.slot_floats;
        mbar_expect_tx(&full[slot], 2u * (uint32_t)(i1 - i0) * rb);
        for (int r = 0; r < i1 - i0; ++r) {
          bulk_g2s(dst + r * RS, A.W1Tq + (size_t)(i0 + r) * RS, rb, &full[slot]);
          bulk_g2s(dst + (G + r) * RS, A.W2cq + (size_t)(i0 + r) * RS, rb, &full[slot]);
        }
        if (++slot == A.geo.R) {
          slot = 0;
          ++use;
        }
      }
    }
    return;
  }
  if (warp > nw) {  // ---------------- emit warps ----------------
    const int e = warp - nw - 1;
    double lp[8 / kHeadEmitWarps];
#pragma unroll
    for (int j = 0; j < 8 / kHeadEmitWarps; ++j) lp[j] = 0.0;
    for (int m = 0; m < nwords; ++m) {
      const int p = m & 1;
      mbar_wait_sleep(&Sd.zdone[p], (m >> 1) & 1);
      const int ib = 32 * m + lane;
#pragma unroll
      for (int j = 0; j < 8 / kHeadEmitWarps; ++j) {
        const int sidx = e + kHeadEmitWarps * j;
        if (sidx < kHeadS * nw) {
          const int b = cta_b0 + sidx;
          const float* zrow = Sd.zb + ((size_t)(p * 8 + sidx) * 2) * 32;
          const float z = zrow[lane], z1 = zrow[32 + lane];
          const bool mine = b < A.B && ib < Hd;
          const float t = mine ? A.thr[(size_t)b * Sd.Hd8 + ib] : INFINITY;
          const int x = (t < z) ? 1 : 0;  // the consumer's draw, recomputed exactly
          if (mine)
            lp[j] += head_emit(b, ib, z, z1, x, A.n, A.h, A.hp, A.np, A.hd1p, A.G1, A.G1h, A.G1l, A.Dh, A.Dl, A.Xf,
                               A.cond);
          const uint32_t word = __ballot_sync(kFull, mine && x);
          if (!GIVEN && b < A.B && lane == 0) A.X[(size_t)b * A.W + m] = word;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&Sd.zfree[p]);
    }
#pragma unroll
    for (int j = 0; j < 8 / kHeadEmitWarps; ++j) {
      const int sidx = e + kHeadEmitWarps * j;
      if (sidx < kHeadS * nw) {
        double v = lp[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        const int b = cta_b0 + sidx;
        if (b < A.B && lane == 0) {
          A.lp_head[b] = v;
          A.Xf[(size_t)b * A.hd1p + Hd] = __float2bfloat16_rn(1.f);  // ones column: gb1 = 1^T dz1
        }
      }
    }
    return;
  }

  // ---------------- consumer warps: samples kHeadS w .. kHeadS w + kHeadS - 1 ----------------
  HeadV3State<KG> S;
#pragma unroll
  for (int t = 0; t < KPL; ++t) {
    const int k = 32 * t + lane;
#pragma unroll
    for (int a = 0; a < kHeadS; ++a) {
      S.z1[a][t] = k < A.h ? A.b1[k] : 0.f;
      S.z2[a][t] = k < Hd ? A.b2[k] : 0.f;
    }
  }
  S.slot = 0;
  S.use = 0;
  S.rows = ring;
  mbar_wait(&full[0], 0);
#pragma unroll
  for (int q = 0; q < KG; ++q) {
    S.wa1[q] = *reinterpret_cast<const float4*>(S.rows + 128 * q + 4 * lane);
    S.wa2[q] = *reinterpret_cast<const float4*>(S.rows + G * RS + 128 * q + 4 * lane);
    S.wb1[q] = make_float4(0.f, 0.f, 0.f, 0.f);  // "pending" rows of the first bit (0 x 0, never NaN)
    S.wb2[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  S.dg = S.wa1[0].x;
#pragma unroll
  for (int a = 0; a < kHeadS; ++a) S.thr_next[a] = A.thr[(size_t)(cta_b0 + kHeadS * warp + a) * Sd.Hd8 + lane];
  const HeadRing Rg{full, empty, ring, G, A.geo.R, A.geo.slot_floats, Hd, (Hd + 7) & ~7};
#ifdef VQMC_HEAD_PROF
  const long long tstart = clock64();
#endif
  head_v3_phases<KG, 0, GIVEN>(S, Rg, Sd, lane, warp, nwords);
#ifdef VQMC_HEAD_PROF
  if (lane == 0 && (blockIdx.x % 64) == 0 && warp == 0)
    printf("HEADPROF block %d warp %d total %lld\n", blockIdx.x, warp, clock64() - tstart);
#endif
  // the last slot
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[S.slot]);
}

// ===========================================================================
// Head sampler v4 (fast structure; staging layout: head4.cuh).
//
// One CTA = 8 consumer warps (one sample each: the N = 8 of the tensor-core updates) + a TMA
// producer warp.  Per 32-bit word m:
//   chain   lane l owns bit 32m + l: z1c / z2c are unit / output 32m + l; the word's own 32 x 32
//           blocks (TRI, staged in shared memory) give the in-word rank-1 updates.  Bit l' on
//           lane l': x = [thr < z2c], g = relu(z1c + x W1[i][i]) (both candidates precomputed),
//           sent in one shuffle (x in the sign bit); every lane then applies 2 FMAs.  Serial
//           chain per bit: compare, select, shuffle, fma.
//   emit    every lane writes its own bit's outputs (G1 + fp16 pair, D pair, spins, log-prob
//           term, conditionals) and the warp ballots the packed spin word.
//   update  x and the fp16 pair of g of the word's 32 bits x 8 samples are staged in shared
//           memory; every warp applies them to the accumulator tiles it owns (tile j of 16 slots
//           -> warp j % 8): z1 += W1[s][word] X (2 MMAs per k-step: x is exact in fp16), z2 +=
//           W2[s][word] (G_hi + G_lo) with the W2 pair (3 MMAs): mma.sync m16n8k16, fp32
//           accumulators in registers (rows = slots, columns = the CTA's 8 samples).  The A
//           operands stream through a ring of 16 KB chunks (TMA bulk copies issued ahead by the
//           producer warp, which also double-buffers the TRI blocks).
//   exchange the owners of the next word's two tiles write them (16 slots x 8 samples, z1 and
//           z2) to shared memory; each chain warp reads its sample's 32 slots.
// Work per bit drops from ~100 dependent FMA/LDS instructions per warp (v3) to the short chain;
// the rank-32 updates run on the tensor cores once per word.
// ===========================================================================
constexpr int kH4Warps = 8;          // consumer warps = samples per CTA
constexpr int kH4Ring = 6;           // 16 KB A-operand chunks in flight
constexpr int kH4Chunk = 16384;
constexpr int kH4Tri = 8192;         // bytes of one word's TRI block ([64][32] floats)
constexpr int kH4BStride = 40;       // halves per sample row of the staged B operand (conflict-free)

struct HeadV4Args {
  int B, n, h, W, nwords, T, Hd8;  // T = 16-slot tiles of the head (ceil(h / 16))
  const __half* AF;
  const float* TRI;
  const float* b1;
  const float* b2;
  uint32_t* X;
  float* G1;
  __half* G1h;
  __half* G1l;
  int hp;
  __half* Dh;
  __half* Dl;
  int np;
  __nv_bfloat16* Xf;
  int hd1p;
  double* lp_head;
  double* cond;
  const float* thr;  // [B][Hd8] logit thresholds (head_thresholds_kernel)
};

__device__ __forceinline__ void h4_mma(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void h4_bar_consumers() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Shared memory: mbarriers @0 | Zx [2][32][8] f32 @128 | B staging 3 x [8][40] f16 @2176 |
// TRI [2][64][32] f32 @4096 | ring [kH4Ring][16 KB] @20480.
template <int KG, bool GIVEN>
__global__ void __launch_bounds__(32 * (kH4Warps + 1), 1) head_v4_kernel(const __grid_constant__ HeadV4Args A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + kH4Ring;
  uint64_t* tfull = empty + kH4Ring;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  float* Zx = reinterpret_cast<float*>(smem_raw + 128);            // [2][32][8] (2 KB)
  __half* Bx = reinterpret_cast<__half*>(smem_raw + 2176);         // [8][40] x
  __half* Bgh = Bx + 8 * kH4BStride;                               // [8][40] g hi
  __half* Bgl = Bgh + 8 * kH4BStride;                              // [8][40] g lo (ends at 4096)
  float* tri_s = reinterpret_cast<float*>(smem_raw + 4096);        // [2][64][32]
  unsigned char* ring = smem_raw + 4096 + 2 * kH4Tri;              // [kH4Ring][16 KB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = A.h, nwords = A.nwords, T = A.T;
  const int cta_b0 = kH4Warps * blockIdx.x;
  if (threadIdx.x == 0) {
    for (int r = 0; r < kH4Ring; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], kH4Warps);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&tfull[p], 1);
      mbar_init(&tempty[p], kH4Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  ptx::pdl_trigger();
  ptx::pdl_wait();  // thresholds (previous kernel) complete
  const int rounds = (T + 7) >> 3;

  if (warp == kH4Warps) {  // ---------------- producer: TRI blocks and A-operand chunks ----------------
    if (lane == 0) {
      int slot = 0, use = 0;
      auto tri_copy = [&](int m) {
        const int p = m & 1;
        if (m >= 2) mbar_wait_sleep(&tempty[p], ((m >> 1) - 1) & 1);
        mbar_expect_tx(&tfull[p], kH4Tri);
        bulk_g2s(tri_s + p * 2048, A.TRI + (size_t)m * 2048, kH4Tri, &tfull[p]);
      };
      tri_copy(0);
      for (int m = 0; m + 1 < nwords; ++m) {
        tri_copy(m + 1);
        for (int r = (2 * m + 2) >> 3; r < rounds; ++r) {
          for (int z = 0; z < 2; ++z) {
            if (use > 0) mbar_wait_sleep(&empty[slot], (use - 1) & 1);
            mbar_expect_tx(&full[slot], kH4Chunk);
            bulk_g2s(ring + (size_t)slot * kH4Chunk, A.AF + head4_chunk_off(KG, m, r, z), kH4Chunk, &full[slot]);
            if (++slot == kH4Ring) {
              slot = 0;
              ++use;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumer warp `warp`: sample b ----------------
  const int w = warp, b = cta_b0 + w;
  const int g = lane >> 2, t4 = lane & 3;
  float acc1[KG][4], acc2[KG][4];  // tiles j = 8 r + w: rows g, g + 8 of the tile, columns 2 t4, 2 t4 + 1
#pragma unroll
  for (int r = 0; r < KG; ++r) {
    const int s0 = 16 * (8 * r + w) + g, s1 = s0 + 8;
    const float a0 = s0 < h ? A.b1[s0] : 0.f, a1 = s1 < h ? A.b1[s1] : 0.f;
    const float c0 = s0 < h ? A.b2[s0] : 0.f, c1 = s1 < h ? A.b2[s1] : 0.f;
    acc1[r][0] = acc1[r][1] = a0;
    acc1[r][2] = acc1[r][3] = a1;
    acc2[r][0] = acc2[r][1] = c0;
    acc2[r][2] = acc2[r][3] = c1;
  }
  const bool bvalid = b < A.B;
  float thr = (bvalid && lane < A.Hd8) ? A.thr[(size_t)b * A.Hd8 + lane] : INFINITY;
  double lp = 0.0;
  int slot = 0, use = 0;
  for (int m = 0; m < nwords; ++m) {
    // ---- exchange: the owners of tiles 2m, 2m + 1 publish word m's slots ----
    {
      const int r = (2 * m) >> 3;
      const bool own0 = w == ((2 * m) & 7), own1 = w == ((2 * m + 1) & 7);
      if (own0 || own1) {
        const int base = own1 ? 16 : 0;
#pragma unroll
        for (int rr = 0; rr < KG; ++rr) {
          if (rr == r) {
            Zx[(base + g) * 8 + 2 * t4] = acc1[rr][0];
            Zx[(base + g) * 8 + 2 * t4 + 1] = acc1[rr][1];
            Zx[(base + g + 8) * 8 + 2 * t4] = acc1[rr][2];
            Zx[(base + g + 8) * 8 + 2 * t4 + 1] = acc1[rr][3];
            Zx[256 + (base + g) * 8 + 2 * t4] = acc2[rr][0];
            Zx[256 + (base + g) * 8 + 2 * t4 + 1] = acc2[rr][1];
            Zx[256 + (base + g + 8) * 8 + 2 * t4] = acc2[rr][2];
            Zx[256 + (base + g + 8) * 8 + 2 * t4 + 1] = acc2[rr][3];
          }
        }
      }
    }
    h4_bar_consumers();
    float z1c = Zx[lane * 8 + w], z2c = Zx[256 + lane * 8 + w];
    // ---- serial chain over the word's 32 bits ----
    const int p = m & 1;
    mbar_wait(&tfull[p], (m >> 1) & 1);
    const float* tw = tri_s + p * 2048 + lane;  // tw[32 l] = W1[32m + lane][32m + l], tw[32 (32 + l)] = W2[...]
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const float t1 = tw[32 * l], t2 = tw[32 * (32 + l)];
      const float g0 = fmaxf(z1c, 0.f), g1 = fmaxf(z1c + t1, 0.f);  // (on lane l: t1 = W1[i][i])
      float v = (thr < z2c) ? -g1 : g0;                             // x in the sign bit
      v = __shfl_sync(kFull, v, l);
      const float xf = (__float_as_uint(v) >> 31) ? 1.f : 0.f;
      z1c = fmaf(xf, t1, z1c);           // lanes >= l (t1 = 0 above this lane's diagonal)
      z2c = fmaf(fabsf(v), t2, z2c);     // lanes > l
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[p]);
    const bool x = thr < z2c;  // this lane's bit (its logit no longer changes)
    const float gl = fmaxf(z1c, 0.f);
    // ---- outputs of the word's bits (one per lane) ----
    {
      const int ib = 32 * m + lane;
      const bool mine = bvalid && ib < h;
      if (mine)
        lp += head_emit(b, ib, z2c, z1c, x ? 1 : 0, A.n, h, A.hp, A.np, A.hd1p, A.G1, A.G1h, A.G1l, A.Dh, A.Dl, A.Xf,
                        A.cond);
      const uint32_t word = __ballot_sync(kFull, mine && x);
      if (!GIVEN && bvalid && lane == 0) A.X[(size_t)b * A.W + m] = word;
    }
    if (m + 1 == nwords) break;
    // ---- stage B = (x, g_hi, g_lo) of the word, [sample][bit] ----
    {
      __half gh, glo;
      ptx::split_f16(gl, gh, glo);
      Bx[w * kH4BStride + lane] = __float2half_rn(x ? 1.f : 0.f);
      Bgh[w * kH4BStride + lane] = gh;
      Bgl[w * kH4BStride + lane] = glo;
      const int ib = 32 * (m + 1) + lane;  // next word's threshold (latency hidden by the MMAs)
      thr = (bvalid && ib < A.Hd8) ? A.thr[(size_t)b * A.Hd8 + ib] : INFINITY;
    }
    h4_bar_consumers();
    uint32_t bx[2][2], bh[2][2], bl[2][2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int o = g * kH4BStride + 16 * ks + 2 * t4;
      bx[ks][0] = *reinterpret_cast<const uint32_t*>(Bx + o);
      bx[ks][1] = *reinterpret_cast<const uint32_t*>(Bx + o + 8);
      bh[ks][0] = *reinterpret_cast<const uint32_t*>(Bgh + o);
      bh[ks][1] = *reinterpret_cast<const uint32_t*>(Bgh + o + 8);
      bl[ks][0] = *reinterpret_cast<const uint32_t*>(Bgl + o);
      bl[ks][1] = *reinterpret_cast<const uint32_t*>(Bgl + o + 8);
    }
    // ---- rank-32 updates of the later tiles (the producer's chunk order: r, then z) ----
    const int r0 = (2 * m + 2) >> 3;
#pragma unroll
    for (int r = 0; r < KG; ++r) {
      if (r < r0 || r >= rounds) continue;
      const int j = 8 * r + w;
      const bool live = j >= 2 * m + 2 && j < T;
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        mbar_wait(&full[slot], use & 1);
        if (live) {
          const unsigned char* cb = ring + (size_t)slot * kH4Chunk + (size_t)w * 2048 + lane * 16;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint4 ah = *reinterpret_cast<const uint4*>(cb + ks * 1024);
            const uint4 al = *reinterpret_cast<const uint4*>(cb + ks * 1024 + 512);
            if (z == 0) {
              h4_mma(acc1[r], ah, bx[ks][0], bx[ks][1]);
              h4_mma(acc1[r], al, bx[ks][0], bx[ks][1]);
            } else {
              h4_mma(acc2[r], ah, bh[ks][0], bh[ks][1]);
              h4_mma(acc2[r], ah, bl[ks][0], bl[ks][1]);
              h4_mma(acc2[r], al, bh[ks][0], bh[ks][1]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == kH4Ring) {
          slot = 0;
          ++use;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lp += __shfl_xor_sync(kFull, lp, o);
  if (bvalid && lane == 0) {
    A.lp_head[b] = lp;
    A.Xf[(size_t)b * A.hd1p + h] = __float2bfloat16_rn(1.f);  // ones column: gb1 = 1^T dz1
  }
}

// ===========================================================================
// Head sampler v5: v4's arithmetic with the chain and the tensor-core updates on separate warps.
//
// In v4 every warp both runs its sample's serial chain and owns tiles of the rank-32 updates, so
// each word pays chain + all of the word's MMAs + two CTA barriers.  But the next word's chain
// only needs ITS OWN 32 slots (tiles 2m + 2, 2m + 3) updated; the updates of the later tiles can
// run while that chain runs.  v5: 8 chain warps (one sample each) and 8 tile warps (tile j is
// owned by warp j mod 8, accumulators for all 8 samples), synchronised by mbarriers:
//   tile warps:  wait B(m) -> MMAs of round r0 = (2m + 2) / 8 (holds tiles 2m + 2, 2m + 3) ->
//                their owners publish Z(m + 1) -> the remaining rounds of word m
//   chain warps: wait Z(m) -> 32-bit chain -> outputs -> stage B(m) = (x, g_hi, g_lo)
// so the critical path per word is chain + one round of MMAs instead of chain + all rounds.
// Z and B are double-buffered by word parity; the producer warp streams TRI and A chunks as in v4.
// Shared memory: mbarriers @0 (256 B) | Zx [2][2][32][8] f32 @256 (4 KB) | B staging
// [2][3][8][40] f16 @4352 (3840 B) | TRI [2][64][32] f32 @8192 | ring [kH4Ring][16 KB] @24576.
// ===========================================================================
constexpr int kH5Smem = 24576 + kH4Ring * kH4Chunk;
#ifdef VQMC_TAIL_TRACE
// per CTA: [0] start, per word m < 15: [1 + 4m] Z(m) received, [2 + 4m] chain done, [3 + 4m] outputs
// done (chain warp 0), [4 + 4m] Z(m) published (its first owner); [63] chain warp 0 end
__device__ unsigned long long g_head_trace[128 * 64];
__device__ __forceinline__ unsigned long long head_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HEAD_TRACE(cond, slot) \
  if ((cond) && blockIdx.x < 128) g_head_trace[blockIdx.x * 64 + (slot)] = head_gtime()
#else
#define HEAD_TRACE(cond, slot)
#endif

template <int KG, bool GIVEN>
__global__ void __launch_bounds__(32 * (2 * kH4Warps + 1), 1) head_v5_kernel(const __grid_constant__ HeadV4Args A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [kH4Ring] A chunks
  uint64_t* empty = full + kH4Ring;                          // [kH4Ring]
  uint64_t* tfull = empty + kH4Ring;                         // [2] TRI blocks
  uint64_t* tempty = tfull + 2;                              // [2]
  uint64_t* zfull = tempty + 2;                              // [2] Z(m) published (64 lanes)
  uint64_t* zempty = zfull + 2;                              // [2] Z(m) read by the chain warps (8)
  uint64_t* bfull = zempty + 2;                              // [2] B(m) staged (256 lanes)
  uint64_t* bempty = bfull + 2;                              // [2] B(m) read by the tile warps (8)
  float* Zx = reinterpret_cast<float*>(smem_raw + 256);      // [2][2][32][8]
  __half* Bs = reinterpret_cast<__half*>(smem_raw + 4352);   // [2][3][8][kH4BStride]
  float* tri_s = reinterpret_cast<float*>(smem_raw + 8192);  // [2][64][32]
  unsigned char* ring = smem_raw + 24576;                    // [kH4Ring][16 KB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = A.h, nwords = A.nwords, T = A.T;
  const int cta_b0 = kH4Warps * blockIdx.x;
  if (threadIdx.x == 0) {
    for (int r = 0; r < kH4Ring; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], kH4Warps);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&tfull[p], 1);
      mbar_init(&tempty[p], kH4Warps);
      mbar_init(&zfull[p], 64);
      mbar_init(&zempty[p], kH4Warps);
      mbar_init(&bfull[p], 32 * kH4Warps);
      mbar_init(&bempty[p], kH4Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  ptx::pdl_trigger();
  ptx::pdl_wait();  // thresholds (previous kernel) complete
  HEAD_TRACE(threadIdx.x == 0, 0);
  const int rounds = (T + 7) >> 3;

  if (warp == 2 * kH4Warps) {  // ---------------- producer: TRI blocks and A-operand chunks ----------------
    if (lane == 0) {
      int slot = 0, use = 0;
      auto tri_copy = [&](int m) {
        const int p = m & 1;
        if (m >= 2) mbar_wait_sleep(&tempty[p], ((m >> 1) - 1) & 1);
        mbar_expect_tx(&tfull[p], kH4Tri);
        bulk_g2s(tri_s + p * 2048, A.TRI + (size_t)m * 2048, kH4Tri, &tfull[p]);
      };
      tri_copy(0);
      for (int m = 0; m + 1 < nwords; ++m) {
        tri_copy(m + 1);
        for (int r = (2 * m + 2) >> 3; r < rounds; ++r) {
          for (int z = 0; z < 2; ++z) {
            if (use > 0) mbar_wait_sleep(&empty[slot], (use - 1) & 1);
            mbar_expect_tx(&full[slot], kH4Chunk);
            bulk_g2s(ring + (size_t)slot * kH4Chunk, A.AF + head4_chunk_off(KG, m, r, z), kH4Chunk, &full[slot]);
            if (++slot == kH4Ring) {
              slot = 0;
              ++use;
            }
          }
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t4 = lane & 3;
  if (warp >= kH4Warps) {  // ---------------- tile warp: tiles j = 8 r + w, all 8 samples ----------------
    const int w = warp - kH4Warps;
    float acc1[KG][4], acc2[KG][4];  // rows g, g + 8 of the tile, columns (samples) 2 t4, 2 t4 + 1
#pragma unroll
    for (int r = 0; r < KG; ++r) {
      const int s0 = 16 * (8 * r + w) + g, s1 = s0 + 8;
      const float a0 = s0 < h ? A.b1[s0] : 0.f, a1 = s1 < h ? A.b1[s1] : 0.f;
      const float c0 = s0 < h ? A.b2[s0] : 0.f, c1 = s1 < h ? A.b2[s1] : 0.f;
      acc1[r][0] = acc1[r][1] = a0;
      acc1[r][2] = acc1[r][3] = a1;
      acc2[r][0] = acc2[r][1] = c0;
      acc2[r][2] = acc2[r][3] = c1;
    }
    // publish Z(m): the owners of tiles 2m, 2m + 1 write their [slot][sample] values
    auto publish = [&](int m) {
      const bool own0 = w == ((2 * m) & 7), own1 = w == ((2 * m + 1) & 7);
      if (!own0 && !own1) return;
      const int pz = m & 1, r = (2 * m) >> 3, base = own1 ? 16 : 0;
      if (m >= 2) mbar_wait(&zempty[pz], ((m >> 1) - 1) & 1);
      float* zx = Zx + pz * 512;
#pragma unroll
      for (int rr = 0; rr < KG; ++rr) {
        if (rr == r) {
          zx[(base + g) * 8 + 2 * t4] = acc1[rr][0];
          zx[(base + g) * 8 + 2 * t4 + 1] = acc1[rr][1];
          zx[(base + g + 8) * 8 + 2 * t4] = acc1[rr][2];
          zx[(base + g + 8) * 8 + 2 * t4 + 1] = acc1[rr][3];
          zx[256 + (base + g) * 8 + 2 * t4] = acc2[rr][0];
          zx[256 + (base + g) * 8 + 2 * t4 + 1] = acc2[rr][1];
          zx[256 + (base + g + 8) * 8 + 2 * t4] = acc2[rr][2];
          zx[256 + (base + g + 8) * 8 + 2 * t4 + 1] = acc2[rr][3];
        }
      }
      mbar_arrive(&zfull[pz]);
      HEAD_TRACE(own0 && lane == 0 && m < 15, 4 + 4 * m);
    };
    publish(0);
    int slot = 0, use = 0;
    for (int m = 0; m + 1 < nwords; ++m) {
      const int pb = m & 1;
      mbar_wait(&bfull[pb], (m >> 1) & 1);
      const __half* Bx = Bs + pb * (3 * 8 * kH4BStride);
      const __half* Bgh = Bx + 8 * kH4BStride;
      const __half* Bgl = Bgh + 8 * kH4BStride;
      uint32_t bx[2][2], bh[2][2], bl[2][2];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int o = g * kH4BStride + 16 * ks + 2 * t4;
        bx[ks][0] = *reinterpret_cast<const uint32_t*>(Bx + o);
        bx[ks][1] = *reinterpret_cast<const uint32_t*>(Bx + o + 8);
        bh[ks][0] = *reinterpret_cast<const uint32_t*>(Bgh + o);
        bh[ks][1] = *reinterpret_cast<const uint32_t*>(Bgh + o + 8);
        bl[ks][0] = *reinterpret_cast<const uint32_t*>(Bgl + o);
        bl[ks][1] = *reinterpret_cast<const uint32_t*>(Bgl + o + 8);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bempty[pb]);
      const int r0 = (2 * m + 2) >> 3;
#pragma unroll
      for (int r = 0; r < KG; ++r) {
        if (r < r0 || r >= rounds) continue;
        const int j = 8 * r + w;
        const bool live = j >= 2 * m + 2 && j < T;
        // the round's two chunks (z = 0: W1 -> acc1, z = 1: W2 -> acc2) feed independent accumulator
        // chains: wait for both, then interleave their MMAs (same per-accumulator order as v4)
        const int s1 = slot + 1 == kH4Ring ? 0 : slot + 1, u1 = slot + 1 == kH4Ring ? use + 1 : use;
        mbar_wait(&full[slot], use & 1);
        mbar_wait(&full[s1], u1 & 1);
        if (live) {
          const unsigned char* c0 = ring + (size_t)slot * kH4Chunk + (size_t)w * 2048 + lane * 16;
          const unsigned char* c1 = ring + (size_t)s1 * kH4Chunk + (size_t)w * 2048 + lane * 16;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint4 ah = *reinterpret_cast<const uint4*>(c0 + ks * 1024);
            const uint4 al = *reinterpret_cast<const uint4*>(c0 + ks * 1024 + 512);
            const uint4 vh = *reinterpret_cast<const uint4*>(c1 + ks * 1024);
            const uint4 vl = *reinterpret_cast<const uint4*>(c1 + ks * 1024 + 512);
            h4_mma(acc1[r], ah, bx[ks][0], bx[ks][1]);
            h4_mma(acc2[r], vh, bh[ks][0], bh[ks][1]);
            h4_mma(acc1[r], al, bx[ks][0], bx[ks][1]);
            h4_mma(acc2[r], vh, bl[ks][0], bl[ks][1]);
            h4_mma(acc2[r], vl, bh[ks][0], bh[ks][1]);
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[slot]);
          mbar_arrive(&empty[s1]);
        }
        slot = s1 + 1 == kH4Ring ? 0 : s1 + 1;
        use = s1 + 1 == kH4Ring ? u1 + 1 : u1;
        if (r == r0) publish(m + 1);  // tiles 2m + 2, 2m + 3 now hold every update of words <= m
      }
    }
    return;
  }

  // ---------------- chain warp `warp`: sample b ----------------
  const int w = warp, b = cta_b0 + w;
  const bool bvalid = b < A.B;
  float thr = (bvalid && lane < A.Hd8) ? A.thr[(size_t)b * A.Hd8 + lane] : INFINITY;
  double lp = 0.0;
  for (int m = 0; m < nwords; ++m) {
    const int pz = m & 1;
    mbar_wait(&zfull[pz], (m >> 1) & 1);
    HEAD_TRACE(w == 0 && lane == 0 && m < 15, 1 + 4 * m);
    float z1c = Zx[pz * 512 + lane * 8 + w], z2c = Zx[pz * 512 + 256 + lane * 8 + w];
    __syncwarp();
    if (lane == 0) mbar_arrive(&zempty[pz]);
    // ---- serial chain over the word's 32 bits ----
    const int p = m & 1;
    mbar_wait(&tfull[p], (m >> 1) & 1);
    const float* tw = tri_s + p * 2048 + lane;  // tw[32 l] = W1[32m + lane][32m + l], tw[32 (32 + l)] = W2[...]
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const float t1 = tw[32 * l], t2 = tw[32 * (32 + l)];
      const float g0 = fmaxf(z1c, 0.f), g1 = fmaxf(z1c + t1, 0.f);  // (on lane l: t1 = W1[i][i])
      float v = (thr < z2c) ? -g1 : g0;                             // x in the sign bit
      v = __shfl_sync(kFull, v, l);
      const float xf = (__float_as_uint(v) >> 31) ? 1.f : 0.f;
      z1c = fmaf(xf, t1, z1c);           // lanes >= l (t1 = 0 above this lane's diagonal)
      z2c = fmaf(fabsf(v), t2, z2c);     // lanes > l
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[p]);
    HEAD_TRACE(w == 0 && lane == 0 && m < 15, 2 + 4 * m);
    const bool x = thr < z2c;  // this lane's bit (its logit no longer changes)
    const float gl = fmaxf(z1c, 0.f);
    if (m + 1 < nwords) {  // ---- stage B(m) = (x, g_hi, g_lo), [sample][bit]: the tile warps wait on it ----
      const int pb = m & 1;
      if (m >= 2) mbar_wait(&bempty[pb], ((m >> 1) - 1) & 1);
      __half* Bx = Bs + pb * (3 * 8 * kH4BStride);
      __half gh, glo;
      ptx::split_f16(gl, gh, glo);
      Bx[w * kH4BStride + lane] = __float2half_rn(x ? 1.f : 0.f);
      Bx[8 * kH4BStride + w * kH4BStride + lane] = gh;
      Bx[16 * kH4BStride + w * kH4BStride + lane] = glo;
      mbar_arrive(&bfull[pb]);
    }
    // ---- outputs of the word's bits (one per lane; off the critical path) ----
    {
      const int ib = 32 * m + lane;
      const bool mine = bvalid && ib < h;
      if (mine)
        lp += head_emit(b, ib, z2c, z1c, x ? 1 : 0, A.n, h, A.hp, A.np, A.hd1p, A.G1, A.G1h, A.G1l, A.Dh, A.Dl, A.Xf,
                        A.cond);
      const uint32_t word = __ballot_sync(kFull, mine && x);
      if (!GIVEN && bvalid && lane == 0) A.X[(size_t)b * A.W + m] = word;
      const int ibn = 32 * (m + 1) + lane;  // next word's threshold
      thr = (bvalid && ibn < A.Hd8) ? A.thr[(size_t)b * A.Hd8 + ibn] : INFINITY;
    }
    HEAD_TRACE(w == 0 && lane == 0 && m < 15, 3 + 4 * m);
  }
  HEAD_TRACE(w == 0 && lane == 0, 63);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lp += __shfl_xor_sync(kFull, lp, o);
  if (bvalid && lane == 0) {
    A.lp_head[b] = lp;
    A.Xf[(size_t)b * A.hd1p + h] = __float2bfloat16_rn(1.f);  // ones column: gb1 = 1^T dz1
  }
}

// Padded, completion-ordered copies of the head blocks (refreshed after every update):
//   W1Tp[j][k] = W1m[k][j]           j < Hd, k < h (row stride hp)
//   W2cp[c][i] = W2m[i][comp_k[c]]   c < h,  i < Hd (row stride Hdp)
// perm: the v3 relative staging order (head_rel_pos) when the fast structure holds, else identity.
__global__ void head_pack_kernel(int h, int Hd, int hp, int Hdp, int perm, const float* __restrict__ W1T,
                                 const float* __restrict__ W2, const int* __restrict__ comp_k,
                                 float* __restrict__ W1Tp, float* __restrict__ W2cp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)Hd * hp, n2 = (int64_t)h * Hdp;
  if (t < n1) {
    const int j = (int)(t / hp), k = (int)(t % hp);
    if (!perm) {
      W1Tp[t] = k < h ? W1T[(size_t)j * h + k] : 0.f;
    } else {  // v3: row j in the relative order of word j / 32; units of earlier words are not staged
      const int m = j >> 5, tt = (k >> 5) - m;
      if (tt >= 0) W1Tp[(size_t)j * hp + head_rel_pos(tt, k & 31)] = k < h ? W1T[(size_t)j * h + k] : 0.f;
    }
  } else if (t < n1 + n2) {
    const int64_t u = t - n1;
    const int c = (int)(u / Hdp), i = (int)(u % Hdp);
    if (!perm) {
      W2cp[u] = i < Hd ? W2[(size_t)i * h + comp_k[c]] : 0.f;
    } else {  // v3: row c (= bit c, fast structure) in the relative order of word c / 32
      const int m = c >> 5, tt = (i >> 5) - m;
      if (tt >= 0) W2cp[(size_t)c * Hdp + head_rel_pos(tt, i & 31)] = i < Hd ? W2[(size_t)i * h + comp_k[c]] : 0.f;
    }
  }
}

// v4 staging (head4.cuh) from the live parameters: every W1T[j][k] (j < Hd) and head W2[i][k]
// (i < Hd) lands in TRI or AF; masked entries (zero) and earlier-word slots are never stored.
__global__ void head4_pack_kernel(int h, int Hd, Head4Stage S, const float* __restrict__ W1T,
                                  const float* __restrict__ W2) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)Hd * h;
  if (t < n1) {
    const int j = (int)(t / h), k = (int)(t % h);
    head4_put_w1(S, j, k, W1T[t]);
  } else if (t < 2 * n1) {
    const int64_t u = t - n1;
    const int i = (int)(u / h), k = (int)(u % h);
    head4_put_w2(S, i, k, W2[u]);
  }
}

static int head_kpl(int h) {
  const int k = (h + 31) / 32;
  return k <= 1 ? 1 : k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
}
static int head_G(int kpl) { return kpl >= 32 ? 8 : 16; }

// Row lengths are padded to 32 * KPL floats so the per-bit updates need no bounds predicates.
static HeadGeom head_geometry(const Handle* H) {
  const Layout& L = H->L;
  HeadGeom g{};
  const int kpl = head_kpl(L.h);
  g.hp = 32 * kpl;
  g.Hdp = H->head_fast ? 32 * kpl : 32 * ((L.Hd + 31) / 32);
  g.R = 3;
  for (int G = head_G(kpl); G >= 1; G >>= 1) {
    int cmax = 0;
    for (int i0 = 0; i0 < L.Hd; i0 += G) {
      const int i1 = std::min(L.Hd, i0 + G);
      cmax = std::max(cmax, H->comp_off_host[i1] - H->comp_off_host[i0]);
    }
    g.G = G;
    g.cmax = cmax;
    g.slot_floats = G * g.hp + cmax * g.Hdp;
    g.slot_floats = (g.slot_floats + 31) & ~31;  // 128-byte aligned slots
    const size_t head = ((16 * g.R + 4 * (L.Hd + 1 + L.h) + 127) / 128) * 128;
    g.smem = head + (size_t)g.R * g.slot_floats * 4;
    if (g.smem <= 225 * 1024) break;
    if (G == 1) throw InvalidArgument("head sampler shared-memory ring does not fit (hidden width too large)");
  }
  g.ngroups = (L.Hd + g.G - 1) / g.G;
  return g;
}

void launch_head_pack(Handle* H) {
  const Layout& L = H->L;
  if (H->head_v4) {
    const int64_t total = 2 * (int64_t)L.Hd * L.h;
    KScope ks(H, "head_pack");
    head4_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(L.h, L.Hd, H->h4, H->P + L.off_w1t,
                                                                             H->P + L.off_w2);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
    return;
  }
  const int hp = H->head_hpk, Hdp = H->head_Hdp;
  const int64_t total = (int64_t)L.Hd * hp + (int64_t)L.h * Hdp;
  KScope ks(H, "head_pack");
  head_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(
      L.h, L.Hd, hp, Hdp, H->head_fast ? 1 : 0, H->P + L.off_w1t, H->P + L.off_w2, H->d_comp_k, H->W1Tp, H->W2cp);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

template <int KPL, bool FAST, bool GIVEN>
static void head_v2_launch(Handle* H, int B, const double* uni, RngSpec rng, double* cond) {
  const Layout& L = H->L;
  const HeadGeom geo = head_geometry(H);
  ensure_smem_attr((const void*)head_v2_kernel<KPL, FAST, GIVEN>, geo.smem);
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, H->device);
  const int nw = std::max(1, std::min(8, (B + dev_sms - 1) / dev_sms));  // <= 8 sample warps + producer
  const int grid = (B + nw - 1) / nw;
  KScope ks(H, GIVEN ? "head_given" : "head_sample");
  head_v2_kernel<KPL, FAST, GIVEN><<<grid, 32 * (nw + 1), geo.smem, H->stream>>>(
      B, L.n, L.h, L.Hd, L.W, geo, H->W1Tp, H->W2cp, H->P + L.off_b1, H->P + L.off_b2, H->d_comp_k,
      H->d_comp_off, uni, rng, H->w1skip ? 1 : 0, H->X, H->G1, H->G1h, H->G1l, H->hp18, H->Dh,
      H->Dl, H->np8, H->Xfb, H->hd18, H->lp_head, cond);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

template <int KPL>
static void head_v2_dispatch(Handle* H, int B, const double* uni, RngSpec rng, bool given, double* cond) {
  if (H->head_fast) {
    if (given) head_v2_launch<KPL, true, true>(H, B, uni, rng, cond);
    else head_v2_launch<KPL, true, false>(H, B, uni, rng, cond);
  } else {
    if (given) head_v2_launch<KPL, false, true>(H, B, uni, rng, cond);
    else head_v2_launch<KPL, false, false>(H, B, uni, rng, cond);
  }
}

// v3 geometry: slot = G bits x (W1 row + W2 row) of 128 KG floats each.
static HeadGeom head_v3_geometry(const Handle* H) {
  const Layout& L = H->L;
  HeadGeom g{};
  const int RS = H->head_hpk;  // 128 * KG
  const int nwords = (L.Hd + 31) / 32;
  g.hp = RS;
  g.Hdp = RS;
  g.cmax = 1;
  g.G = 8;  // one ring slot = 8 bits (the unrolled group)
  g.slot_floats = 2 * g.G * RS;
  g.ring_off = 256;  // full[R] + empty[R] + zdone[2] + zfree[2] mbarriers (<= 16)
  const size_t side = (size_t)2 * 8 * 2 * 32 * 4;  // (z2, z1) hand-off to the emit warps
  (void)nwords;
  const size_t limit = 227 * 1024;
  g.R = 0;
  for (int R = 6; R >= 2; --R) {
    g.smem = g.ring_off + (size_t)R * g.slot_floats * 4 + side;
    if (g.smem <= limit) {
      g.R = R;
      break;
    }
  }
  if (!g.R) throw InvalidArgument("head sampler shared-memory ring does not fit (hidden width too large)");
  g.ngroups = (L.Hd + g.G - 1) / g.G;  // rows padded to Hd8 = 8 ngroups
  return g;
}

template <int KG, bool GIVEN>
static void head_v3_launch(Handle* H, int B, const double* uni, RngSpec rng, double* cond) {
  const Layout& L = H->L;
  const HeadGeom geo = head_v3_geometry(H);
  ensure_smem_attr((const void*)head_v3_kernel<KG, GIVEN>, geo.smem);
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, H->device);
  const int groups = (B + kHeadS - 1) / kHeadS;  // consumer warps needed
  // <= 8 / kHeadS consumer warps (8 samples per CTA: the emit hand-off buffer) + producer + emit warps
  const int nw = std::max(1, std::min(8 / kHeadS, (groups + dev_sms - 1) / dev_sms));
  const int grid = (groups + nw - 1) / nw;
  const int Hd8 = (L.Hd + 7) & ~7;
  {
    KScope ks(H, "head_thresholds");
    const int64_t total = (int64_t)B * (Hd8 / 4);
    launch_k(H, head_thresholds_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, B, L.Hd, Hd8, L.W, uni,
             rng, H->X, GIVEN ? 1 : 0, H->thr);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  KScope ks(H, GIVEN ? "head_given" : "head_sample");
  const HeadV3Args args{B,      L.n,     L.h,    L.W,    geo,     H->W1Tp,  H->W2cp, H->P + L.off_b1,
                        H->P + L.off_b2, uni, rng, H->X, H->G1, H->G1h, H->G1l, H->hp18, H->Dh, H->Dl, H->np8,
                        H->Xfb, H->hd18, H->lp_head, cond, H->thr};
  launch_k(H, head_v3_kernel<KG, GIVEN>, dim3(grid), dim3(32 * (nw + 1 + kHeadEmitWarps)), geo.smem, args);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

template <int KG, bool GIVEN>
static void head_v4_launch(Handle* H, int B, const double* uni, RngSpec rng, double* cond) {
  const Layout& L = H->L;
  const size_t smem = H->head_v5 ? (size_t)kH5Smem : 4096 + 2 * kH4Tri + (size_t)kH4Ring * kH4Chunk;
  ensure_smem_attr((const void*)head_v4_kernel<KG, GIVEN>, 4096 + 2 * kH4Tri + (size_t)kH4Ring * kH4Chunk);
  ensure_smem_attr((const void*)head_v5_kernel<KG, GIVEN>, kH5Smem);
  const int grid = (B + kH4Warps - 1) / kH4Warps;
  const int Hd8 = (L.Hd + 7) & ~7;
  {
    KScope ks(H, "head_thresholds");
    const int64_t total = (int64_t)B * (Hd8 / 4);
    launch_k(H, head_thresholds_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, B, L.Hd, Hd8, L.W, uni,
             rng, H->X, GIVEN ? 1 : 0, H->thr);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  KScope ks(H, GIVEN ? "head_given" : "head_sample");
  const HeadV4Args args{B,        L.n,      L.h,          L.W,      (L.h + 31) / 32, (L.h + 15) / 16,
                        Hd8,      H->h4.AF, H->h4.TRI,    H->P + L.off_b1, H->P + L.off_b2, H->X,
                        H->G1,    H->G1h,   H->G1l,       H->hp18,  H->Dh,           H->Dl,
                        H->np8,   H->Xfb,   H->hd18,      H->lp_head, cond,          H->thr};
  if (H->head_v5)
    launch_k(H, head_v5_kernel<KG, GIVEN>, dim3(grid), dim3(32 * (2 * kH4Warps + 1)), smem, args);
  else
    launch_k(H, head_v4_kernel<KG, GIVEN>, dim3(grid), dim3(32 * (kH4Warps + 1)), smem, args);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

template <int KG>
static void head_v4_dispatch(Handle* H, int B, const double* uni, RngSpec rng, bool given, double* cond) {
  if (given) head_v4_launch<KG, true>(H, B, uni, rng, cond);
  else head_v4_launch<KG, false>(H, B, uni, rng, cond);
}

template <int KG>
static void head_v3_dispatch(Handle* H, int B, const double* uni, RngSpec rng, bool given, double* cond) {
  if (given) head_v3_launch<KG, true>(H, B, uni, rng, cond);
  else head_v3_launch<KG, false>(H, B, uni, rng, cond);
}

void launch_head_v2(Handle* H, int B, const double* uni, RngSpec rng, bool given, double* cond) {
  if (H->head_v4) {
    switch (H->h4.KG) {
      case 1: head_v4_dispatch<1>(H, B, uni, rng, given, cond); return;
      case 2: head_v4_dispatch<2>(H, B, uni, rng, given, cond); return;
      case 3: head_v4_dispatch<3>(H, B, uni, rng, given, cond); return;
      case 4: head_v4_dispatch<4>(H, B, uni, rng, given, cond); return;
      case 5: head_v4_dispatch<5>(H, B, uni, rng, given, cond); return;
      case 6: head_v4_dispatch<6>(H, B, uni, rng, given, cond); return;
      case 7: head_v4_dispatch<7>(H, B, uni, rng, given, cond); return;
      case 8: head_v4_dispatch<8>(H, B, uni, rng, given, cond); return;
      default: throw InvalidArgument("head sampler: hidden width > 1024 is not supported");
    }
  }
  if (H->head_fast) {
    switch (H->head_hpk / 128) {
      case 1: head_v3_dispatch<1>(H, B, uni, rng, given, cond); return;
      case 2: head_v3_dispatch<2>(H, B, uni, rng, given, cond); return;
      case 3: head_v3_dispatch<3>(H, B, uni, rng, given, cond); return;
      case 4: head_v3_dispatch<4>(H, B, uni, rng, given, cond); return;
      case 5: head_v3_dispatch<5>(H, B, uni, rng, given, cond); return;
      case 6: head_v3_dispatch<6>(H, B, uni, rng, given, cond); return;
      case 7: head_v3_dispatch<7>(H, B, uni, rng, given, cond); return;
      case 8: head_v3_dispatch<8>(H, B, uni, rng, given, cond); return;
      default: throw InvalidArgument("head sampler: hidden width > 1024 is not supported");
    }
  }
  const int kpl = (H->L.h + 31) / 32;
  if (kpl <= 1) head_v2_dispatch<1>(H, B, uni, rng, given, cond);
  else if (kpl <= 2) head_v2_dispatch<2>(H, B, uni, rng, given, cond);
  else if (kpl <= 4) head_v2_dispatch<4>(H, B, uni, rng, given, cond);
  else if (kpl <= 8) head_v2_dispatch<8>(H, B, uni, rng, given, cond);
  else if (kpl <= 16) head_v2_dispatch<16>(H, B, uni, rng, given, cond);
  else head_v2_dispatch<32>(H, B, uni, rng, given, cond);
}

}  // namespace vqmc_b200

#ifdef VQMC_TAIL_TRACE
// Trace hook (trace build only): one production head launch on B samples, timeline out.
extern "C" int vqmc_test_head_trace(vqmc_gpu_t* g, int B, unsigned long long* out) {
  using namespace vqmc_b200;
  Handle* H = reinterpret_cast<Handle*>(g);
  try {
    H->ensure_batch(B);
    RngSpec rng{1, 1, 0, B, nullptr};
    launch_head_v2(H, B, nullptr, rng, false, nullptr);
    void* tp = nullptr;
    VQMC_CUDA(cudaGetSymbolAddress(&tp, g_head_trace));
    VQMC_CUDA(cudaMemset(tp, 0, sizeof(g_head_trace)));
    launch_head_v2(H, B, nullptr, rng, false, nullptr);
    VQMC_CUDA(cudaStreamSynchronize(H->stream));
    VQMC_CUDA(cudaMemcpyFromSymbol(out, g_head_trace, sizeof(g_head_trace)));
  } catch (const std::exception& ex) {
    set_error(ex.what());
    return status_of(ex);
  }
  return VQMC_OK;
}
#endif
