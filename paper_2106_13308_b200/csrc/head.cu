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

// Padded, completion-ordered copies of the head blocks (refreshed after every update):
//   W1Tp[j][k] = W1m[k][j]           j < Hd, k < h (row stride hp)
//   W2cp[c][i] = W2m[i][comp_k[c]]   c < h,  i < Hd (row stride Hdp)
__global__ void head_pack_kernel(int h, int Hd, int hp, int Hdp, const float* __restrict__ W1T,
                                 const float* __restrict__ W2, const int* __restrict__ comp_k,
                                 float* __restrict__ W1Tp, float* __restrict__ W2cp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)Hd * hp, n2 = (int64_t)h * Hdp;
  if (t < n1) {
    const int j = (int)(t / hp), k = (int)(t % hp);
    W1Tp[t] = k < h ? W1T[(size_t)j * h + k] : 0.f;
  } else if (t < n1 + n2) {
    const int64_t u = t - n1;
    const int c = (int)(u / Hdp), i = (int)(u % Hdp);
    W2cp[u] = i < Hd ? W2[(size_t)i * h + comp_k[c]] : 0.f;
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
  const int hp = 32 * head_kpl(L.h), Hdp = H->head_fast ? hp : 32 * ((L.Hd + 31) / 32);
  const int64_t total = (int64_t)L.Hd * hp + (int64_t)L.h * Hdp;
  KScope ks(H, "head_pack");
  head_pack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(
      L.h, L.Hd, hp, Hdp, H->P + L.off_w1t, H->P + L.off_w2, H->d_comp_k, H->W1Tp, H->W2cp);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

template <int KPL, bool FAST, bool GIVEN>
static void head_v2_launch(Handle* H, int B, const double* uni, RngSpec rng, double* cond) {
  const Layout& L = H->L;
  const HeadGeom geo = head_geometry(H);
  static size_t attr_set = 0;
  if (attr_set < geo.smem) {
    VQMC_CUDA(cudaFuncSetAttribute(head_v2_kernel<KPL, FAST, GIVEN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)geo.smem));
    attr_set = geo.smem;
  }
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

void launch_head_v2(Handle* H, int B, const double* uni, RngSpec rng, bool given, double* cond) {
  const int kpl = (H->L.h + 31) / 32;
  if (kpl <= 1) head_v2_dispatch<1>(H, B, uni, rng, given, cond);
  else if (kpl <= 2) head_v2_dispatch<2>(H, B, uni, rng, given, cond);
  else if (kpl <= 4) head_v2_dispatch<4>(H, B, uni, rng, given, cond);
  else if (kpl <= 8) head_v2_dispatch<8>(H, B, uni, rng, given, cond);
  else if (kpl <= 16) head_v2_dispatch<16>(H, B, uni, rng, given, cond);
  else head_v2_dispatch<32>(H, B, uni, rng, given, cond);
}

}  // namespace vqmc_b200
