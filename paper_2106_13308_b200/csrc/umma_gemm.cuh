// tcgen05 3-pass GEMM for sm_100a ("fp32-grade" tensor-core GEMM on split operands: tf32, bf16 or fp16 pairs):
//
//   C[M x N] (fp32, TMEM) = sum_k A(m, k) B(n, k),  computed as
//   A_hi B_hi + A_hi B_lo + A_lo B_hi          (operands stored as tf32 hi/lo pairs)
//
// Warp-specialised, one 128 x BN output tile per CTA (split-K over blockIdx.z):
//   warp 0  TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier complete_tx)
//   warp 1  MMA issuer (one elected lane issues tcgen05.mma.kind::tf32, commits to mbarriers)
//   warp 2  TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld 32 lanes x 32 columns -> registers -> Epi functor
// Operands may be K-major (2D tensor map {K, MN}, box {32, MN}) or MN-major (3D map
// {32, K, MN/32}, box {32, 32, MN/32}); the smem tiles are the canonical UMMA layouts:
//   K-major : 128-byte rows (32 fp32 of K), 8-row groups 1024 B apart, SWIZZLE_128B
//             (LBO 16, SBO 1024; one MMA (K = 8) = 32 bytes of the row)
//   MN-major: 32-element MN atoms of 32 K-rows (4096 B apart), 4-row groups 512 B apart,
//             SWIZZLE_128B_BASE32B (LBO 4096, SBO 512; one MMA = 8 K-rows = 1024 bytes)
// and for 16-bit pairs (EK = bf16 / fp16): K-major as above (one MMA = K 16 = 32 bytes); MN-major
// 64-element atoms of 64 K-rows (8192 B apart), SWIZZLE_128B, 8-row groups (LBO 8192,
// SBO 1024; one MMA = 16 K-rows = 2048 bytes).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"

namespace vqmc_b200 {

constexpr int kUmmaBM = 128;
constexpr int kUmmaBK = 32;  // fp32 elements per 128-byte row (bf16: 64)

// Operand element kind EK: 0 = tf32 pairs (3 x kind::tf32, MMA K = 8); 1 = bf16 pairs, 2 = fp16
// pairs (3 x kind::f16, MMA K = 16).
enum : int { kElemTF32 = 0, kElemBF16 = 1, kElemF16 = 2, kElemU8 = 3 /* 8-bit (fp8 / int8) single operands */ };
template <int EK>
struct UmmaElem {
  static constexpr int kBytes = EK ? 2 : 4;
  static constexpr int kBK = 128 / kBytes;     // elements per 128-byte smem row = K per stage
  static constexpr int kMmaK = 32 / kBytes;    // K of one MMA (32 bytes)
  static constexpr int kMNAtom = 128 / kBytes; // MN-major atom width (elements)
};

template <int BN>
struct UmmaCfg {  // tile bytes are the same for both element types (128-byte rows)
  static constexpr int kStages = BN >= 256 ? 2 : 3;
  static constexpr int kABytes = kUmmaBM * kUmmaBK * 4;  // 16 KB
  static constexpr int kBBytes = BN * kUmmaBK * 4;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int kEpiSets = BN / 32 < 4 ? BN / 32 : 4;  // epilogue warp sets (4 warps each)
  static constexpr int kThreads = 128 + 128 * kEpiSets;  // 4 control warps + epilogue warps
  static constexpr size_t kSmem = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + 256;
};

struct UmmaArgs {
  int M, N, K;
  int kblk_per_split;  // k-blocks (of 32) per split
  int tiles_n, tiles_m, splits;
};

// Tile coordinates handed to the epilogue functor.
struct UmmaTile {
  int tn, tm, z;
};

// Persistent: CTA b processes tiles b, b + grid, ...; tile t -> (n = t % tiles_n,
// m = (t / tiles_n) % tiles_m, split = t / (tiles_n tiles_m)).  The accumulator is
// double-buffered in TMEM (2 x BN columns) so the epilogue of tile j overlaps the
// mainloop of tile j + 1.
//   warp 0  TMA producer     warp 1  MMA issuer     warp 2  TMEM allocator
//   warps 4..  epilogue (kEpiSets sets of 4 warps; set s takes 32-column chunks s, s + kEpiSets, ...)
// A_EXACT: A is exactly representable (e.g. 0/1 spins): A_lo is neither loaded nor used.
template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT = false, int EK = kElemTF32>
__global__ void __launch_bounds__(UmmaCfg<BN>::kThreads, 1)
    umma3p_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                       const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                       UmmaArgs args, Epi epi) {
  using Cfg = UmmaCfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using E = UmmaElem<EK>;
  const int nkb = (args.K + E::kBK - 1) / E::kBK;
  const int ntiles = args.tiles_n * args.tiles_m * args.splits;
  auto tile_of = [&](int t) {
    UmmaTile c;
    c.tn = t % args.tiles_n;
    c.tm = (t / args.tiles_n) % args.tiles_m;
    c.z = t / (args.tiles_n * args.tiles_m);
    return c;
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tA_hi);
    ptx::prefetch_tmap(&tA_lo);
    ptx::prefetch_tmap(&tB_hi);
    ptx::prefetch_tmap(&tB_lo);
    for (int s = 0; s < Cfg::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 4 * Cfg::kEpiSets);  // one arrive per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_trigger();
  ptx::pdl_wait();  // predecessor's outputs (the operands) are complete from here on

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int s = 0, use = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const UmmaTile c = tile_of(t);
        const int m0 = c.tm * kUmmaBM, n0 = c.tn * BN;
        const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
          unsigned char* st = base + (size_t)s * Cfg::kStageBytes;
          ptx::mbar_expect_tx(&full[s], A_EXACT ? Cfg::kStageBytes - Cfg::kABytes : Cfg::kStageBytes);
          const int kc = kb * E::kBK;
          if (A_MN) {
            ptx::tma_load_3d(st, &tA_hi, &full[s], 0, kc, m0 / E::kMNAtom);
            if (!A_EXACT) ptx::tma_load_3d(st + Cfg::kABytes, &tA_lo, &full[s], 0, kc, m0 / E::kMNAtom);
          } else {
            ptx::tma_load_2d(st, &tA_hi, &full[s], kc, m0);
            if (!A_EXACT) ptx::tma_load_2d(st + Cfg::kABytes, &tA_lo, &full[s], kc, m0);
          }
          unsigned char* sb = st + 2 * Cfg::kABytes;
          if (B_MN) {
            ptx::tma_load_3d(sb, &tB_hi, &full[s], 0, kc, n0 / E::kMNAtom);
            ptx::tma_load_3d(sb + Cfg::kBBytes, &tB_lo, &full[s], 0, kc, n0 / E::kMNAtom);
          } else {
            ptx::tma_load_2d(sb, &tB_hi, &full[s], kc, n0);
            ptx::tma_load_2d(sb + Cfg::kBBytes, &tB_lo, &full[s], kc, n0);
          }
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = EK ? ptx::idesc_f16(BN, A_MN, B_MN, EK == kElemBF16) : ptx::idesc_tf32(BN, A_MN, B_MN);
      // MN-major: atom stride = kBK K-rows x 128 B; K-row groups of 4 (tf32, BASE32B) or 8 (bf16)
      constexpr uint32_t mn_lbo = E::kBK * 128, mn_sbo = EK ? 1024 : 512, mn_step = E::kMmaK * 128;
      constexpr uint32_t mn_lay = EK ? 2 : 1;
      constexpr uint32_t a_lbo = A_MN ? mn_lbo : 16, a_sbo = A_MN ? mn_sbo : 1024, a_step = A_MN ? mn_step : 32;
      constexpr uint32_t b_lbo = B_MN ? mn_lbo : 16, b_sbo = B_MN ? mn_sbo : 1024, b_step = B_MN ? mn_step : 32;
      constexpr uint32_t a_lay = A_MN ? mn_lay : 2, b_lay = B_MN ? mn_lay : 2;
      int s = 0, use = 0, j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const UmmaTile c = tile_of(t);
        const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
        const int buf = j & 1;
        if (j >= 2) ptx::mbar_wait(&tempty[buf], ((j >> 1) - 1) & 1);  // epilogue drained this buffer
        ptx::tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[s], use & 1);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(base + (size_t)s * Cfg::kStageBytes);
          const uint32_t sal = sa + Cfg::kABytes;
          const uint32_t sb = sa + 2 * Cfg::kABytes;
          const uint32_t sbl = sb + Cfg::kBBytes;
#pragma unroll
          for (int k = 0; k < E::kBK / E::kMmaK; ++k) {
            const uint64_t ah = ptx::sdesc(sa + k * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t al = ptx::sdesc(sal + k * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t bh = ptx::sdesc(sb + k * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t bl = ptx::sdesc(sbl + k * b_step, b_lbo, b_sbo, b_lay);
            const uint32_t acc0 = (kb > kb0 || k > 0) ? 1u : 0u;
            if (EK) {
              ptx::mma_f16(acc, ah, bh, idesc, acc0);
              ptx::mma_f16(acc, ah, bl, idesc, 1u);
              if (!A_EXACT) ptx::mma_f16(acc, al, bh, idesc, 1u);
            } else {
              ptx::mma_tf32(acc, ah, bh, idesc, acc0);
              ptx::mma_tf32(acc, ah, bl, idesc, 1u);
              if (!A_EXACT) ptx::mma_tf32(acc, al, bh, idesc, 1u);
            }
          }
          ptx::mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
        ptx::mma_commit(&tfull[buf]);  // accumulator of this tile complete
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue ----------------
    const int q = warp & 3, part = (warp - 4) >> 2;
    Epi e = epi;
    e.init();  // per-thread state that does not change between tiles
    int j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const UmmaTile c = tile_of(t);
      const int m0 = c.tm * kUmmaBM, n0 = c.tn * BN;
      const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
      const int buf = j & 1;
      const int row = m0 + 32 * q + lane;
      ptx::mbar_wait(&tfull[buf], (j >> 1) & 1);
      ptx::tc_fence_after();
      e.part = part;
      e.tile = c;
      e.begin_row(row, args);
      const bool has_k = kb1 > kb0;
#pragma unroll 1
      for (int cc = 32 * part; cc < BN; cc += 32 * Cfg::kEpiSets) {
        if (n0 + cc >= args.N) break;
        float v[32];
        if (has_k) {
          ptx::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN + cc), v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        e.chunk(row, n0 + cc, v, args);
      }
      e.end_row(row, args);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
}

}  // namespace vqmc_b200
