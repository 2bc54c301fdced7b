// tcgen05 GEMM for sm_100a with a 3xTF32 split ("fp32-grade" tensor-core GEMM):
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
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"

namespace vqmc_b200 {

constexpr int kUmmaBM = 128;
constexpr int kUmmaBK = 32;  // fp32 elements per 128-byte row

template <int BN>
struct UmmaCfg {
  static constexpr int kStages = BN >= 256 ? 2 : 3;
  static constexpr int kABytes = kUmmaBM * kUmmaBK * 4;  // 16 KB
  static constexpr int kBBytes = BN * kUmmaBK * 4;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr size_t kSmem = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + 256;
};

struct UmmaArgs {
  int M, N, K;
  int kblk_per_split;  // k-blocks (of 32) per split
};

template <int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(256, 1)
    umma_tf32x3_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                       const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                       UmmaArgs args, Epi epi) {
  using Cfg = UmmaCfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kUmmaBM, n0 = blockIdx.x * BN;
  const int nkb = (args.K + kUmmaBK - 1) / kUmmaBK;
  const int kb0 = blockIdx.z * args.kblk_per_split;
  const int kb1 = min(nkb, kb0 + args.kblk_per_split);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tA_hi);
    ptx::prefetch_tmap(&tA_lo);
    ptx::prefetch_tmap(&tB_hi);
    ptx::prefetch_tmap(&tB_lo);
    for (int s = 0; s < Cfg::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      for (int kb = kb0; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % Cfg::kStages, use = it / Cfg::kStages;
        if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
        unsigned char* st = base + (size_t)s * Cfg::kStageBytes;
        ptx::mbar_expect_tx(&full[s], Cfg::kStageBytes);
        const int kc = kb * kUmmaBK;
        if (A_MN) {
          ptx::tma_load_3d(st, &tA_hi, &full[s], 0, kc, m0 / 32);
          ptx::tma_load_3d(st + Cfg::kABytes, &tA_lo, &full[s], 0, kc, m0 / 32);
        } else {
          ptx::tma_load_2d(st, &tA_hi, &full[s], kc, m0);
          ptx::tma_load_2d(st + Cfg::kABytes, &tA_lo, &full[s], kc, m0);
        }
        unsigned char* sb = st + 2 * Cfg::kABytes;
        if (B_MN) {
          ptx::tma_load_3d(sb, &tB_hi, &full[s], 0, kc, n0 / 32);
          ptx::tma_load_3d(sb + Cfg::kBBytes, &tB_lo, &full[s], 0, kc, n0 / 32);
        } else {
          ptx::tma_load_2d(sb, &tB_hi, &full[s], kc, n0);
          ptx::tma_load_2d(sb + Cfg::kBBytes, &tB_lo, &full[s], kc, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = ptx::idesc_tf32(BN, A_MN, B_MN);
      // descriptor geometry (bytes): LBO / SBO and the per-MMA (K = 8) start advance
      constexpr uint32_t a_lbo = A_MN ? 32 * 128 : 16, a_sbo = A_MN ? 512 : 1024, a_step = A_MN ? 1024 : 32;
      constexpr uint32_t b_lbo = B_MN ? 32 * 128 : 16, b_sbo = B_MN ? 512 : 1024, b_step = B_MN ? 1024 : 32;
      constexpr uint32_t a_lay = A_MN ? 1 : 2, b_lay = B_MN ? 1 : 2;
      for (int kb = kb0; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % Cfg::kStages, use = it / Cfg::kStages;
        ptx::mbar_wait(&full[s], use & 1);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(base + (size_t)s * Cfg::kStageBytes);
        const uint32_t sal = sa + Cfg::kABytes;
        const uint32_t sb = sa + 2 * Cfg::kABytes;
        const uint32_t sbl = sb + Cfg::kBBytes;
#pragma unroll
        for (int k = 0; k < kUmmaBK / 8; ++k) {
          const uint64_t ah = ptx::sdesc(sa + k * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t al = ptx::sdesc(sal + k * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t bh = ptx::sdesc(sb + k * b_step, b_lbo, b_sbo, b_lay);
          const uint64_t bl = ptx::sdesc(sbl + k * b_step, b_lbo, b_sbo, b_lay);
          const uint32_t acc0 = (kb > kb0 || k > 0) ? 1u : 0u;
          ptx::mma_tf32(tmem, ah, bh, idesc, acc0);
          ptx::mma_tf32(tmem, ah, bl, idesc, 1u);
          ptx::mma_tf32(tmem, al, bh, idesc, 1u);
        }
        ptx::mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
      }
      ptx::mma_commit(tfull);  // accumulator complete
    }
  }
  // ---------------- epilogue: all 8 warps ----------------
  // warp w reads TMEM lanes 32 (w % 4) .. +31 (its row quarter); warps 4-7 take the even
  // 32-column chunks and warps 0-3 (done with TMA / MMA / allocation) the odd ones.
  __syncwarp();
  {
    const int q = warp & 3, part = warp < 4 ? 1 : 0;
    const int row = m0 + 32 * q + lane;
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
    Epi e = epi;
    e.part = part;
    e.begin_row(row, args);
    const bool has_k = kb1 > kb0;
#pragma unroll 1
    for (int c = 32 * part; c < BN; c += 64) {
      if (n0 + c >= args.N) break;
      float v[32];
      if (has_k) {
        ptx::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      e.chunk(row, n0 + c, v, args);
    }
    e.end_row(row, args);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
}

}  // namespace vqmc_b200
