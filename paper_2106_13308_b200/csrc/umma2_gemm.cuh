// CTA-pair (cta_group::2) variant of the 3-pass tcgen05 GEMM in umma_gemm.cuh.
//
// A cluster of two CTAs on one TPC computes 256 x BN output tiles: CTA rank r holds rows
// m0 + 128 r of A and columns n0 + (BN / 2) r of B in its shared memory (identical layouts in
// both CTAs), and the leader (rank 0) issues tcgen05.mma.cta_group::2 (M = 256), which reads
// both CTAs' operands and writes each CTA's 128 accumulator rows into that CTA's TMEM.  Per SM
// this halves the B bytes per FLOP and doubles the MMA work per stage, which is what lifts
// these (L2 -> SM bandwidth-bound) 3-pass GEMMs.
//
//   both CTAs, warp 0   TMA producer: its halves of A and B, completing on the LEADER's
//                       full[s] barrier (cta_group::2 bulk tensor copies with the peer bit clear)
//   leader,    warp 1   MMA issuer: waits full[s], 3 x (BK / MMA_K) MMAs, commits to empty[s] of
//                       both CTAs (multicast); at the tile end commits tfull[buf] of both CTAs
//   both CTAs, warp 2   TMEM allocator (tcgen05.alloc.cta_group::2, same warp id in both)
//   both CTAs, warps 4+ epilogue on the CTA's own 128 rows; then arrive on the LEADER's
//                       tempty[buf] (count 2 x epilogue warps)
// The accumulator is double-buffered in TMEM (2 BN columns) as in the single-CTA kernel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"
#include "umma_gemm.cuh"

namespace vqmc_b200 {
#ifdef VQMC_TAIL_TRACE
// per CTA: [0] start, then per local tile j < 6: [1 + 4j] MMA start, [2 + 4j] MMA end (commit issued),
// [3 + 4j] epilogue start (accumulator ready), [4 + 4j] epilogue end (set 0, warp 4); [31] CTA end
__device__ unsigned long long g_tail_trace[148 * 32];
__device__ int g_tail_exp;  // experiment mask of the tail epilogue (1: no D stores, 2: no Philox)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TAIL_TRACE(slot) g_tail_trace[blockIdx.x * 32 + (slot)] = gtime()
#else
#define TAIL_TRACE(slot)
#endif
namespace ptx {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Relaxed remote arrive: the accumulator-drained signal carries no memory hand-off (the TMEM
// reads are ordered by tcgen05.fence::before_thread_sync), so the epilogue's global stores need
// not drain first (a release at cluster scope would wait for them).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // clears the pair-peer bit: the leader CTA's copy
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerBitMask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & kPeerBitMask)
      : "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// Instruction descriptor for kind::f16, M = 256 (pair).
__host__ __device__ constexpr uint32_t idesc_f16_m256(int N, bool a_mn, bool b_mn, bool bf16) {
  return (1u << 4) | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

}  // namespace ptx

// SETS: epilogue warp sets (0 = automatic); CHUNK: accumulator columns per epilogue call (32 or 16;
// 16-column chunks let 4 sets share a 192-column tile evenly).
template <int BN, int SETS = 0, int CHUNK = 32>
struct Umma2Cfg {  // 16-bit operand pairs only; per CTA: A 128 rows, B BN / 2 rows
  static constexpr int kBK = 64;                            // K per stage (128-byte rows)
  static constexpr int kABytes = kUmmaBM * 128;             // 16 KB
  static constexpr int kBBytes = (BN / 2) * 128;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes > 6 ? 6 : (200 * 1024) / kStageBytes;
  static constexpr int kTmemCols = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int kChunk = CHUNK;
  static constexpr int kChunks = BN / CHUNK;
  // epilogue warp sets of 4 warps, each taking whole chunks (balanced: 6 chunks -> 3 sets)
  static constexpr int kEpiSets =
      SETS ? SETS : (kChunks % 4 == 0 ? 4 : (kChunks % 3 == 0 ? 3 : (kChunks < 4 ? kChunks : 4)));
  static constexpr int kThreads = 128 + 128 * kEpiSets;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
  static_assert(BN % 32 == 0 && BN >= 64 && BN <= 256, "pair tile N");
  static_assert(CHUNK == 16 || CHUNK == 32, "epilogue chunk");
};

// Pair tile t -> (n = t % tiles_n, m = (t / tiles_n) % tiles_m, split = t / (tiles_n tiles_m)); tiles_m
// counts 256-row tiles.  Epilogue rows are m0 + 128 rank + 32 q + lane (UmmaTile.tm = 2 tm + rank).
template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT, int EK, int SETS = 0, int CHUNK = 32>
__global__ void __launch_bounds__(Umma2Cfg<BN, SETS, CHUNK>::kThreads, 1)
    umma2_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                 const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo, UmmaArgs args,
                 Epi epi) {
  using Cfg = Umma2Cfg<BN, SETS, CHUNK>;
  static_assert(EK != kElemTF32, "pair kernel: 16-bit operand pairs");
  static_assert(!B_MN || (BN / 2) % 64 == 0, "MN-major B: each CTA's half must be whole 64-element atoms");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2] (leader's are used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nkb = (args.K + Cfg::kBK - 1) / Cfg::kBK;
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
      ptx::mbar_init(&tempty[b], 2 * 4 * Cfg::kEpiSets);  // every epilogue warp of both CTAs
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (threadIdx.x == 0) TAIL_TRACE(0);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs) ----------------
      constexpr int kMNa = 64;  // 16-bit MN-major atom (128 bytes)
      int s = 0, use = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        const UmmaTile c = tile_of(t);
        const int m0 = c.tm * 2 * kUmmaBM + (int)rank * kUmmaBM, n0 = c.tn * BN + (int)rank * (BN / 2);
        const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
          unsigned char* st = base + (size_t)s * Cfg::kStageBytes;
          if (leader)  // both CTAs' bytes land on the leader's barrier
            ptx::mbar_expect_tx(&full[s], 2u * (uint32_t)(A_EXACT ? Cfg::kStageBytes - Cfg::kABytes : Cfg::kStageBytes));
          const int kc = kb * Cfg::kBK;
          if (A_MN) {
            ptx::tma_load_3d_pair(st, &tA_hi, &full[s], 0, kc, m0 / kMNa);
            if (!A_EXACT) ptx::tma_load_3d_pair(st + Cfg::kABytes, &tA_lo, &full[s], 0, kc, m0 / kMNa);
          } else {
            ptx::tma_load_2d_pair(st, &tA_hi, &full[s], kc, m0);
            if (!A_EXACT) ptx::tma_load_2d_pair(st + Cfg::kABytes, &tA_lo, &full[s], kc, m0);
          }
          unsigned char* sb = st + 2 * Cfg::kABytes;
          if (B_MN) {
            ptx::tma_load_3d_pair(sb, &tB_hi, &full[s], 0, kc, n0 / kMNa);
            ptx::tma_load_3d_pair(sb + Cfg::kBBytes, &tB_lo, &full[s], 0, kc, n0 / kMNa);
          } else {
            ptx::tma_load_2d_pair(sb, &tB_hi, &full[s], kc, n0);
            ptx::tma_load_2d_pair(sb + Cfg::kBBytes, &tB_lo, &full[s], kc, n0);
          }
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader) ----------------
      constexpr uint32_t idesc = ptx::idesc_f16_m256(BN, A_MN, B_MN, EK == kElemBF16);
      // K-major: SWIZZLE_128B rows (LBO 16, SBO 1024, one MMA = 32 bytes of K); MN-major: 64-element
      // atoms of 64 K-rows (8192 B apart), 8-row groups (SBO 1024), one MMA = 16 K-rows (2048 bytes)
      constexpr uint32_t a_lbo = A_MN ? 8192 : 16, a_sbo = 1024, a_step = A_MN ? 2048 : 32;
      constexpr uint32_t b_lbo = B_MN ? 8192 : 16, b_sbo = 1024, b_step = B_MN ? 2048 : 32;
      int s = 0, use = 0, j = 0;
      for (int t = pair; t < ntiles; t += npairs, ++j) {
        const UmmaTile c = tile_of(t);
        const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
        const int buf = j & 1;
        if (j >= 2) ptx::mbar_wait(&tempty[buf], ((j >> 1) - 1) & 1);  // both epilogues drained it
        if (j < 6) TAIL_TRACE(1 + 4 * j);
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
          for (int k = 0; k < Cfg::kBK / 16; ++k) {
            const uint64_t ah = ptx::sdesc(sa + k * a_step, a_lbo, a_sbo, 2);
            const uint64_t al = ptx::sdesc(sal + k * a_step, a_lbo, a_sbo, 2);
            const uint64_t bh = ptx::sdesc(sb + k * b_step, b_lbo, b_sbo, 2);
            const uint64_t bl = ptx::sdesc(sbl + k * b_step, b_lbo, b_sbo, 2);
            const uint32_t acc0 = (kb > kb0 || k > 0) ? 1u : 0u;
            ptx::mma_f16_pair(acc, ah, bh, idesc, acc0);
            ptx::mma_f16_pair(acc, ah, bl, idesc, 1u);
            if (!A_EXACT) ptx::mma_f16_pair(acc, al, bh, idesc, 1u);
          }
          ptx::mma_commit_pair(&empty[s]);  // frees stage s in both CTAs once the MMAs read it
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
        ptx::mma_commit_pair(&tfull[buf]);  // both CTAs' accumulators of this tile are complete
        if (j < 6) TAIL_TRACE(2 + 4 * j);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs) ----------------
    const int q = warp & 3, part = (warp - 4) >> 2;
    const uint32_t tempty_leader0 = ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = ptx::mapa_shared(ptx::smem_u32(&tempty[1]), 0);
    Epi e = epi;
    e.init();  // per-thread state that does not change between tiles
    int j = 0;
    for (int t = pair; t < ntiles; t += npairs, ++j) {
      UmmaTile c = tile_of(t);
      const int kb0 = c.z * args.kblk_per_split, kb1 = min(nkb, kb0 + args.kblk_per_split);
      const int m0 = c.tm * 2 * kUmmaBM + (int)rank * kUmmaBM, n0 = c.tn * BN;
      c.tm = 2 * c.tm + (int)rank;  // the epilogue's 128-row tile index
      const int buf = j & 1;
      const int row = m0 + 32 * q + lane;
      ptx::mbar_wait(&tfull[buf], (j >> 1) & 1);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && j < 6) TAIL_TRACE(3 + 4 * j);
      e.part = part;
      e.tile = c;
      e.begin_row(row, args);
      const bool has_k = kb1 > kb0;
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN);
#pragma unroll 1
      for (int cc = CHUNK * part; cc < BN; cc += CHUNK * Cfg::kEpiSets) {
        if (n0 + cc >= args.N) break;
        float v[CHUNK];
        if (has_k) {
          if constexpr (CHUNK == 32) ptx::tmem_ld32(trow + (uint32_t)cc, v);
          else ptx::tmem_ld16(trow + (uint32_t)cc, v);
        } else {
#pragma unroll
          for (int i = 0; i < CHUNK; ++i) v[i] = 0.f;
        }
        e.chunk(row, n0 + cc, v, args);
      }
      e.end_row(row, args);
      if (warp == 4 && lane == 0 && j < 6) TAIL_TRACE(4 + 4 * j);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(buf ? tempty_leader1 : tempty_leader0);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs done (the leader's MMAs read the peer's smem until here)
  if (threadIdx.x == 0) TAIL_TRACE(31);
  if (warp == 2) ptx::tmem_dealloc_pair<Cfg::kTmemCols>(tmem);
}

}  // namespace vqmc_b200
