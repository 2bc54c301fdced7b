// Dense-graph Max-Cut energies on the tensor cores (the reference generator's G(n, 3/4) instances,
// proj/src/hamiltonian.cpp:144-160; SURVEY.md §7 hard part #5).
//
// For spins x in {0,1}^n and the strictly upper adjacency U (U[i][j] = 1 for edges (i, j), i < j):
//   cut(x) = sum_E [x_i != x_j] = sum_i x_i deg_i - 2 sum_{(i,j) in E} x_i x_j
//          = sum_i x_i (deg_i - 2 Y_i),    Y = X U^T,  Y_bi = sum_{j > i} U_ij x_bj.
// (hamiltonian.cpp:61-69 with beta_ij = -1/4: l = (|E| - 2 cut) / 4.)  Y is one GEMM with exactly
// representable 0/1 operands: fp8 e4m3 (1.0 = 0x38) through tcgen05.mma.kind::f8f6f4 with fp32
// accumulation in TMEM - exact, since every Y_bi <= n < 2^24.  Because U is strictly upper
// triangular, the output tile of nodes [i0, i0 + BN) only needs K = j >= i0: half the dense FLOPs.
//
// Kernel: persistent CTA pairs (cta_group::2, M = 256 samples x N = 256 nodes per pair tile), TMA
// producer warp, single-thread MMA issuer on the leader, TMEM double-buffered accumulator, 8
// epilogue warps that reduce each row's 32-column chunks to sum x_i (deg_i - 2 Y_bi) and write one
// int32 partial per (row, column tile, epilogue set) into cpart; the statistics kernel sums the
// partials of a row in a fixed order (exact integers, like the edge-list kernel's).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "ptx.cuh"
#include "umma2_gemm.cuh"
#include "umma_gemm.cuh"

namespace vqmc_b200 {
namespace ptx {
__device__ __forceinline__ void mma_f8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// kind::f8f6f4, A and B e4m3 (format 0), fp32 accumulate, both K-major, M = 256 (pair).
__host__ __device__ constexpr uint32_t idesc_f8_m256(int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
}  // namespace ptx

constexpr uint8_t kFp8One = 0x38;  // e4m3 1.0

struct QfCfg {
  static constexpr int BN = 256;                        // nodes per pair tile (128 per CTA's B half)
  static constexpr int kBK = 128;                       // K per stage: one 128-byte row of 8-bit elements
  static constexpr int kABytes = kUmmaBM * 128;         // 16 KB: the CTA's 128 sample rows
  static constexpr int kBBytes = (BN / 2) * 128;        // 16 KB: the CTA's half of the node rows
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = 6;
  static constexpr int kTmemCols = 2 * BN;              // double-buffered accumulator (512 columns)
  static constexpr int kEpiSets = 2;                    // 2 x 4 epilogue warps, alternate 32-column chunks
  static constexpr int kThreads = 128 + 128 * kEpiSets;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256;
};

struct QfArgs {
  int B, n, W;
  int tiles_m, tiles_n;
  int nkb;                    // K blocks over all n columns
  const uint32_t* X;          // packed spins [B][W] (the epilogue's x_i)
  const int32_t* deg;         // [n] node degrees
  int32_t* cpart;             // [tiles_n * kEpiSets][B]
};

// Tile sequence of pair p: waves of npairs tiles in a boustrophedon order over the tile list, which
// is sorted by decreasing work (column tile tn needs K blocks tn * BN / 128 ..): the heavy and light
// tiles of consecutive waves pair up.  Tile index -> (tm = t % tiles_m, tn = t / tiles_m): the
// M tiles of one column tile run together, so its node rows are read from HBM once (L2 reuse).
__device__ __forceinline__ int qf_tile(int j, int pair, int npairs) {
  const int wave = j, pos = (wave & 1) ? npairs - 1 - pair : pair;
  return wave * npairs + pos;
}

__global__ void __launch_bounds__(QfCfg::kThreads, 1)
    qform_cut_kernel(const __grid_constant__ CUtensorMap tX, const __grid_constant__ CUtensorMap tU, QfArgs a) {
  using Cfg = QfCfg;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int ntiles = a.tiles_m * a.tiles_n;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tX);
    ptx::prefetch_tmap(&tU);
    for (int s = 0; s < Cfg::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * 4 * Cfg::kEpiSets);
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

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs) ----------------
      int s = 0, use = 0;
      for (int j = 0;; ++j) {
        const int t = qf_tile(j, pair, npairs);
        if (j * npairs >= ntiles) break;
        if (t >= ntiles) continue;
        const int tm = t % a.tiles_m, tn = t / a.tiles_m;
        const int m0 = tm * 2 * kUmmaBM + (int)rank * kUmmaBM;
        const int n0 = tn * Cfg::BN + (int)rank * (Cfg::BN / 2);
        for (int kb = tn * Cfg::BN / Cfg::kBK; kb < a.nkb; ++kb) {
          if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
          unsigned char* st = base + (size_t)s * Cfg::kStageBytes;
          if (leader) ptx::mbar_expect_tx(&full[s], 2u * (uint32_t)Cfg::kStageBytes);
          ptx::tma_load_2d_pair(st, &tX, &full[s], kb * Cfg::kBK, m0);
          ptx::tma_load_2d_pair(st + Cfg::kABytes, &tU, &full[s], kb * Cfg::kBK, n0);
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader) ----------------
      constexpr uint32_t idesc = ptx::idesc_f8_m256(Cfg::BN);
      int s = 0, use = 0, jj = 0;
      for (int j = 0;; ++j) {
        const int t = qf_tile(j, pair, npairs);
        if (j * npairs >= ntiles) break;
        if (t >= ntiles) continue;
        const int tn = t / a.tiles_m;
        const int buf = jj & 1;
        if (jj >= 2) ptx::mbar_wait(&tempty[buf], ((jj >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * Cfg::BN);
        const int kb0 = tn * Cfg::BN / Cfg::kBK;
        for (int kb = kb0; kb < a.nkb; ++kb) {
          ptx::mbar_wait(&full[s], use & 1);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(base + (size_t)s * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < Cfg::kBK / 32; ++k) {  // one MMA = K 32 (32 bytes of the 128-byte row)
            const uint64_t ad = ptx::sdesc(sa + 32 * k, 16, 1024, 2);
            const uint64_t bd = ptx::sdesc(sb + 32 * k, 16, 1024, 2);
            ptx::mma_f8_pair(acc, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          ptx::mma_commit_pair(&empty[s]);
          if (++s == Cfg::kStages) {
            s = 0;
            ++use;
          }
        }
        ptx::mma_commit_pair(&tfull[buf]);
        ++jj;
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs) ----------------
    const int q = warp & 3, part = (warp - 4) >> 2;
    const uint32_t tl0 = ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t tl1 = ptx::mapa_shared(ptx::smem_u32(&tempty[1]), 0);
    int jj = 0;
    for (int j = 0;; ++j) {
      const int t = qf_tile(j, pair, npairs);
      if (j * npairs >= ntiles) break;
      if (t >= ntiles) continue;
      const int tm = t % a.tiles_m, tn = t / a.tiles_m;
      const int buf = jj & 1;
      const int b = tm * 2 * kUmmaBM + (int)rank * kUmmaBM + 32 * q + lane;
      const int n0 = tn * Cfg::BN;
      ptx::mbar_wait(&tfull[buf], (jj >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * Cfg::BN);
      int acc = 0;
#pragma unroll 1
      for (int cc = 32 * part; cc < Cfg::BN; cc += 32 * Cfg::kEpiSets) {
        const int c0 = n0 + cc;
        if (c0 >= a.n) break;
        float v[32];
        ptx::tmem_ld32(trow + (uint32_t)cc, v);
        const uint32_t word = b < a.B ? __ldg(&a.X[(size_t)b * a.W + (c0 >> 5)]) : 0u;
        const int dj = c0 + lane < a.n ? __ldg(&a.deg[c0 + lane]) : 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int di = __shfl_sync(kFull, dj, i);  // deg of node c0 + i (the same for every row)
          const int y = (int)v[i];                   // exact: Y <= n < 2^24
          acc += ((word >> i) & 1u) ? di - 2 * y : 0;
        }
      }
      if (b < a.B) a.cpart[(size_t)(tn * Cfg::kEpiSets + part) * a.B + b] = acc;
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(buf ? tl1 : tl0);
      ++jj;
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) ptx::tmem_dealloc_pair<Cfg::kTmemCols>(tmem);
}

// X bits [B][W] -> fp8 spins [B][32 W] (1.0 = 0x38): 32 bytes per thread (two 16-byte stores).
__global__ void expand_spins_fp8_kernel(int64_t words, const uint32_t* __restrict__ X, uint8_t* __restrict__ Xf) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= words) return;
  const uint32_t w = X[t];
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) r |= ((w >> (4 * q + k)) & 1u) ? ((uint32_t)kFp8One << (8 * k)) : 0u;
    o[q] = r;
  }
  uint4* dst = reinterpret_cast<uint4*>(Xf + 32 * t);
  dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

// U[i][j] = 1.0 (fp8) for every edge (i, j), i < j (strictly upper triangle; the rest stays 0).
__global__ void scatter_upper_kernel(int64_t nE, const int2* __restrict__ edges, int64_t ld, uint8_t* __restrict__ U,
                                     int32_t* __restrict__ deg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nE; e += (int64_t)gridDim.x * blockDim.x) {
    const int2 ed = edges[e];
    U[(size_t)ed.x * ld + ed.y] = kFp8One;
    atomicAdd(&deg[ed.x], 1);
    atomicAdd(&deg[ed.y], 1);
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
// Dense path when the quadratic form is cheaper than the edge list: the GEMM does ~n^2 / 2 fp8 MACs
// per sample at ~100x the bit-sliced edge rate (VQMC_ENERGY=edges|dense overrides).
bool dense_energy_preferred(int n, int64_t nE) {
  if (const char* e = std::getenv("VQMC_ENERGY")) {
    if (e[0] == 'd') return n >= 32;
    if (e[0] == 'e') return false;
  }
  return n >= 512 && nE * 128 >= (int64_t)n * n;
}

void free_dense_energy(Handle* H) {
  if (H->Uf8) cudaFree(H->Uf8);
  if (H->Xf8) cudaFree(H->Xf8);
  if (H->d_degn) cudaFree(H->d_degn);
  H->Uf8 = nullptr;
  H->Xf8 = nullptr;
  H->d_degn = nullptr;
  H->xf8_cap = 0;
  H->dense_energy = false;
}

// (Re)build the fp8 upper adjacency and the degrees from the handle's edge list.
void setup_dense_energy(Handle* H) {
  free_dense_energy(H);
  const int n = H->L.n;
  if (!dense_energy_preferred(n, H->num_edges)) return;
  const int64_t ld = 32LL * H->L.W;
  VQMC_CUDA(cudaMalloc((void**)&H->Uf8, (size_t)n * ld));
  VQMC_CUDA(cudaMemsetAsync(H->Uf8, 0, (size_t)n * ld, H->stream));
  VQMC_CUDA(cudaMalloc((void**)&H->d_degn, (size_t)n * sizeof(int32_t)));
  VQMC_CUDA(cudaMemsetAsync(H->d_degn, 0, (size_t)n * sizeof(int32_t), H->stream));
  if (H->num_edges > 0) {
    const int grid = (int)std::min<int64_t>(148 * 8, (H->num_edges + 255) / 256);
    scatter_upper_kernel<<<grid, 256, 0, H->stream>>>(H->num_edges, H->d_edges, ld, H->Uf8, H->d_degn);
    VQMC_CUDA(cudaGetLastError());
  }
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  H->dense_energy = true;
}

void launch_energy_dense(Handle* H, int B) {
  const int n = H->L.n, W = H->L.W;
  const int64_t ld = 32LL * W;
  if ((int64_t)B > H->xf8_cap) {
    if (H->capturing) throw std::runtime_error("fp8 spin buffer reallocation during graph capture");
    H->invalidate_graph();
    if (H->Xf8) VQMC_CUDA(cudaFree(H->Xf8));
    VQMC_CUDA(cudaMalloc((void**)&H->Xf8, (size_t)B * ld));
    H->xf8_cap = B;
  }
  {
    const int64_t words = (int64_t)B * W;
    KScope ks(H, "expand_spins_fp8");
    launch_k(H, expand_spins_fp8_kernel, dim3((unsigned)((words + 255) / 256)), dim3(256), 0, words,
             (const uint32_t*)H->X, H->Xf8);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  using Cfg = QfCfg;
  QfArgs a;
  a.B = B;
  a.n = n;
  a.W = W;
  a.tiles_m = (B + 2 * kUmmaBM - 1) / (2 * kUmmaBM);
  a.tiles_n = (n + Cfg::BN - 1) / Cfg::BN;
  a.nkb = (n + Cfg::kBK - 1) / Cfg::kBK;
  a.X = H->X;
  a.deg = H->d_degn;
  H->ensure_cpart((int64_t)a.tiles_n * Cfg::kEpiSets * B);
  a.cpart = H->cpart;
  H->cut_chunks = a.tiles_n * Cfg::kEpiSets;
  const CUtensorMap tX = tmap_kmajor(H->Xf8, n, B, ld, kUmmaBM, kElemU8);
  const CUtensorMap tU = tmap_kmajor(H->Uf8, n, n, ld, Cfg::BN / 2, kElemU8);
  ensure_smem_attr((const void*)qform_cut_kernel, Cfg::kSmem);
  const int ntiles = a.tiles_m * a.tiles_n;
  const int pairs = std::max(1, std::min(ntiles, gemm_sms(H) / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = H->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KScope ks(H, "maxcut_energy_dense");
  VQMC_CUDA(cudaLaunchKernelEx(&cfg, qform_cut_kernel, tX, tU, a));
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

}  // namespace vqmc_b200
