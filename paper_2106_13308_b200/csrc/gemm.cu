// tcgen05 (3xTF32) GEMMs of the VQMC step and their fused epilogues:
//
//   tail sampler   Z[b][i]  = G1[b] . W2m[i] + b2[i], i >= Hd      (A = G1 K-major, B = W2 K-major)
//                  epilogue: draw x = [u < p], pack bits, D = 0.5 (x - p_raw), log-prob partials
//   dg1 (split-K)  E[b][k]  = sum_i D[b][i] W2m[i][k]              (A = D K-major, B = W2 MN-major)
//   gW2 (+ gb2)    gW2[i][k] = sum_b D[b][i] w_b G1[b][k]          (A = D^T MN-major, B = wG1 MN-major)
//
// Reference: made_forward / auto_sample / weighted_grad_log_psi, proj/src/models.cpp:51-62,
// 175-198 and proj/src/sampler.cpp:47-55.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "ptx.cuh"
#include "umma_gemm.cuh"

namespace vqmc_b200 {

// ---------------------------------------------------------------------------
// Tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point).
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    VQMC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// K-major operand: element (mn, k) at ptr[mn * ld + k]; box {32 (K), box_mn}.
CUtensorMap tmap_kmajor(const float* ptr, int64_t K, int64_t MN, int64_t ld, int box_mn) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)MN};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_mn};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (K-major) failed: " + std::to_string((int)r));
  return m;
}

// MN-major operand: element (mn, k) at ptr[k * ld + mn]; 3D view {32, K, ceil(MN/32)},
// box {32, 32, box_mn / 32}, 128-byte swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B).  Reads up to 31 elements past MN on the last chunk: the
// allocation must be padded and those rows/columns of the result are discarded.
CUtensorMap tmap_mnmajor(const float* ptr, int64_t MN, int64_t K, int64_t ld, int box_mn) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)((MN + 31) / 32)};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
  const cuuint32_t box[3] = {32, 32, (cuuint32_t)(box_mn / 32)};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (MN-major) failed: " + std::to_string((int)r));
  return m;
}

template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT = false>
static void launch_umma(Handle* H, const char* name, const CUtensorMap& ah, const CUtensorMap& al,
                        const CUtensorMap& bh, const CUtensorMap& bl, int M, int N, int K, int splits, Epi epi,
                        cudaStream_t stream) {
  using Cfg = UmmaCfg<BN>;
  auto kern = umma_tf32x3_kernel<BN, A_MN, B_MN, Epi, A_EXACT>;
  static bool attr = false;
  if (!attr) {
    VQMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr = true;
  }
  const int nkb = (K + kUmmaBK - 1) / kUmmaBK;
  UmmaArgs args{M, N, K, (nkb + splits - 1) / splits, (N + BN - 1) / BN, (M + kUmmaBM - 1) / kUmmaBM, splits};
  const int ntiles = args.tiles_n * args.tiles_m * splits;
  static int sms = 0;
  if (!sms) VQMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = std::min(ntiles, sms);
  if (H) {
    KScope ks(H, name);
    kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(ah, al, bh, bl, args, epi);
    H->launches++;
  } else {
    kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(ah, al, bh, bl, args, epi);
  }
  VQMC_CUDA(cudaGetLastError());
}

// ===========================================================================
// Epilogues
// ===========================================================================
struct StoreEpi {  // test: C[row][col] = acc
  float* C;
  int ldc;
  int part;
  UmmaTile tile;
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int row, int col0, const float (&v)[32], const UmmaArgs& a) {
    if (row >= a.M) return;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < a.N) C[(size_t)row * ldc + col0 + j] = v[j];
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// Tail sampler: rows = samples, columns = outputs colbase + col (col0 aligned to 32).
// Two epilogue warp sets share a row (alternate 32-column chunks): each writes its own
// log-prob partial (lp_part[2 * tile + part]), so the reduction stays deterministic.
struct TailSampleEpi {
  int B, n, np, W, colbase, col_lo;  // outputs in [col_lo, n) are drawn here
  const float* b2;
  const double* uni;
  RngSpec rng;
  uint32_t* X;
  float* Dhi;
  float* Dlo;
  double* lp_part;
  int part;
  UmmaTile tile;
  double lps;
  __device__ void begin_row(int, const UmmaArgs&) { lps = 0.0; }
  __device__ void chunk(int b, int col0, const float (&v)[32], const UmmaArgs&) {
    if (b >= B) return;
    const int cb = colbase + col0;
    const size_t rowD = (size_t)b * np;
    const bool full = cb >= col_lo && cb + 32 <= n;
    uint32_t word = 0;
    float lsum = 0.f;  // 32 log terms in fp32, then one fp64 add
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float thr[4];  // draw x = [u < p]: u = (r + 1/2) 2^-32 < p  <=>  r + 1/2 < p 2^32
      uint32_t r[4];
      if (uni == nullptr) rng.quad(b, cb + j, r);
      float hi4[4], lo4[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = cb + j + t;
        const bool valid = c >= col_lo && c < n;
        const float z = v[j + t] + (valid ? b2[c] : 0.f);
        const UnitPre q = unit_pre(z);
        int x;
        if (uni == nullptr) {
          thr[t] = (float)(q.p() * 4294967296.0);
          x = (valid && (float)r[t] + 0.5f < thr[t]) ? 1 : 0;
        } else {
          x = (valid && uni[(size_t)c * B + b] < q.p()) ? 1 : 0;
        }
        word |= (uint32_t)x << (j + t);
        const Unit o = unit_post(q, x);
        ptx::split_tf32(o.D, hi4[t], lo4[t]);
        if (valid) lsum += o.logt;
      }
      if (full) {
        *reinterpret_cast<float4*>(Dhi + rowD + cb + j) = make_float4(hi4[0], hi4[1], hi4[2], hi4[3]);
        *reinterpret_cast<float4*>(Dlo + rowD + cb + j) = make_float4(lo4[0], lo4[1], lo4[2], lo4[3]);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = cb + j + t;
          if (c >= col_lo && c < n) {
            Dhi[rowD + c] = hi4[t];
            Dlo[rowD + c] = lo4[t];
          }
        }
      }
    }
    lps += (double)lsum;
    if (word) atomicOr(&X[(size_t)b * W + (cb >> 5)], word);
  }
  __device__ void end_row(int b, const UmmaArgs&) {
    if (b < B) lp_part[(size_t)(kParts * tile.tn + part) * B + b] = lps;
  }
  static constexpr int kParts = UmmaCfg<128>::kEpiSets;
};

struct PartialEpi {  // split-K partial: out[z][row][col]
  float* out;
  int rows, cols;
  int part;
  UmmaTile tile;
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int row, int col0, const float (&v)[32], const UmmaArgs&) {
    if (row >= rows) return;
    float* o = out + ((size_t)tile.z * rows + row) * cols;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < cols) o[col0 + j] = v[j];
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

struct Gw2Epi {  // rows = outputs i, columns = hidden k (k == h: bias column -> gb2)
  int n, h;
  int part;
  UmmaTile tile;
  const int32_t* deg;
  float* gW2;
  float* gb2;
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int i, int col0, const float (&v)[32], const UmmaArgs&) {
    if (i >= n) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int k = col0 + j;
      if (k < h) gW2[(size_t)i * h + k] = (deg[k] < i + 1) ? v[j] : 0.f;  // M2(i, k)
      else if (k == h) gb2[i] = v[j];
    }
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// ===========================================================================
// Helper kernels: tf32 splits of operands
// ===========================================================================
__global__ void split_rows_kernel(int rows, int cols, int ld_in, int ld_out, const float* __restrict__ in,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * ld_out) return;
  const int r = (int)(t / ld_out), c = (int)(t % ld_out);
  float x = c < cols ? in[(size_t)r * ld_in + c] : 0.f;
  float a, b;
  ptx::split_tf32(x, a, b);
  hi[t] = a;
  lo[t] = b;
}

// wG1[b][k] = w_b * G1[b][k] (k < h), w_b (k == h), 0 (k > h); split into tf32 hi/lo.
__global__ void wg1_kernel(int B, int h, int hp1, const float* __restrict__ G1, const float* __restrict__ w,
                           float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * hp1) return;
  const int b = (int)(t / hp1), k = (int)(t % hp1);
  const float x = k < h ? w[b] * G1[(size_t)b * h + k] : (k == h ? w[b] : 0.f);
  float a, c;
  ptx::split_tf32(x, a, c);
  hi[t] = a;
  lo[t] = c;
}

void launch_split_w2(Handle* H) {
  const Layout& L = H->L;
  const int64_t total = (int64_t)L.n * H->hp;
  KScope ks(H, "split_w2");
  split_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(L.n, L.h, L.h, H->hp, H->P + L.off_w2,
                                                                            H->W2hi, H->W2lo);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
}

// ===========================================================================
// Production launchers
// ===========================================================================
void launch_tail_umma(Handle* H, int B, const double* uni, RngSpec rng) {
  const Layout& L = H->L;
  const int colbase = (L.Hd / 32) * 32;
  const int ncols = L.n - colbase;
  if (L.Hd >= L.n) {
    H->tail_tiles = 0;
    return;
  }
  constexpr int BN = 128;
  const CUtensorMap ah = tmap_kmajor(H->G1hi, L.h, B, H->hp, kUmmaBM);
  const CUtensorMap al = tmap_kmajor(H->G1lo, L.h, B, H->hp, kUmmaBM);
  const CUtensorMap bh = tmap_kmajor(H->W2hi + (size_t)colbase * H->hp, L.h, ncols, H->hp, BN);
  const CUtensorMap bl = tmap_kmajor(H->W2lo + (size_t)colbase * H->hp, L.h, ncols, H->hp, BN);
  TailSampleEpi e{B, L.n, H->np, L.W, colbase, L.Hd, H->P + L.off_b2, uni, rng, H->X, H->Dhi, H->Dlo, H->lp_part, 0, {}, 0.0};
  H->tail_tiles = TailSampleEpi::kParts * ((ncols + BN - 1) / BN);  // one partial per epilogue set
  launch_umma<BN, false, false>(H, "z2_tail_umma", ah, al, bh, bl, B, ncols, L.h, 1, e, H->stream);
}

void launch_dg1_umma(Handle* H, int B) {
  const Layout& L = H->L;
  constexpr int BN = 256;
  const int mt = (B + kUmmaBM - 1) / kUmmaBM, nt = (L.h + BN - 1) / BN;
  const int nkb = (L.n + kUmmaBK - 1) / kUmmaBK;
  int splits = std::max(1, std::min(nkb, 148 / (mt * nt)));  // one tile per SM
  splits = std::min(splits, H->max_splits);
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  H->splits = splits;
  const CUtensorMap ah = tmap_kmajor(H->Dhi, L.n, B, H->np, kUmmaBM);
  const CUtensorMap al = tmap_kmajor(H->Dlo, L.n, B, H->np, kUmmaBM);
  const CUtensorMap bh = tmap_mnmajor(H->W2hi, L.h, L.n, H->hp, BN);
  const CUtensorMap bl = tmap_mnmajor(H->W2lo, L.h, L.n, H->hp, BN);
  PartialEpi e{H->Epart, B, L.h, 0, {}};
  launch_umma<BN, false, true>(H, "bw_dg1_umma", ah, al, bh, bl, B, L.h, L.n, splits, e, H->stream);
}

void launch_gw2_umma(Handle* H, int B) {  // BN = 128: 3-stage ring, 4 column tiles of h + 1
  const Layout& L = H->L;
  {
    const int64_t total = (int64_t)B * H->hp1;
    KScope ks(H, "wg1_split");
    wg1_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(B, L.h, H->hp1, H->G1, H->w, H->wG1hi,
                                                                       H->wG1lo);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  constexpr int BN = 128;
  const CUtensorMap ah = tmap_mnmajor(H->Dhi, L.n, B, H->np, kUmmaBM);
  const CUtensorMap al = tmap_mnmajor(H->Dlo, L.n, B, H->np, kUmmaBM);
  const CUtensorMap bh = tmap_mnmajor(H->wG1hi, L.h + 1, B, H->hp1, BN);
  const CUtensorMap bl = tmap_mnmajor(H->wG1lo, L.h + 1, B, H->hp1, BN);
  Gw2Epi e{L.n, L.h, 0, {}, H->d_deg, H->G + L.off_w2, H->G + L.off_b2};
  launch_umma<BN, true, true>(H, "bw_gw2_umma", ah, al, bh, bl, L.n, L.h + 1, B, 1, e, H->stream);
}

// gW1T[j][k] = sum_b X[b][j] dz1[b][k] (j < Hd) and gb1[k] (the ones column j = Hd):
// split-K partials into gw1_part, reduced and masked by gw1_finalize_kernel.  The spins
// are exact in tf32, so A is single (two MMA passes).
void launch_gw1_umma(Handle* H, int B, int& splits_out) {
  const Layout& L = H->L;
  constexpr int BN = 128;
  const int mt = (L.Hd + 1 + kUmmaBM - 1) / kUmmaBM, nt = (L.h + BN - 1) / BN;
  const int nkb = (B + kUmmaBK - 1) / kUmmaBK;
  int splits = std::max(1, std::min(std::min(nkb, kGw1MaxSplits), 148 / (mt * nt)));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  splits_out = splits;
  const CUtensorMap a = tmap_mnmajor(H->Xf, L.Hd + 1, B, H->hd1p, kUmmaBM);
  const CUtensorMap bh = tmap_mnmajor(H->dz1hi, L.h, B, H->hp, BN);
  const CUtensorMap bl = tmap_mnmajor(H->dz1lo, L.h, B, H->hp, BN);
  PartialEpi e{H->gw1_part, L.Hd + 1, L.h, 0, {}};
  launch_umma<BN, true, true, PartialEpi, true>(H, "bw_gw1_umma", a, a, bh, bl, L.Hd + 1, L.h, B, splits, e,
                                                 H->stream);
}

}  // namespace vqmc_b200

// ===========================================================================
// Test hook: C = A B^T through the 3xTF32 tcgen05 kernel on host fp32 arrays.
//   a_mn = 0: A is [M][K] (K-major); 1: A is [K][M] (MN-major).  Same for B with N.
// ===========================================================================
using namespace vqmc_b200;

extern "C" int vqmc_test_umma_gemm(int M, int N, int K, int a_mn, int b_mn, int bn, int splits,
                                   const float* A, const float* Bm, float* C) {
  float *dA = nullptr, *dB = nullptr, *dAh = nullptr, *dAl = nullptr, *dBh = nullptr, *dBl = nullptr,
        *dC = nullptr;
  try {
    const int lda = a_mn ? ((M + 3) & ~3) : ((K + 3) & ~3);
    const int arows = a_mn ? K : M, acols = a_mn ? M : K;
    const int ldb = b_mn ? ((N + 3) & ~3) : ((K + 3) & ~3);
    const int brows = b_mn ? K : N, bcols = b_mn ? N : K;
    const size_t pad = 64;
    VQMC_CUDA(cudaMalloc(&dA, sizeof(float) * arows * acols));
    VQMC_CUDA(cudaMalloc(&dB, sizeof(float) * brows * bcols));
    VQMC_CUDA(cudaMalloc(&dAh, sizeof(float) * ((size_t)arows * lda + pad)));
    VQMC_CUDA(cudaMalloc(&dAl, sizeof(float) * ((size_t)arows * lda + pad)));
    VQMC_CUDA(cudaMalloc(&dBh, sizeof(float) * ((size_t)brows * ldb + pad)));
    VQMC_CUDA(cudaMalloc(&dBl, sizeof(float) * ((size_t)brows * ldb + pad)));
    VQMC_CUDA(cudaMalloc(&dC, sizeof(float) * (size_t)splits * M * N));
    VQMC_CUDA(cudaMemcpy(dA, A, sizeof(float) * arows * acols, cudaMemcpyHostToDevice));
    VQMC_CUDA(cudaMemcpy(dB, Bm, sizeof(float) * brows * bcols, cudaMemcpyHostToDevice));
    VQMC_CUDA(cudaMemset(dAh, 0, sizeof(float) * ((size_t)arows * lda + pad)));
    VQMC_CUDA(cudaMemset(dAl, 0, sizeof(float) * ((size_t)arows * lda + pad)));
    VQMC_CUDA(cudaMemset(dBh, 0, sizeof(float) * ((size_t)brows * ldb + pad)));
    VQMC_CUDA(cudaMemset(dBl, 0, sizeof(float) * ((size_t)brows * ldb + pad)));
    split_rows_kernel<<<(unsigned)(((int64_t)arows * lda + 255) / 256), 256>>>(arows, acols, acols, lda, dA, dAh, dAl);
    split_rows_kernel<<<(unsigned)(((int64_t)brows * ldb + 255) / 256), 256>>>(brows, bcols, bcols, ldb, dB, dBh, dBl);
    VQMC_CUDA(cudaGetLastError());
    CUtensorMap ah, al, bh, bl;
    const int bnv = bn == 256 ? 256 : 128;
    if (a_mn) { ah = tmap_mnmajor(dAh, M, K, lda, kUmmaBM); al = tmap_mnmajor(dAl, M, K, lda, kUmmaBM); }
    else { ah = tmap_kmajor(dAh, K, M, lda, kUmmaBM); al = tmap_kmajor(dAl, K, M, lda, kUmmaBM); }
    if (b_mn) { bh = tmap_mnmajor(dBh, N, K, ldb, bnv); bl = tmap_mnmajor(dBl, N, K, ldb, bnv); }
    else { bh = tmap_kmajor(dBh, K, N, ldb, bnv); bl = tmap_kmajor(dBl, K, N, ldb, bnv); }
    PartialEpi e{dC, M, N, 0, {}};
#define GO(BNV, AM, BM_)                                                                       \
  launch_umma<BNV, AM, BM_>(nullptr, "test", ah, al, bh, bl, M, N, K, splits, e, (cudaStream_t)0)
    if (bnv == 128) {
      if (!a_mn && !b_mn) GO(128, false, false);
      else if (!a_mn && b_mn) GO(128, false, true);
      else if (a_mn && !b_mn) GO(128, true, false);
      else GO(128, true, true);
    } else {
      if (!a_mn && !b_mn) GO(256, false, false);
      else if (!a_mn && b_mn) GO(256, false, true);
      else if (a_mn && !b_mn) GO(256, true, false);
      else GO(256, true, true);
    }
#undef GO
    VQMC_CUDA(cudaDeviceSynchronize());
    VQMC_CUDA(cudaMemcpy(C, dC, sizeof(float) * (size_t)splits * M * N, cudaMemcpyDeviceToHost));
  } catch (const std::exception& ex) {
    set_error(ex.what());
    for (float* p : {dA, dB, dAh, dAl, dBh, dBl, dC}) if (p) cudaFree(p);
    return status_of(ex);
  }
  for (float* p : {dA, dB, dAh, dAl, dBh, dBl, dC}) if (p) cudaFree(p);
  return VQMC_OK;
}
