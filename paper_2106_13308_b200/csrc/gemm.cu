// tcgen05 (3xTF32) GEMMs of the VQMC step and their fused epilogues:
//
//   tail sampler   Z[b][i]  = G1[b] . W2m[i] + b2[i], i >= Hd      (A = G1 K-major, B = W2 K-major)
//                  epilogue: draw x = [u < p], pack bits, D = 0.5 (x - p_raw), log-prob partials
//   dg1 (split-K)  E[b][k]  = sum_i D[b][i] W2m[i][k]              (A = D K-major, B = W2 MN-major)
//   gW2 (+ gb2)    gW2[i][k] = sum_b D[b][i] w_b G1[b][k]          (A = D^T MN-major, B = wG1 MN-major)
// The tail sampler uses 3xTF32 (the draw x = [u < p] needs fp32-grade logits); the backward
// GEMMs use bf16 pairs (3 x kind::f16: 2x the tf32 rate, half the operand bytes; gradient
// error ~2^-16 relative, inside the stated 1e-4 tolerance).
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

// K-major operand: element (mn, k) at ptr[mn * ld + k]; box {128 bytes of K, box_mn}.
CUtensorMap tmap_kmajor(const void* ptr, int64_t K, int64_t MN, int64_t ld, int box_mn, bool bf16 = false) {
  CUtensorMap m;
  const int es = bf16 ? 2 : 4;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)MN};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)box_mn};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                           const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (K-major) failed: " + std::to_string((int)r));
  return m;
}

// MN-major operand: element (mn, k) at ptr[k * ld + mn]; 3D view {A, K, ceil(MN/A)} with
// A = 128 bytes of MN (the UMMA atom), box {A, 128 bytes of K, box_mn / A}.  tf32 uses the
// 128-byte swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B), bf16 the plain 128-byte one.
// Reads up to one atom past MN on the last chunk: the allocation must be padded and those
// rows/columns of the result are discarded.
CUtensorMap tmap_mnmajor(const void* ptr, int64_t MN, int64_t K, int64_t ld, int box_mn, bool bf16 = false) {
  CUtensorMap m;
  const int es = bf16 ? 2 : 4, A = 128 / es;
  const cuuint64_t dims[3] = {(cuuint64_t)A, (cuuint64_t)K, (cuuint64_t)((MN + A - 1) / A)};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * es, 128};
  const cuuint32_t box[3] = {(cuuint32_t)A, (cuuint32_t)A, (cuuint32_t)(box_mn / A)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (MN-major) failed: " + std::to_string((int)r));
  return m;
}

template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT = false, bool BF16 = false>
static void launch_umma(Handle* H, const char* name, const CUtensorMap& ah, const CUtensorMap& al,
                        const CUtensorMap& bh, const CUtensorMap& bl, int M, int N, int K, int splits, Epi epi,
                        cudaStream_t stream) {
  using Cfg = UmmaCfg<BN>;
  auto kern = umma_tf32x3_kernel<BN, A_MN, B_MN, Epi, A_EXACT, BF16>;
  static bool attr = false;
  if (!attr) {
    VQMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr = true;
  }
  const int nkb = (K + UmmaElem<BF16>::kBK - 1) / UmmaElem<BF16>::kBK;
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
  __nv_bfloat16* Dh;  // D as bf16 pairs [B][np] (operand of the bf16x3 backward GEMMs)
  __nv_bfloat16* Dl;
  double* lp_part;  // nullptr: the caller does not need log psi (training step): skip the log terms
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
      __nv_bfloat16 hi4[4], lo4[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = cb + j + t;
        const bool valid = c >= col_lo && c < n;
        const float z = v[j + t] + (valid ? b2[c] : 0.f);
        const UnitPre q = lp_part ? unit_pre(z) : unit_pre_nolog(z);
        int x;
        if (uni == nullptr) {
          thr[t] = (float)(q.p() * 4294967296.0);
          x = (valid && (float)r[t] + 0.5f < thr[t]) ? 1 : 0;
        } else {
          x = (valid && uni[(size_t)c * B + b] < q.p()) ? 1 : 0;
        }
        word |= (uint32_t)x << (j + t);
        const Unit o = unit_post(q, x);
        ptx::split_bf16(o.D, hi4[t], lo4[t]);
        if (lp_part && valid) lsum += o.logt;
      }
      if (full) {
        *reinterpret_cast<uint2*>(Dh + rowD + cb + j) = *reinterpret_cast<const uint2*>(hi4);
        *reinterpret_cast<uint2*>(Dl + rowD + cb + j) = *reinterpret_cast<const uint2*>(lo4);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = cb + j + t;
          if (c >= col_lo && c < n) {
            Dh[rowD + c] = hi4[t];
            Dl[rowD + c] = lo4[t];
          }
        }
      }
    }
    lps += (double)lsum;
    if (word) atomicOr(&X[(size_t)b * W + (cb >> 5)], word);
  }
  __device__ void end_row(int b, const UmmaArgs&) {
    if (lp_part && b < B) lp_part[(size_t)(kParts * tile.tn + part) * B + b] = lps;
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

__global__ void split_rows_bf16_kernel(int rows, int cols, int ld_in, int ld_out, const float* __restrict__ in,
                                       __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * ld_out) return;
  const int r = (int)(t / ld_out), c = (int)(t % ld_out);
  const float x = c < cols ? in[(size_t)r * ld_in + c] : 0.f;
  ptx::split_bf16(x, hi[t], lo[t]);
}

// wG1[b][k] = w_b * G1[b][k] (k < h), w_b (k == h), 0 (k > h); split into bf16 hi/lo.
__global__ void wg1_kernel(int B, int h, int ld, const float* __restrict__ G1, const float* __restrict__ w,
                           __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * ld) return;
  const int b = (int)(t / ld), k = (int)(t % ld);
  const float x = k < h ? w[b] * G1[(size_t)b * h + k] : (k == h ? w[b] : 0.f);
  ptx::split_bf16(x, hi[t], lo[t]);
}

// W2m -> tf32 pair (tail sampler GEMM) and bf16 pair (dg1 GEMM), after set_params.
void launch_split_w2(Handle* H) {
  const Layout& L = H->L;
  KScope ks(H, "split_w2");
  int64_t total = (int64_t)L.n * H->hp;
  split_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(L.n, L.h, L.h, H->hp, H->P + L.off_w2,
                                                                            H->W2hi, H->W2lo);
  VQMC_CUDA(cudaGetLastError());
  total = (int64_t)L.n * H->hp8;
  split_rows_bf16_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(
      L.n, L.h, L.h, H->hp8, H->P + L.off_w2, H->W2bh, H->W2bl);
  VQMC_CUDA(cudaGetLastError());
  H->launches += 2;
}

// ===========================================================================
// Production launchers
// ===========================================================================
void launch_tail_umma(Handle* H, int B, const double* uni, RngSpec rng, bool want_lp) {
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
  TailSampleEpi e{B, L.n, H->np8, L.W, colbase, L.Hd, H->P + L.off_b2, uni, rng, H->X, H->Dbh, H->Dbl,
                  want_lp ? H->lp_part : nullptr, 0, {}, 0.0};
  H->tail_tiles = TailSampleEpi::kParts * ((ncols + BN - 1) / BN);  // one partial per epilogue set
  launch_umma<BN, false, false>(H, "z2_tail_umma", ah, al, bh, bl, B, ncols, L.h, 1, e, H->stream);
}

void launch_dg1_umma(Handle* H, int B) {
  const Layout& L = H->L;
  constexpr int BN = 256;
  const int mt = (B + kUmmaBM - 1) / kUmmaBM, nt = (L.h + BN - 1) / BN;
  const int nkb = (L.n + UmmaElem<true>::kBK - 1) / UmmaElem<true>::kBK;
  int splits = std::max(1, std::min(nkb, 148 / (mt * nt)));  // one tile per SM
  splits = std::min(splits, H->max_splits);
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  H->splits = splits;
  const CUtensorMap ah = tmap_kmajor(H->Dbh, L.n, B, H->np8, kUmmaBM, true);
  const CUtensorMap al = tmap_kmajor(H->Dbl, L.n, B, H->np8, kUmmaBM, true);
  const CUtensorMap bh = tmap_mnmajor(H->W2bh, L.h, L.n, H->hp8, BN, true);
  const CUtensorMap bl = tmap_mnmajor(H->W2bl, L.h, L.n, H->hp8, BN, true);
  PartialEpi e{H->Epart, B, L.h, 0, {}};
  launch_umma<BN, false, true, PartialEpi, false, true>(H, "bw_dg1_umma", ah, al, bh, bl, B, L.h, L.n, splits, e,
                                                         H->stream);
}

void launch_gw2_umma(Handle* H, int B) {  // BN = 128: 3-stage ring, 4 column tiles of h + 1
  const Layout& L = H->L;
  {
    const int64_t total = (int64_t)B * H->hp18;
    KScope ks(H, "wg1_split");
    wg1_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(B, L.h, H->hp18, H->G1, H->w, H->wG1bh,
                                                                       H->wG1bl);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  constexpr int BN = 128;
  const CUtensorMap ah = tmap_mnmajor(H->Dbh, L.n, B, H->np8, kUmmaBM, true);
  const CUtensorMap al = tmap_mnmajor(H->Dbl, L.n, B, H->np8, kUmmaBM, true);
  const CUtensorMap bh = tmap_mnmajor(H->wG1bh, L.h + 1, B, H->hp18, BN, true);
  const CUtensorMap bl = tmap_mnmajor(H->wG1bl, L.h + 1, B, H->hp18, BN, true);
  Gw2Epi e{L.n, L.h, 0, {}, H->d_deg, H->G + L.off_w2, H->G + L.off_b2};
  launch_umma<BN, true, true, Gw2Epi, false, true>(H, "bw_gw2_umma", ah, al, bh, bl, L.n, L.h + 1, B, 1, e,
                                                    H->stream);
}

// gW1T[j][k] = sum_b X[b][j] dz1[b][k] (j < Hd) and gb1[k] (the ones column j = Hd):
// split-K partials into gw1_part, reduced and masked by gw1_finalize_kernel.  The spins
// are exact in bf16, so A is single (two MMA passes).
void launch_gw1_umma(Handle* H, int B, int& splits_out) {
  const Layout& L = H->L;
  constexpr int BN = 128;
  const int mt = (L.Hd + 1 + kUmmaBM - 1) / kUmmaBM, nt = (L.h + BN - 1) / BN;
  const int nkb = (B + UmmaElem<true>::kBK - 1) / UmmaElem<true>::kBK;
  int splits = std::max(1, std::min(std::min(nkb, kGw1MaxSplits), 148 / (mt * nt)));
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  splits_out = splits;
  const CUtensorMap a = tmap_mnmajor(H->Xfb, L.Hd + 1, B, H->hd18, kUmmaBM, true);
  const CUtensorMap bh = tmap_mnmajor(H->dz1bh, L.h, B, H->hp8, BN, true);
  const CUtensorMap bl = tmap_mnmajor(H->dz1bl, L.h, B, H->hp8, BN, true);
  PartialEpi e{H->gw1_part, L.Hd + 1, L.h, 0, {}};
  launch_umma<BN, true, true, PartialEpi, true, true>(H, "bw_gw1_umma", a, a, bh, bl, L.Hd + 1, L.h, B, splits, e,
                                                       H->stream);
}

}  // namespace vqmc_b200

// ===========================================================================
// Test hook: C = A B^T through the 3xTF32 tcgen05 kernel on host fp32 arrays.
//   a_mn = 0: A is [M][K] (K-major); 1: A is [K][M] (MN-major).  Same for B with N.
// ===========================================================================
using namespace vqmc_b200;

extern "C" int vqmc_test_umma_gemm(int M, int N, int K, int a_mn, int b_mn, int bn, int splits, int bf16,
                                   const float* A, const float* Bm, float* C) {
  void *dA = nullptr, *dB = nullptr, *dAh = nullptr, *dAl = nullptr, *dBh = nullptr, *dBl = nullptr;
  float* dC = nullptr;
  auto release = [&]() {
    for (void* p : {dA, dB, dAh, dAl, dBh, dBl, (void*)dC})
      if (p) cudaFree(p);
  };
  try {
    const int q = bf16 ? 8 : 4, es = bf16 ? 2 : 4;
    const int lda = a_mn ? ((M + q - 1) / q * q) : ((K + q - 1) / q * q);
    const int arows = a_mn ? K : M, acols = a_mn ? M : K;
    const int ldb = b_mn ? ((N + q - 1) / q * q) : ((K + q - 1) / q * q);
    const int brows = b_mn ? K : N, bcols = b_mn ? N : K;
    const size_t pad = 128;
    const size_t asz = ((size_t)arows * lda + pad) * es, bsz = ((size_t)brows * ldb + pad) * es;
    VQMC_CUDA(cudaMalloc(&dA, sizeof(float) * arows * acols));
    VQMC_CUDA(cudaMalloc(&dB, sizeof(float) * brows * bcols));
    VQMC_CUDA(cudaMalloc(&dAh, asz));
    VQMC_CUDA(cudaMalloc(&dAl, asz));
    VQMC_CUDA(cudaMalloc(&dBh, bsz));
    VQMC_CUDA(cudaMalloc(&dBl, bsz));
    VQMC_CUDA(cudaMalloc(&dC, sizeof(float) * (size_t)splits * M * N));
    VQMC_CUDA(cudaMemcpy(dA, A, sizeof(float) * arows * acols, cudaMemcpyHostToDevice));
    VQMC_CUDA(cudaMemcpy(dB, Bm, sizeof(float) * brows * bcols, cudaMemcpyHostToDevice));
    for (void* p : {dAh, dAl}) VQMC_CUDA(cudaMemset(p, 0, asz));
    for (void* p : {dBh, dBl}) VQMC_CUDA(cudaMemset(p, 0, bsz));
    const unsigned ga = (unsigned)(((int64_t)arows * lda + 255) / 256), gb = (unsigned)(((int64_t)brows * ldb + 255) / 256);
    if (bf16) {
      split_rows_bf16_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, (__nv_bfloat16*)dAh,
                                          (__nv_bfloat16*)dAl);
      split_rows_bf16_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, (__nv_bfloat16*)dBh,
                                          (__nv_bfloat16*)dBl);
    } else {
      split_rows_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, (float*)dAh, (float*)dAl);
      split_rows_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, (float*)dBh, (float*)dBl);
    }
    VQMC_CUDA(cudaGetLastError());
    const int bnv = bn == 256 ? 256 : 128;
    const bool b16 = bf16 != 0;
    CUtensorMap ah, al, bh, bl;
    if (a_mn) { ah = tmap_mnmajor(dAh, M, K, lda, kUmmaBM, b16); al = tmap_mnmajor(dAl, M, K, lda, kUmmaBM, b16); }
    else { ah = tmap_kmajor(dAh, K, M, lda, kUmmaBM, b16); al = tmap_kmajor(dAl, K, M, lda, kUmmaBM, b16); }
    if (b_mn) { bh = tmap_mnmajor(dBh, N, K, ldb, bnv, b16); bl = tmap_mnmajor(dBl, N, K, ldb, bnv, b16); }
    else { bh = tmap_kmajor(dBh, K, N, ldb, bnv, b16); bl = tmap_kmajor(dBl, K, N, ldb, bnv, b16); }
    PartialEpi e{dC, M, N, 0, {}};
#define GO(BNV, AM, BM_, BF)                                                                          \
  launch_umma<BNV, AM, BM_, PartialEpi, false, BF>(nullptr, "test", ah, al, bh, bl, M, N, K, splits, e, \
                                                  (cudaStream_t)0)
#define GO4(BNV, BF)                             \
  if (!a_mn && !b_mn) GO(BNV, false, false, BF); \
  else if (!a_mn && b_mn) GO(BNV, false, true, BF); \
  else if (a_mn && !b_mn) GO(BNV, true, false, BF); \
  else GO(BNV, true, true, BF)
    if (bnv == 128) {
      if (b16) { GO4(128, true); } else { GO4(128, false); }
    } else {
      if (b16) { GO4(256, true); } else { GO4(256, false); }
    }
#undef GO4
#undef GO
    VQMC_CUDA(cudaDeviceSynchronize());
    VQMC_CUDA(cudaMemcpy(C, dC, sizeof(float) * (size_t)splits * M * N, cudaMemcpyDeviceToHost));
  } catch (const std::exception& ex) {
    set_error(ex.what());
    release();
    return status_of(ex);
  }
  release();
  return VQMC_OK;
}
