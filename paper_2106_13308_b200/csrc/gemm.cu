// tcgen05 3-pass (fp16-pair) GEMMs of the VQMC step and their fused epilogues:
//
//   tail sampler   Z[b][i]  = [G1[b] 1] . [W2m[i] b2[i]], i >= Hd  (A = G1 K-major, B = W2 K-major)
//                  epilogue: draw x = [u < p], pack bits, D = 0.5 (x - p_raw), log-prob partials
//   dg1 (split-K)  E[b][k]  = sum_i D[b][i] W2m[i][k]              (A = D K-major, B = W2 MN-major)
//   gW2 (+ gb2)    gW2[i][k] = sum_b D[b][i] w_b G1[b][k]          (A = D^T MN-major, B = wG1 MN-major)
//   gW1 (+ gb1)    gW1T[j][k] = sum_b X[b][j] dz1[b][k]            (A = X^T MN-major, B = dz1 MN-major)
// Operands are stored as fp16 pairs x = hi + lo (22 significant bits) and every GEMM runs three
// kind::f16 passes hi.hi + hi.lo + lo.hi with fp32 accumulation in TMEM: fp32-grade logits for
// the draw x = [u < p] at 2x the tf32 rate and half its bytes.  fp16's range is kept safe by
// construction: D in [-1/2, 1/2], REINFORCE weights normalised to |w'| <= 1 (the epilogues
// multiply by the power-of-two wscale), and a sticky flag for non-finite logits.  gW1 keeps
// bf16 pairs (dz1 is unbounded; the spins are exact).
//
// Reference: made_forward / auto_sample / weighted_grad_log_psi, proj/src/models.cpp:51-62,
// 175-198 and proj/src/sampler.cpp:47-55.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "internal.cuh"
#include "ptx.cuh"
#include "umma_gemm.cuh"
#include "umma2_gemm.cuh"

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

static CUtensorMapDataType tmap_dtype(int ek) {
  return ek == kElemTF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                         : ek == kElemBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                         : ek == kElemU8   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
}
static int tmap_esize(int ek) { return ek == kElemTF32 ? 4 : ek == kElemU8 ? 1 : 2; }

// K-major operand: element (mn, k) at ptr[mn * ld + k]; box {128 bytes of K, box_mn}.
CUtensorMap tmap_kmajor(const void* ptr, int64_t K, int64_t MN, int64_t ld, int box_mn, int ek = kElemTF32) {
  CUtensorMap m;
  const int es = tmap_esize(ek);
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)MN};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)box_mn};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, tmap_dtype(ek), 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (K-major) failed: " + std::to_string((int)r));
  return m;
}

// MN-major operand: element (mn, k) at ptr[k * ld + mn]; 3D view {A, K, ceil(MN/A)} with
// A = 128 bytes of MN (the UMMA atom), box {A, 128 bytes of K, box_mn / A}.  tf32 uses the
// 128-byte swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B), 16-bit types the plain 128-byte one.
// Reads up to one atom past MN on the last chunk: the allocation must be padded and those
// rows/columns of the result are discarded.
CUtensorMap tmap_mnmajor(const void* ptr, int64_t MN, int64_t K, int64_t ld, int box_mn, int ek = kElemTF32) {
  CUtensorMap m;
  const int es = ek ? 2 : 4, A = 128 / es;
  const cuuint64_t dims[3] = {(cuuint64_t)A, (cuuint64_t)K, (cuuint64_t)((MN + A - 1) / A)};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * es, 128};
  const cuuint32_t box[3] = {(cuuint32_t)A, (cuuint32_t)A, (cuuint32_t)(box_mn / A)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, tmap_dtype(ek), 3, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           ek ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (MN-major) failed: " + std::to_string((int)r));
  return m;
}

int gemm_sms(const Handle* H) {
  static int sms = 0;
  if (!sms) VQMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (!H) return sms;
  int n = sms - H->gemm_sm_reserve;
  if (H->gemm_sm_cap > 0) n = std::min(n, H->gemm_sm_cap);
  return std::max(2, n & ~1);
}

template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT = false, int EK = kElemTF32>
static void launch_umma(Handle* H, const char* name, const CUtensorMap& ah, const CUtensorMap& al,
                        const CUtensorMap& bh, const CUtensorMap& bl, int M, int N, int K, int splits, Epi epi,
                        cudaStream_t stream) {
  using Cfg = UmmaCfg<BN>;
  auto kern = umma3p_kernel<BN, A_MN, B_MN, Epi, A_EXACT, EK>;
  ensure_smem_attr((const void*)kern, Cfg::kSmem);
  const int nkb = (K + UmmaElem<EK>::kBK - 1) / UmmaElem<EK>::kBK;
  UmmaArgs args{M, N, K, (nkb + splits - 1) / splits, (N + BN - 1) / BN, (M + kUmmaBM - 1) / kUmmaBM, splits};
  const int ntiles = args.tiles_n * args.tiles_m * splits;
  const int grid = std::min(ntiles, gemm_sms(H));
  if (H) {
    KScope ks(H, name);
    launch_k(H, kern, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, ah, al, bh, bl, args, epi);
    H->launches++;
  } else {
    kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(ah, al, bh, bl, args, epi);
  }
  VQMC_CUDA(cudaGetLastError());
}

// CTA-pair launch: clusters of 2, one pair per 2 SMs (persistent over pair tiles of 256 x BN).
template <int BN, bool A_MN, bool B_MN, class Epi, bool A_EXACT, int EK, int SETS = 0, int CHUNK = 32>
static void launch_umma2(Handle* H, const char* name, const CUtensorMap& ah, const CUtensorMap& al,
                         const CUtensorMap& bh, const CUtensorMap& bl, int M, int N, int K, int splits, Epi epi,
                         cudaStream_t stream) {
  using Cfg = Umma2Cfg<BN, SETS, CHUNK>;
  auto kern = umma2_kernel<BN, A_MN, B_MN, Epi, A_EXACT, EK, SETS, CHUNK>;
  ensure_smem_attr((const void*)kern, Cfg::kSmem);
  const int nkb = (K + Cfg::kBK - 1) / Cfg::kBK;
  UmmaArgs args{M, N, K, (nkb + splits - 1) / splits, (N + BN - 1) / BN, (M + 2 * kUmmaBM - 1) / (2 * kUmmaBM), splits};
  const int ntiles = args.tiles_n * args.tiles_m * splits;
  const int pairs = std::min(ntiles, gemm_sms(H) / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  int na = 1;
  if (H && H->pdl) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (H && (stream == H->stream || H->ktimer == 2)) {  // (timeline mode: events on the side stream too)
    KScope ks(H, name, stream);
    VQMC_CUDA(cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, args, epi));
    H->launches++;
  } else {
    VQMC_CUDA(cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, args, epi));
    if (H) H->launches++;
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
  __device__ void init() {}
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int row, int col0, const float (&v)[32], const UmmaArgs& a) {
    if (row >= a.M) return;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < a.N) C[(size_t)row * ldc + col0 + j] = v[j];
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// Tail sampler: rows = samples, columns = outputs colbase + col (col0 aligned to 32, so a
// chunk is exactly one word of the packed spins).  The logit arrives complete (b2 rides in the
// GEMM as column h), so per output the epilogue is: sigmoid (ex2 + rcp), the draw, D and its fp16
// pair; Philox keys are per row.  The epilogue warp sets take alternate 32-column chunks and
// each writes its own log-prob partial (lp_part[kParts * tile + part]): deterministic.
// (kTailBN: internal.cuh)
// kTailCh: accumulator columns per epilogue call of the tail sampler; the 12 16-column chunks of a
// 192-column tile split evenly over 3 epilogue sets (12 epilogue warps at up to 128 registers:
// 43.0 us; 4 sets at 96 registers: 44.3 us).
constexpr int kTailCh = 16;
constexpr int kTailSets = kTailCh == 16 ? 3 : 0;
template <bool PROD>  // PROD: production draws (Philox) and no log-probabilities (the training step)
struct TailSampleEpiT {
  static constexpr int CH = kTailCh;
  int B, n, np, W, colbase, col_lo;  // outputs in [col_lo, n) are drawn here
  const double* uni;
  RngSpec rng;
  uint32_t* X;
  __half* Dh;  // D as fp16 pairs [B][np] (operand of the backward GEMMs)
  __half* Dl;
  double* lp_part;  // nullptr: the caller does not need log psi (training step): skip the log terms
  uint32_t* flag;   // set when a logit is not finite (fp16 operand overflow)
  int part;
  UmmaTile tile;
  double lps;
  uint32_t k0, k1, c1, c2, c3;  // Philox key and counter words of this row (production draws)
  __device__ void init() {
    if (PROD || uni == nullptr) {
      const uint64_t call = rng.c();  // (device step counter: loaded once per thread)
      c2 = (uint32_t)call;
      c3 = (uint32_t)(call >> 32);
    }
  }
  __device__ void begin_row(int b, const UmmaArgs&) {
    if (!PROD) lps = 0.0;
    if ((PROD || uni == nullptr) && b < B) {
      const int s = b / rng.seg;
      const uint64_t key = mix_seed_dev(rng.seed, rng.stream0 + (uint64_t)s);
      k0 = (uint32_t)key;
      k1 = (uint32_t)(key >> 32);
      c1 = (uint32_t)(b - s * rng.seg);
    }
  }
  __device__ void chunk(int b, int col0, const float (&v)[CH], const UmmaArgs& a) {
    if (b >= B) return;
    const int cb = colbase + col0;
    if (cb >= col_lo && cb + CH <= n) chunk_t<true>(b, cb, v);  // every output of the chunk is drawn here
    else chunk_t<false>(b, cb, v);
  }
  template <bool FULL>
  __device__ __forceinline__ void chunk_t(int b, int cb, const float (&v)[CH]) {
    constexpr bool full = FULL;
    constexpr float kThrLo = (float)(kProbEps * 4294967296.0), kThrHi = (float)((1.0 - kProbEps) * 4294967296.0);
    const size_t rowD = (size_t)b * np;
    uint32_t word = 0;
    float lsum = 0.f;  // CH log terms in fp32, then one fp64 add
    float nanacc = 0.f;
#pragma unroll
    for (int jh = 0; jh < CH; jh += 16) {  // halves of 16 outputs: 16-byte stores, fewer live registers
      uint32_t dh[8], dl[8];
#pragma unroll
      for (int j = jh; j < jh + 16; j += 4) {
        uint32_t r[4];
#ifdef VQMC_TAIL_TRACE
        if (g_tail_exp & 2) {
          r[0] = r[1] = r[2] = r[3] = c1 * 2654435761u + (uint32_t)(cb + j);
        } else
#endif
        if (PROD || uni == nullptr) philox4_k(k0, k1, (uint32_t)((cb + j) >> 2), c1, c2, c3, r);
        float d[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = cb + j + t;
          const bool valid = full || (c >= col_lo && c < n);
          const float z = v[j + t];
          const float a = fabsf(z);
          nanacc = fmaf(a, 0.f, nanacc);  // (stays 0 unless a logit is inf / NaN: one op per output)
          const float e = ptx::ex2_approx(a * -1.4426950408889634f);  // exp(-|z|)
          const float rr = ptx::rcp_approx(1.f + e);
          const float er = e * rr;
          const float praw = z >= 0.f ? rr : er, qraw = z >= 0.f ? er : rr;  // sigmoid(z), 1 - sigmoid(z)
          const bool clamp = a >= kLogitHi;                                     // models.hpp:26 clamp active
          bool x;
          if (PROD || uni == nullptr) {  // u = (r + 1/2) 2^-32 < clamp(p), as r < clamp(p) 2^32 - 1/2
            x = (float)r[t] < fminf(fmaxf(fmaf(praw, 4294967296.f, -0.5f), kThrLo - 0.5f), kThrHi - 0.5f);
          } else {
            const double p = clamp ? (z > 0.f ? 1.0 - kProbEps : kProbEps) : (double)praw;
            x = valid && uni[(size_t)c * B + b] < p;
          }
          x = x && valid;
          word |= (uint32_t)x << (j + t);
          d[t] = (clamp || !valid) ? 0.f : 0.5f * (x ? qraw : -praw);  // made_dz2, models.cpp:163-171
          if (!PROD && lp_part && valid) {
            const float L = log1pf(e);
            const float lg = clamp ? ((z > 0.f) == x ? -1.00000005e-7f : -16.11809565095832f)
                                   : -(x ? fmaxf(-z, 0.f) + L : fmaxf(z, 0.f) + L);
            lsum += lg;
          }
        }
        ptx::split_f16x2(d[0], d[1], dh[(j - jh) / 2], dl[(j - jh) / 2]);
        ptx::split_f16x2(d[2], d[3], dh[(j - jh) / 2 + 1], dl[(j - jh) / 2 + 1]);
      }
#ifdef VQMC_TAIL_TRACE
      if (g_tail_exp & 1) {
        if (dh[0] == 0x7fffffffu && dl[1] == 0x7fffffffu) atomicOr(flag, 4u);  // (keep the values live)
      } else
#endif
      if (full) {  // one full 32-byte sector per row and half (np % 16 == 0, cb % 16 == 0)
        ptx::st_global_v8(Dh + rowD + cb + jh, dh);
        ptx::st_global_v8(Dl + rowD + cb + jh, dl);
      } else {
        const __half* hh = reinterpret_cast<const __half*>(dh);
        const __half* hl = reinterpret_cast<const __half*>(dl);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int c = cb + jh + t;
          if (c >= col_lo && c < n) {
            Dh[rowD + c] = hh[t];
            Dl[rowD + c] = hl[t];
          }
        }
      }
    }
    if (!(nanacc == 0.f)) atomicOr(flag, 1u);
    uint32_t* xw = &X[(size_t)b * W + (cb >> 5)];
    if (CH == 32) {
      if (cb < col_lo) atomicOr(xw, word);  // shares the word with the head
      else *xw = word;
    } else {  // a 16-bit half of the word
      if (cb < col_lo) atomicOr(xw, word << (cb & 16));
      else reinterpret_cast<uint16_t*>(xw)[(cb >> 4) & 1] = (uint16_t)word;
    }
    if (!PROD) lps += (double)lsum;
  }
  __device__ void end_row(int b, const UmmaArgs&) {
    if (!PROD && lp_part && b < B) lp_part[(size_t)(kParts * tile.tn + part) * B + b] = lps;
  }
  static constexpr int kParts = Umma2Cfg<kTailBN, kTailSets, kTailCh>::kEpiSets;  // one log-prob partial per set
};

struct PartialEpi {  // split-K partial: out[z][row][col]
  float* out;
  int rows, cols;
  int part;
  UmmaTile tile;
  __device__ void init() {}
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int row, int col0, const float (&v)[32], const UmmaArgs&) {
    if (row >= rows) return;
    float* o = out + ((size_t)tile.z * rows + row) * cols;
    if ((cols & 3) == 0 && col0 + 32 <= cols) {  // 16-byte stores (row stride and col0 are multiples of 4)
      float4* o4 = reinterpret_cast<float4*>(o + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < cols) o[col0 + j] = v[j];
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// gW1 without split-K: rows j (j == Hd: the ones row -> gb1), columns k; (.) M1^T and x wscale.
struct Gw1Epi {
  int h, Hd;
  int part;
  UmmaTile tile;
  const int32_t* deg;
  const float* wscale;
  float* gW1T;
  float* gb1;
  float sc;
  __device__ void init() { sc = *wscale; }
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int j, int col0, const float (&v)[32], const UmmaArgs&) {
    if (j > Hd) return;
    if (j == Hd) {
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (col0 + t < h) gb1[col0 + t] = v[t] * sc;
      return;
    }
    float* o = gW1T + (size_t)j * h + col0;
    if ((h & 3) == 0 && col0 + 32 <= h) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 r;
        r.x = (j + 1 <= deg[col0 + 4 * q + 0]) ? v[4 * q + 0] * sc : 0.f;  // M1(k, j)
        r.y = (j + 1 <= deg[col0 + 4 * q + 1]) ? v[4 * q + 1] * sc : 0.f;
        r.z = (j + 1 <= deg[col0 + 4 * q + 2]) ? v[4 * q + 2] * sc : 0.f;
        r.w = (j + 1 <= deg[col0 + 4 * q + 3]) ? v[4 * q + 3] * sc : 0.f;
        reinterpret_cast<float4*>(o)[q] = r;
      }
      return;
    }
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (col0 + t < h) o[t] = (j + 1 <= deg[col0 + t]) ? v[t] * sc : 0.f;
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

struct Gw2Epi {  // rows = outputs i, columns = hidden k (k == h: bias column -> gb2)
  int n, h;
  int part;
  UmmaTile tile;
  const int32_t* deg;
  const float* wscale;  // the B operand carries w' = w / wscale
  float* gW2;
  float* gb2;
  __device__ void init() {}
  __device__ void begin_row(int, const UmmaArgs&) {}
  __device__ void chunk(int i, int col0, const float (&v)[32], const UmmaArgs&) {
    if (i >= n) return;
    const float sc = *wscale;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int k = col0 + j;
      if (k < h) gW2[(size_t)i * h + k] = (deg[k] < i + 1) ? v[j] * sc : 0.f;  // M2(i, k)
      else if (k == h) gb2[i] = v[j] * sc;
    }
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// gW2 computed transposed (pair kernel): rows = hidden k (k == h: the bias row -> gb2), columns =
// outputs i.  For a fixed column the 32 lanes (consecutive k) store 128 contiguous bytes.
struct Gw2TEpi {
  int n, h;
  int part;
  UmmaTile tile;
  const int32_t* deg;
  const float* wscale;  // the A operand carries w' = w / wscale
  float* gW2;
  float* gb2;
  float sc;
  int dk;
  __device__ void init() {}
  __device__ void begin_row(int k, const UmmaArgs&) {
    sc = *wscale;
    dk = k < h ? deg[k] : 0;
  }
  __device__ void chunk(int k, int col0, const float (&v)[32], const UmmaArgs&) {
    if (k > h) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int i = col0 + j;
      if (i >= n) break;
      if (k < h) gW2[(size_t)i * h + k] = (dk < i + 1) ? v[j] * sc : 0.f;  // M2(i, k)
      else gb2[i] = v[j] * sc;
    }
  }
  __device__ void end_row(int, const UmmaArgs&) {}
};

// SR operator (stochastic reconfiguration, optimizer.cpp:46-92): the W2 | b2 half of S p,
// sum_i D[b][i] Z[b][i] with Z = [G1 | 1] . [P2 | p2]^T the logits of the direction p.  Rows b,
// columns i over all n outputs; one fp64 partial per row and epilogue set per column tile.
struct SpDotEpi {
  int B, n, np;
  const __half* Dh;  // D (unweighted made_dz2) as an fp16 pair, [B][np]
  const __half* Dl;
  double* out;  // [kParts * tiles_n][B]
  int part;
  UmmaTile tile;
  double acc;
  static constexpr int kParts = Umma2Cfg<kTailBN>::kEpiSets;
  __device__ void init() {}
  __device__ void begin_row(int, const UmmaArgs&) { acc = 0.0; }
  __device__ void chunk(int b, int col0, const float (&v)[32], const UmmaArgs&) {
    if (b >= B) return;
    const __half* dh = Dh + (size_t)b * np + col0;
    const __half* dl = Dl + (size_t)b * np + col0;
    float s = 0.f;
    if (col0 + 32 <= n) {  // (np % 8 == 0 and col0 % 32 == 0: 16-byte loads)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 hv = reinterpret_cast<const uint4*>(dh)[q], lv = reinterpret_cast<const uint4*>(dl)[q];
        const __half2* h2 = reinterpret_cast<const __half2*>(&hv);
        const __half2* l2 = reinterpret_cast<const __half2*>(&lv);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 a = __half22float2(h2[t]), c = __half22float2(l2[t]);
          s = fmaf(a.x + c.x, v[8 * q + 2 * t], s);
          s = fmaf(a.y + c.y, v[8 * q + 2 * t + 1], s);
        }
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < n; ++j) s = fmaf(__half2float(dh[j]) + __half2float(dl[j]), v[j], s);
    }
    acc += (double)s;
  }
  __device__ void end_row(int b, const UmmaArgs&) {
    if (b < B) out[(size_t)(kParts * tile.tn + part) * B + b] = acc;
  }
};

// Forward of GIVEN configurations (made_forward + bernoulli_log_likelihood, models.cpp:51-70):
// rows = samples, columns = every output i (the layer-1 activations [G1 | 1] come from
// z1_given_kernel, so no sampling chain is involved).  Per output: the clamped conditional, the
// log term of the given bit (fp32, 32 per fp64 add), D = 0.5 (x - p_raw) as an fp16 pair (the
// backward's operand) and optionally p, log p_i(x_i) and log p_i(1 - x_i) - log p_i(x_i).
//
// NBR: the rows are single-site-flipped neighbours (estimator.hpp:64-72): row r is sample
// b0 + r % Bc with bit sites[r / Bc] flipped; only outputs i >= that site are summed (the earlier
// conditionals and terms are the unflipped sample's), and nothing but the log-prob partials is
// written.
template <bool NBR>
struct GivenEpiT {
  int rows, n, np, W;
  const uint32_t* X;
  __half* Dh;  // [B][np] (!NBR; nullptr: not written)
  __half* Dl;
  double* lp_part;  // [kParts * tiles_n][rows]
  double* cond;     // [B][n] clamped p (optional, !NBR)
  float* lterm;     // [B][n] log p_i(x_i) (optional, !NBR)
  float* fterm;     // [B][n] log p_i(1 - x_i) - log p_i(x_i) (optional, !NBR)
  uint32_t* flag;   // non-finite logit (fp16 operand overflow)
  int Bc, b0;       // NBR row map
  const int32_t* sites;
  int part;
  UmmaTile tile;
  double lps;
  int rb, rk;
  static constexpr int kParts = Umma2Cfg<kTailBN>::kEpiSets;
  __device__ void init() {}
  __device__ void begin_row(int r, const UmmaArgs&) {
    lps = 0.0;
    rb = r;
    rk = 0;
    if (NBR && r < rows) {
      rb = b0 + r % Bc;
      rk = sites[r / Bc];
    }
  }
  __device__ void chunk(int r, int cb, const float (&v)[32], const UmmaArgs&) {
    if (r >= rows) return;
    if (NBR && cb + 32 <= rk) return;  // every output of the chunk precedes the flipped site
    uint32_t word = X[(size_t)rb * W + (cb >> 5)];
    if (NBR && (rk >> 5) == (cb >> 5)) word ^= 1u << (rk & 31);
    const size_t rowe = (size_t)rb * n, rowD = (size_t)rb * np;
    float lsum = 0.f;
    bool bad = false;
#pragma unroll
    for (int jh = 0; jh < 32; jh += 16) {
      uint32_t dh[8], dl[8];
#pragma unroll
      for (int j = jh; j < jh + 16; j += 2) {
        float d[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int c = cb + j + t;
          const bool valid = c < n && (!NBR || c >= rk);
          const float z = v[j + t];
          bad |= !(fabsf(z) < INFINITY);
          const int x = (word >> (j + t)) & 1;
          const UnitPre q = unit_pre(z);
          const Unit u = unit_post(q, x);
          if (valid) lsum += u.logt;
          d[t] = valid ? u.D : 0.f;
          if (!NBR && valid) {
            if (cond) cond[rowe + c] = u.p;
            if (lterm) lterm[rowe + c] = u.logt;
            if (fterm) fterm[rowe + c] = unit_post(q, 1 - x).logt - u.logt;
          }
        }
        if (!NBR) ptx::split_f16x2(d[0], d[1], dh[(j - jh) / 2], dl[(j - jh) / 2]);
      }
      if (!NBR && Dh) {
        if (cb + 32 <= n) {
          ptx::st_global_v8(Dh + rowD + cb + jh, dh);
          ptx::st_global_v8(Dl + rowD + cb + jh, dl);
        } else {
          const __half* hh = reinterpret_cast<const __half*>(dh);
          const __half* hl = reinterpret_cast<const __half*>(dl);
          for (int t = 0; t < 16 && cb + jh + t < n; ++t) {
            Dh[rowD + cb + jh + t] = hh[t];
            Dl[rowD + cb + jh + t] = hl[t];
          }
        }
      }
    }
    if (bad) atomicOr(flag, 1u);
    lps += (double)lsum;
  }
  __device__ void end_row(int r, const UmmaArgs&) {
    if (r < rows) lp_part[(size_t)(kParts * tile.tn + part) * rows + r] = lps;
  }
};

// ===========================================================================
// Helper kernels: 16-bit pairs of operands
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

// rows x ld_out fp16 pair of [in | extra]: column `cols` holds extra[r] (if extra), zeros beyond.
__global__ void split_rows_f16_kernel(int rows, int cols, int ld_in, int ld_out, const float* __restrict__ in,
                                      const float* __restrict__ extra, __half* __restrict__ hi,
                                      __half* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)rows * ld_out) return;
  const int r = (int)(t / ld_out), c = (int)(t % ld_out);
  const float x = c < cols ? in[(size_t)r * ld_in + c] : ((c == cols && extra) ? extra[r] : 0.f);
  ptx::split_f16(x, hi[t], lo[t]);
}

// wG1[b][k] = w'_b * G1[b][k] (k < h), w'_b (k == h), 0 (k > h); split into an fp16 pair.
__global__ void wg1_kernel(int B, int h, int ld, const float* __restrict__ G1, const float* __restrict__ w,
                           __half* __restrict__ hi, __half* __restrict__ lo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * ld) return;
  const int b = (int)(t / ld), k = (int)(t % ld);
  const float x = k < h ? w[b] * G1[(size_t)b * h + k] : (k == h ? w[b] : 0.f);
  ptx::split_f16(x, hi[t], lo[t]);
}

// [W2m | b2] -> fp16 pair (tail sampler and dg1 GEMMs), after set_params.
void launch_split_w2(Handle* H) {
  const Layout& L = H->L;
  KScope ks(H, "split_w2");
  const int64_t total = (int64_t)L.n * H->hp18;
  split_rows_f16_kernel<<<(unsigned)((total + 255) / 256), 256, 0, H->stream>>>(
      L.n, L.h, L.h, H->hp18, H->P + L.off_w2, H->P + L.off_b2, H->W2h, H->W2l);
  VQMC_CUDA(cudaGetLastError());
  H->launches++;
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
  constexpr int BN = kTailBN;  // CTA pairs: 256 samples x 192 outputs per tile (96 outputs per CTA's B half)
  const int K = L.h + 1;   // [G1 | 1] . [W2 | b2]
  const CUtensorMap ah = tmap_kmajor(H->G1h, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_kmajor(H->G1l, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_kmajor(H->W2h + (size_t)colbase * H->hp18, K, ncols, H->hp18, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_kmajor(H->W2l + (size_t)colbase * H->hp18, K, ncols, H->hp18, BN / 2, kElemF16);
  H->tail_tiles = TailSampleEpiT<false>::kParts * ((ncols + BN - 1) / BN);  // one partial per epilogue set
  if (uni == nullptr && !want_lp) {  // training step: Philox draws, no log-probabilities
    TailSampleEpiT<true> e{B, L.n, H->np8, L.W, colbase, L.Hd, nullptr, rng, H->X, H->Dh, H->Dl, nullptr,
                           H->d_flag, 0, {}, 0.0, 0, 0, 0, 0, 0};
    launch_umma2<BN, false, false, TailSampleEpiT<true>, false, kElemF16, kTailSets, kTailCh>(
        H, "z2_tail_umma", ah, al, bh, bl, B, ncols, K, 1, e, H->stream);
  } else {
    TailSampleEpiT<false> e{B,   L.n, H->np8, L.W, colbase, L.Hd, uni, rng, H->X, H->Dh, H->Dl,
                            want_lp ? H->lp_part : nullptr, H->d_flag, 0, {}, 0.0, 0, 0, 0, 0, 0};
    launch_umma2<BN, false, false, TailSampleEpiT<false>, false, kElemF16, kTailSets, kTailCh>(
        H, "z2_tail_umma", ah, al, bh, bl, B, ncols, K, 1, e, H->stream);
  }
}

template <int BN>
static void launch_dg1_bn(Handle* H, int B) {
  const Layout& L = H->L;
  const int mt = (B + 2 * kUmmaBM - 1) / (2 * kUmmaBM), nt = (L.h + BN - 1) / BN;
  const int nkb = (L.n + Umma2Cfg<BN>::kBK - 1) / Umma2Cfg<BN>::kBK;
  // split count from the SMs the concurrent backward gives dg1 (whole GPU minus gW2's partition),
  // one pair tile per SM pair in one round; a function of the configuration only, so the serial
  // and concurrent schedules sum the same partials (results independent of the schedule)
  const int avail = gemm_sms(nullptr) - H->gemm_sm_reserve;
  const int dg1_sms = H->concurrent_bw ? avail - std::min(H->gw2_sms, avail - 16) : avail;
  int splits = std::max(1, std::min(nkb, (dg1_sms / 2) / (mt * nt)));
  splits = std::min(splits, H->max_splits);
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  H->splits = splits;
  const CUtensorMap ah = tmap_kmajor(H->Dh, L.n, B, H->np8, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_kmajor(H->Dl, L.n, B, H->np8, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_mnmajor(H->W2h, L.h, L.n, H->hp18, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_mnmajor(H->W2l, L.h, L.n, H->hp18, BN / 2, kElemF16);
  PartialEpi e{H->Epart, B, L.h, 0, {}};
  launch_umma2<BN, false, true, PartialEpi, false, kElemF16>(H, "bw_dg1_umma", ah, al, bh, bl, B, L.h, L.n, splits,
                                                             e, H->stream);
}

// dg1 on CTA pairs: 256 samples x BN hidden units per tile, split-K over the outputs (the MN-major B
// halves must be whole 64-element atoms: BN in {128, 256}).  Measured (B = 1024, scripts/gemm_rate
// hook): h = 424, K = 10^4: BN 256 30.7 us vs 128 33.7-42.2; h = 363, K = 5000: 128 26.8 vs 256
// 39.3; h = 239, K = 1000: 128 18.6 vs 256 26.8-30.7.
void launch_dg1_umma(Handle* H, int B) {
  if (H->L.h > 384) launch_dg1_bn<256>(H, B);
  else launch_dg1_bn<128>(H, B);
}

void launch_gw2_umma(Handle* H, int B, bool wg1_done, cudaStream_t stream) {
  const Layout& L = H->L;
  if (!stream) stream = H->stream;
  if (!wg1_done) {  // (the training step fuses this split into the statistics kernel)
    const int64_t total = (int64_t)B * H->hp18;
    KScope ks(H, "wg1_split");
    wg1_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(B, L.h, H->hp18, H->G1, H->w, H->wG1h,
                                                                       H->wG1l);
    VQMC_CUDA(cudaGetLastError());
    H->launches++;
  }
  // gW2^T = [w' G1 | w']^T D on CTA pairs: 256 hidden units x 256 outputs per tile (M = h + 1
  // rows: the bias row h gives gb2), K = batch
  constexpr int BN = 128;  // 2 x 79 pair tiles at N = 10k: 2.1 waves of 74 pairs (BN 256: 80 tiles, 2 full waves)
  const CUtensorMap ah = tmap_mnmajor(H->wG1h, L.h + 1, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_mnmajor(H->wG1l, L.h + 1, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_mnmajor(H->Dh, L.n, B, H->np8, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_mnmajor(H->Dl, L.n, B, H->np8, BN / 2, kElemF16);
  Gw2TEpi e{L.n, L.h, 0, {}, H->d_deg, H->d_wscale, H->G + L.off_w2, H->G + L.off_b2, 1.f, 0};
  launch_umma2<BN, true, true, Gw2TEpi, false, kElemF16>(H, "bw_gw2_umma", ah, al, bh, bl, L.h + 1, L.n, B, 1, e,
                                                         stream);
}

// S p (W2 | b2 half): [G1 | 1] . [P2 | p2]^T on CTA pairs with the D-dot epilogue; returns the
// number of partials per row (SpDotEpi::kParts x column tiles).
int launch_sp_umma(Handle* H, int B) {
  const Layout& L = H->L;
  constexpr int BN = kTailBN;
  const int K = L.h + 1;
  const CUtensorMap ah = tmap_kmajor(H->G1h, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_kmajor(H->G1l, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_kmajor(H->SRh, K, L.n, H->hp18, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_kmajor(H->SRl, K, L.n, H->hp18, BN / 2, kElemF16);
  SpDotEpi e{B, L.n, H->np8, H->Dh, H->Dl, H->sp_part, 0, {}, 0.0};
  launch_umma2<BN, false, false, SpDotEpi, false, kElemF16>(H, "sr_sp_umma", ah, al, bh, bl, B, L.n, K, 1, e,
                                                           H->stream);
  return SpDotEpi::kParts * ((L.n + BN - 1) / BN);
}

// Forward of the configurations in H->X over every output (after z1_given_kernel wrote [G1 | 1]):
// log-prob partials into lp_part (H->tail_tiles of them per row), D pairs, optional p / log terms.
void launch_given_umma(Handle* H, int B, double* cond, float* lterm, float* fterm) {
  const Layout& L = H->L;
  constexpr int BN = kTailBN;
  const int K = L.h + 1;
  const CUtensorMap ah = tmap_kmajor(H->G1h, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_kmajor(H->G1l, K, B, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_kmajor(H->W2h, K, L.n, H->hp18, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_kmajor(H->W2l, K, L.n, H->hp18, BN / 2, kElemF16);
  GivenEpiT<false> e{B,     L.n,  H->np8, L.W,     H->X,  H->Dh,   H->Dl,   H->lp_part, cond, lterm,
                     fterm, H->d_flag, 0,   0,       nullptr, 0,     {},      0.0,        0,    0};
  H->tail_tiles = GivenEpiT<false>::kParts * ((L.n + BN - 1) / BN);
  launch_umma2<BN, false, false, GivenEpiT<false>, false, kElemF16>(H, "z2_given_umma", ah, al, bh, bl, B, L.n, K,
                                                                    1, e, H->stream);
}

// Flipped-neighbour forward (TIM local energy): `rows` = Bc samples x sites rows of [G1' | 1] in
// Nh / Nl; per row the fp64 partials of sum_{i >= site} log p_i(x'_i) into part
// [kParts * tiles][rows]; returns the partial count per row.
int launch_nbr_umma(Handle* H, int rows, int Bc, int b0, const int32_t* sites, const __half* Nh, const __half* Nl,
                    double* part) {
  const Layout& L = H->L;
  constexpr int BN = kTailBN;
  const int K = L.h + 1;
  const CUtensorMap ah = tmap_kmajor(Nh, K, rows, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap al = tmap_kmajor(Nl, K, rows, H->hp18, kUmmaBM, kElemF16);
  const CUtensorMap bh = tmap_kmajor(H->W2h, K, L.n, H->hp18, BN / 2, kElemF16);
  const CUtensorMap bl = tmap_kmajor(H->W2l, K, L.n, H->hp18, BN / 2, kElemF16);
  GivenEpiT<true> e{rows, L.n, H->np8, L.W, H->X, nullptr, nullptr, part, nullptr, nullptr,
                    nullptr, H->d_flag, Bc, b0, sites, 0, {}, 0.0, 0, 0};
  launch_umma2<BN, false, false, GivenEpiT<true>, false, kElemF16>(H, "tim_nbr_umma", ah, al, bh, bl, rows, L.n, K, 1,
                                                                   e, H->stream);
  return GivenEpiT<true>::kParts * ((L.n + BN - 1) / BN);
}

// gW1T[j][k] = sum_b X[b][j] dz1[b][k] (j < Hd) and gb1[k] (the ones column j = Hd):
// split-K partials into gw1_part, reduced and masked by gw1_finalize_kernel.  The spins
// are exact in bf16, so A is single (two MMA passes).
void launch_gw1_umma(Handle* H, int B, int& splits_out) {
  const Layout& L = H->L;
  constexpr int BN = 128;
  const int mt = (L.Hd + 1 + kUmmaBM - 1) / kUmmaBM, nt = (L.h + BN - 1) / BN;
  const int nkb = (B + UmmaElem<true>::kBK - 1) / UmmaElem<true>::kBK;
  int splits = std::max(1, std::min(std::min(nkb, kGw1MaxSplits), gemm_sms(nullptr) / (mt * nt)));
  if (H->gw1_splits > 0) splits = std::min(splits, H->gw1_splits);
  const int per = (nkb + splits - 1) / splits;
  splits = (nkb + per - 1) / per;
  splits_out = splits;
  const CUtensorMap a = tmap_mnmajor(H->Xfb, L.Hd + 1, B, H->hd18, kUmmaBM, kElemBF16);
  const CUtensorMap bh = tmap_mnmajor(H->dz1bh, L.h, B, H->hp8, BN, kElemBF16);
  const CUtensorMap bl = tmap_mnmajor(H->dz1bl, L.h, B, H->hp8, BN, kElemBF16);
  if (splits == 1) {  // whole K per tile: the epilogue writes gW1T / gb1 directly (no finalize pass)
    Gw1Epi e{L.h, L.Hd, 0, {}, H->d_deg, H->d_wscale, H->G + L.off_w1t, H->G + L.off_b1, 1.f};
    launch_umma<BN, true, true, Gw1Epi, true, kElemBF16>(H, "bw_gw1_umma", a, a, bh, bl, L.Hd + 1, L.h, B, 1, e,
                                                         H->stream);
    return;
  }
  PartialEpi e{H->gw1_part, L.Hd + 1, L.h, 0, {}};
  launch_umma<BN, true, true, PartialEpi, true, kElemBF16>(H, "bw_gw1_umma", a, a, bh, bl, L.Hd + 1, L.h, B, splits,
                                                           e, H->stream);
}

}  // namespace vqmc_b200

// ===========================================================================
// Test hook: C = A B^T through the 3-pass tcgen05 kernel on host fp32 arrays.
//   a_mn = 0: A is [M][K] (K-major); 1: A is [K][M] (MN-major).  Same for B with N.
//   ek: operand pairs 0 = tf32, 1 = bf16, 2 = fp16.
// ===========================================================================
using namespace vqmc_b200;

static float g_test_ms = 0.f;  // average kernel time of the last test-hook GEMM (VQMC_TEST_REPS launches)
extern "C" float vqmc_test_last_ms(void) { return g_test_ms; }
static int test_reps() {
  const char* e = std::getenv("VQMC_TEST_REPS");
  return e ? std::max(1, atoi(e)) : 1;
}

extern "C" int vqmc_test_umma_gemm(int M, int N, int K, int a_mn, int b_mn, int bn, int splits, int ek,
                                   const float* A, const float* Bm, float* C) {
  void *dA = nullptr, *dB = nullptr, *dAh = nullptr, *dAl = nullptr, *dBh = nullptr, *dBl = nullptr;
  float* dC = nullptr;
  auto release = [&]() {
    for (void* p : {dA, dB, dAh, dAl, dBh, dBl, (void*)dC})
      if (p) cudaFree(p);
  };
  try {
    if (ek < 0 || ek > 2) throw InvalidArgument("element kind must be 0 (tf32), 1 (bf16) or 2 (fp16)");
    const int q = ek ? 8 : 4, es = ek ? 2 : 4;
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
    if (ek == kElemBF16) {
      split_rows_bf16_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, (__nv_bfloat16*)dAh,
                                          (__nv_bfloat16*)dAl);
      split_rows_bf16_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, (__nv_bfloat16*)dBh,
                                          (__nv_bfloat16*)dBl);
    } else if (ek == kElemF16) {
      split_rows_f16_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, nullptr, (__half*)dAh,
                                         (__half*)dAl);
      split_rows_f16_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, nullptr, (__half*)dBh,
                                         (__half*)dBl);
    } else {
      split_rows_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, (float*)dAh, (float*)dAl);
      split_rows_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, (float*)dBh, (float*)dBl);
    }
    VQMC_CUDA(cudaGetLastError());
    const int bnv = bn == 256 ? 256 : 128;
    CUtensorMap ah, al, bh, bl;
    if (a_mn) { ah = tmap_mnmajor(dAh, M, K, lda, kUmmaBM, ek); al = tmap_mnmajor(dAl, M, K, lda, kUmmaBM, ek); }
    else { ah = tmap_kmajor(dAh, K, M, lda, kUmmaBM, ek); al = tmap_kmajor(dAl, K, M, lda, kUmmaBM, ek); }
    if (b_mn) { bh = tmap_mnmajor(dBh, N, K, ldb, bnv, ek); bl = tmap_mnmajor(dBl, N, K, ldb, bnv, ek); }
    else { bh = tmap_kmajor(dBh, K, N, ldb, bnv, ek); bl = tmap_kmajor(dBl, K, N, ldb, bnv, ek); }
    PartialEpi e{dC, M, N, 0, {}};
#define GO(BNV, AM, BM_, EKV)                                                                          \
  launch_umma<BNV, AM, BM_, PartialEpi, false, EKV>(nullptr, "test", ah, al, bh, bl, M, N, K, splits, e, \
                                                   (cudaStream_t)0)
#define GO4(BNV, EKV)                                \
  if (!a_mn && !b_mn) GO(BNV, false, false, EKV);     \
  else if (!a_mn && b_mn) GO(BNV, false, true, EKV);  \
  else if (a_mn && !b_mn) GO(BNV, true, false, EKV);  \
  else GO(BNV, true, true, EKV)
#define GO_EK(BNV)                                       \
  if (ek == kElemBF16) { GO4(BNV, kElemBF16); }          \
  else if (ek == kElemF16) { GO4(BNV, kElemF16); }       \
  else { GO4(BNV, kElemTF32); }
    if (bnv == 128) {
      GO_EK(128)
    } else {
      GO_EK(256)
    }
#undef GO_EK
#undef GO2K
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

// Test hook: the CTA-pair kernel (16-bit pairs only), same conventions as vqmc_test_umma_gemm;
// bn in {128, 192, 256}.
extern "C" int vqmc_test_umma2_gemm(int M, int N, int K, int a_mn, int b_mn, int bn, int splits, int ek,
                                    const float* A, const float* Bm, float* C) {
  void *dA = nullptr, *dB = nullptr, *dAh = nullptr, *dAl = nullptr, *dBh = nullptr, *dBl = nullptr;
  float* dC = nullptr;
  auto release = [&]() {
    for (void* p : {dA, dB, dAh, dAl, dBh, dBl, (void*)dC})
      if (p) cudaFree(p);
  };
  try {
    if (ek != kElemBF16 && ek != kElemF16) throw InvalidArgument("pair kernel: element kind must be 1 or 2");
    const int q = 8;
    const int lda = a_mn ? ((M + q - 1) / q * q) : ((K + q - 1) / q * q);
    const int arows = a_mn ? K : M, acols = a_mn ? M : K;
    const int ldb = b_mn ? ((N + q - 1) / q * q) : ((K + q - 1) / q * q);
    const int brows = b_mn ? K : N, bcols = b_mn ? N : K;
    const size_t pad = 512;
    const size_t asz = ((size_t)arows * lda + pad) * 2, bsz = ((size_t)brows * ldb + pad) * 2;
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
    if (ek == kElemBF16) {
      split_rows_bf16_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, (__nv_bfloat16*)dAh,
                                          (__nv_bfloat16*)dAl);
      split_rows_bf16_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, (__nv_bfloat16*)dBh,
                                          (__nv_bfloat16*)dBl);
    } else {
      split_rows_f16_kernel<<<ga, 256>>>(arows, acols, acols, lda, (const float*)dA, nullptr, (__half*)dAh,
                                         (__half*)dAl);
      split_rows_f16_kernel<<<gb, 256>>>(brows, bcols, bcols, ldb, (const float*)dB, nullptr, (__half*)dBh,
                                         (__half*)dBl);
    }
    VQMC_CUDA(cudaGetLastError());
    const int half = bn / 2;
    CUtensorMap ah, al, bh, bl;
    if (a_mn) { ah = tmap_mnmajor(dAh, M, K, lda, kUmmaBM, ek); al = tmap_mnmajor(dAl, M, K, lda, kUmmaBM, ek); }
    else { ah = tmap_kmajor(dAh, K, M, lda, kUmmaBM, ek); al = tmap_kmajor(dAl, K, M, lda, kUmmaBM, ek); }
    if (b_mn) { bh = tmap_mnmajor(dBh, N, K, ldb, half, ek); bl = tmap_mnmajor(dBl, N, K, ldb, half, ek); }
    else { bh = tmap_kmajor(dBh, K, N, ldb, half, ek); bl = tmap_kmajor(dBl, K, N, ldb, half, ek); }
    PartialEpi e{dC, M, N, 0, {}};
#define GO(BNV, AM, BM_, EKV)                                                                            \
  launch_umma2<BNV, AM, BM_, PartialEpi, false, EKV>(nullptr, "test", ah, al, bh, bl, M, N, K, splits, e, \
                                                    (cudaStream_t)0)
#define GO4(BNV, EKV)                                \
  if (!a_mn && !b_mn) GO(BNV, false, false, EKV);     \
  else if (!a_mn && b_mn) GO(BNV, false, true, EKV);  \
  else if (a_mn && !b_mn) GO(BNV, true, false, EKV);  \
  else GO(BNV, true, true, EKV)
#define GO2K(BNV, EKV)                               \
  if (b_mn) throw InvalidArgument("pair kernel: bn 192 needs a K-major B"); \
  else if (!a_mn) GO(BNV, false, false, EKV);         \
  else GO(BNV, true, false, EKV)
#define GO_EK(BNV)                                 \
  if (ek == kElemBF16) { GO4(BNV, kElemBF16); }    \
  else { GO4(BNV, kElemF16); }
    const int reps = test_reps();
    cudaEvent_t e0, e1;
    VQMC_CUDA(cudaEventCreate(&e0));
    VQMC_CUDA(cudaEventCreate(&e1));
    for (int rep = 0; rep <= reps; ++rep) {  // rep 0: warm-up
      if (rep == 1) VQMC_CUDA(cudaEventRecord(e0));
      if (bn == 128) { GO_EK(128) }
      else if (bn == 192) {
        if (ek == kElemBF16) { GO2K(192, kElemBF16); } else { GO2K(192, kElemF16); }
      }
      else if (bn == 256) { GO_EK(256) }
      else throw InvalidArgument("pair kernel: bn must be 128, 192 or 256");
    }
    VQMC_CUDA(cudaEventRecord(e1));
    VQMC_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    VQMC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    g_test_ms = reps > 0 ? ms / reps : 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
#undef GO_EK
#undef GO2K
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

#ifdef VQMC_TAIL_TRACE
// Trace hook (built only with -DVQMC_TAIL_TRACE): run the tail sampler GEMM of B samples once on
// the handle and copy the per-CTA timeline (g_tail_trace) out.
extern "C" int vqmc_test_tail_trace(vqmc_gpu_t* g, int B, unsigned long long* out, int exp_mask) {
  using namespace vqmc_b200;
  Handle* H = reinterpret_cast<Handle*>(g);
  try {
    VQMC_CUDA(cudaMemcpyToSymbol(g_tail_exp, &exp_mask, sizeof(int)));
    H->ensure_batch(B);
    RngSpec rng{1, 1, 0, B, nullptr};
    void* tp = nullptr;
    VQMC_CUDA(cudaGetSymbolAddress(&tp, g_tail_trace));
    VQMC_CUDA(cudaMemset(tp, 0, sizeof(g_tail_trace)));
    launch_tail_umma(H, B, nullptr, rng, false);
    launch_tail_umma(H, B, nullptr, rng, false);
    VQMC_CUDA(cudaStreamSynchronize(H->stream));
    VQMC_CUDA(cudaMemcpyFromSymbol(out, g_tail_trace, sizeof(g_tail_trace)));
  } catch (const std::exception& ex) {
    set_error(ex.what());
    return status_of(ex);
  }
  return VQMC_OK;
}
#endif
