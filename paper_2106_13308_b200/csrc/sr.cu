// Stochastic reconfiguration (SR, natural gradient) on the GPU — SURVEY §8f row 2.
//
// Reference: score_matrix (proj/src/models.cpp:221-244), FisherEstimate (centred scores,
// F v = S^T (S v) / B; proj/include/vqmc/estimator.hpp:146-168), sr_direction /
// conjugate_gradient (proj/src/optimizer.cpp:36-92), the SGD-SR update (trainer.cpp:189-199,
// 223-225).
//
// The reference materialises S (B x d fp64: 70 GB at N = 10k).  Here S is never formed: the CG
// operator F p = S~^T S~ p / B + lambda p is applied through the MADE structure of the scores
// (row b of S = 2 grad log psi(x_b)):
//   q_b = grad log psi(x_b) . p
//       = sum_i D[b][i] ([G1_b 1] . [P2 p2]_i)          (tcgen05 pair GEMM, D-dot epilogue)
//       + sum_k dz1[b][k] (p1_k + sum_{j < deg_k} x_b[j] P1[k][j])   (per-sample SIMT pass)
//   F p   = sum_b y_b grad log psi(x_b),  y = (4 / B) (q - mean q)     (the REINFORCE backward
//                                                                      with weights y)
// so one CG iteration costs one forward-shaped GEMM and the backward GEMMs of a training step,
// all at fp32 grade (fp16 pairs); the CG vectors and scalars are fp64 like the reference, with
// fixed-order reductions (deterministic).  The solve runs the reference's CG for every d (the
// reference switches to a dense LDLT for d <= 2000; both accept a solution only when the relative
// residual is <= tol).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "device_common.cuh"
#include "internal.cuh"
#include "ptx.cuh"
#include "umma2_gemm.cuh"

namespace vqmc_b200 {

namespace {

constexpr int kVecBlocks = 148 * 4, kVecThreads = 256;

__device__ __forceinline__ double block_sum256(double s) {
  __shared__ double red[kVecThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kVecThreads / 32; ++i) t += red[i];
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kVecThreads) sr_sum_kernel(int cnt, const double* __restrict__ part,
                                                            double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum256(s);
  if (threadIdx.x == 0) *out = s;
}

// g = G * scale (the training step's summed gradient -> allreduce_mean's mean)
__global__ void sr_grad_kernel(int64_t total, const float* __restrict__ G, double scale, double* __restrict__ g) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    g[t] = (double)G[t] * scale;
}

// x = 0, r = p = g; partial sums of g.g (conjugate_gradient, optimizer.cpp:48-56)
__global__ void __launch_bounds__(kVecThreads) cg_init_kernel(int64_t total, const double* __restrict__ g,
                                                             double* __restrict__ x, double* __restrict__ r,
                                                             double* __restrict__ p, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = g[t];
    x[t] = 0.0;
    r[t] = v;
    p[t] = v;
    s += v * v;
  }
  s = block_sum256(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// p . (F p + lambda p), F p in G (fp32, the backward's output)
__global__ void __launch_bounds__(kVecThreads) cg_pap_kernel(int64_t total, const float* __restrict__ G,
                                                            const double* __restrict__ p, double lambda,
                                                            double* __restrict__ part) {
  double s = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[t];
    s += pv * ((double)G[t] + lambda * pv);
  }
  s = block_sum256(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// alpha = rs / (p . A p) on the device (scal[0] = rs, scal[1] = alpha): no host round trip
__global__ void __launch_bounds__(kVecThreads) cg_alpha_kernel(int cnt, const double* __restrict__ part,
                                                              double* __restrict__ scal) {
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum256(s);
  if (threadIdx.x == 0) scal[1] = scal[0] / s;
}

// x += alpha p; r -= alpha (F p + lambda p); partial sums of r.r
__global__ void __launch_bounds__(kVecThreads) cg_xr_kernel(int64_t total, const double* __restrict__ scal,
                                                           const float* __restrict__ G, const double* __restrict__ p,
                                                           double lambda, double* __restrict__ x,
                                                           double* __restrict__ r, double* __restrict__ part) {
  const double alpha = scal[1];
  double s = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[t], ap = (double)G[t] + lambda * pv;
    x[t] += alpha * pv;
    const double rv = r[t] - alpha * ap;
    r[t] = rv;
    s += rv * rv;
  }
  s = block_sum256(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// p = r + beta p, and max |p| over the [W2 | b2] range [lo, total) for the next operand split
__global__ void __launch_bounds__(kVecThreads) cg_p_kernel(int64_t total, int64_t lo, double beta,
                                                          const double* __restrict__ r, double* __restrict__ p,
                                                          unsigned* __restrict__ pmax) {
  float m = 0.f;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = r[t] + beta * p[t];
    p[t] = v;
    if (t >= lo) m = fmaxf(m, (float)fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(pmax, __float_as_uint(m));
}

// params - lr * delta (sgd_step, optimizer.hpp:57-59) on the fp32 master copy
__global__ void sr_apply_kernel(int64_t total, double lr, const double* __restrict__ delta, float* __restrict__ P) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    P[t] = (float)((double)P[t] - lr * delta[t]);
}

// Device-resident CG loop (one captured iteration under a conditional WHILE node): the convergence
// test of conjugate_gradient (optimizer.cpp:58-60) on the device.  st = scal + 4: [0] rs0 = g.g,
// [1] final r.r, [2] iterations, [3] beta.  Stops the loop (and leaves p stale) on convergence or at
// the iteration budget, else prepares beta, rs and the p-range maximum for the p update.
__global__ void __launch_bounds__(kVecThreads) cg_check_kernel(cudaGraphConditionalHandle cond, int cnt,
                                                              const double* __restrict__ part,
                                                              double* __restrict__ scal, double tol, int max_it,
                                                              unsigned* __restrict__ pmax) {
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum256(s);
  if (threadIdx.x == 0) {
    double* st = scal + 4;
    const int it = (int)st[2] + 1;
    st[2] = (double)it;
    if (sqrt(s) <= tol * sqrt(st[0]) || it >= max_it) {  // (the host loop's test, same roundings)
      st[1] = s;
      cudaGraphSetConditional(cond, 0);
    } else {
      st[3] = s / scal[0];
      scal[0] = s;
      *pmax = 0u;
    }
  }
}
__global__ void cg_state_init_kernel(double* __restrict__ scal) {
  scal[4] = scal[0];
  scal[5] = scal[0];
  scal[6] = 0.0;
}
// p = r + beta p with beta from the device state
__global__ void __launch_bounds__(kVecThreads) cg_p_dev_kernel(int64_t total, int64_t lo,
                                                              const double* __restrict__ scal,
                                                              const double* __restrict__ r, double* __restrict__ p,
                                                              unsigned* __restrict__ pmax) {
  const double beta = scal[7];
  float m = 0.f;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = r[t] + beta * p[t];
    p[t] = v;
    if (t >= lo) m = fmaxf(m, (float)fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(pmax, __float_as_uint(m));
}

// max |p| over the [W2 | b2] range (float bits; atomicMax of non-negative floats is order-free)
__global__ void sr_pmax_kernel(int64_t lo, int64_t hi, const double* __restrict__ p, unsigned* __restrict__ pmax) {
  float m = 0.f;
  for (int64_t t = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, (float)fabs(p[t]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(pmax, __float_as_uint(m));
}

__device__ __forceinline__ int pmax_exp(const unsigned* pmax) {
  const float m = __uint_as_float(*pmax);
  int e = 0;
  if (m > 0.f) frexpf(m, &e);  // m < 2^e
  return e;
}

// [P2m | p2] * 2^-e as an fp16 pair, the B operand of the S p GEMM (rows i, stride hp18)
__global__ void sr_split_kernel(int n, int h, int ld, const double* __restrict__ p, int64_t off_w2, int64_t off_b2,
                                const int32_t* __restrict__ deg, const unsigned* __restrict__ pmax,
                                __half* __restrict__ hi, __half* __restrict__ lo) {
  // one CTA per row i (columns strided over the threads); x 2^-e as one exact fp64 multiply
  const int i = blockIdx.x;
  if (i >= n) return;
  const double sc = ldexp(1.0, -pmax_exp(pmax));
  for (int c = threadIdx.x; c < ld; c += blockDim.x) {
    double x = 0.0;
    if (c < h) x = deg[c] < i + 1 ? p[off_w2 + (int64_t)i * h + c] : 0.0;  // M2(i, c)
    else if (c == h) x = p[off_b2 + i];
    const size_t t = (size_t)i * ld + c;
    ptx::split_f16((float)(x * sc), hi[t], lo[t]);
  }
}

// dz1 = (D W2m) relu'(z1) of the batch (unweighted; fixed during a solve), from dg1's split-K partials
__global__ void sr_dz1_kernel(int B, int h, int splits, const float* __restrict__ Epart, const float* __restrict__ G1,
                              float* __restrict__ dz1) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * h) return;
  float e = 0.f;
  for (int z = 0; z < splits; ++z) e += Epart[(size_t)z * B * h + t];
  dz1[t] = G1[t] > 0.f ? e : 0.f;  // relu'(z1) = [g1 > 0]
}

// The W1 block of the direction as masked fp32 rows P1f[j][k] = P1[k][j] M1(k, j) (row stride ld)
__global__ void sr_p1f_kernel(int Hd, int h, int ld, const double* __restrict__ p1, const int32_t* __restrict__ deg,
                              float* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)Hd * ld) return;
  const int j = (int)(t / ld), k = (int)(t % ld);
  out[t] = (k < h && j + 1 <= deg[k]) ? (float)p1[(size_t)j * h + k] : 0.f;
}

// W1 half of q without the bias term: sum_k dz1_b[k] sum_{j: x_b[j] = 1} P1f[j][k], one CTA per
// sample, 16-byte row loads.  part[b] (one partial per sample).
constexpr int kQ1Threads = 128;
// Warp w takes the spin words m = w, w + 4, ...: the CTA's four warps walk four disjoint sets of
// rows at once (a quarter of the serial L2 round trips of one row set per CTA); lane l holds the
// float4 columns l + 32 u (U of them), R set-bit rows in flight per lane.
template <int U, int R>
__global__ void __launch_bounds__(kQ1Threads) sr_q1_kernel(int B, int h, int Hd, int W, int ld,
                                                           const uint32_t* __restrict__ X, const float* __restrict__ dz1,
                                                           const float* __restrict__ P1f, double* __restrict__ part) {
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int nq = ld / 4;  // float4 columns per row
  int jl[R];
  int cnt = 0;
  auto flush = [&](int n) {
    float4 v[R][U];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = lane + 32 * u;
        v[r][u] = (r < n && c < nq) ? reinterpret_cast<const float4*>(P1f + (size_t)jl[r] * ld)[c]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x += v[r][u].x;
        acc[u].y += v[r][u].y;
        acc[u].z += v[r][u].z;
        acc[u].w += v[r][u].w;
      }
  };
  for (int w = warp; w * 32 < Hd; w += kQ1Threads / 32) {
    uint32_t bits = X[(size_t)b * W + w];
    if (Hd - 32 * w < 32) bits &= (1u << (Hd - 32 * w)) - 1u;
    while (bits) {
      jl[cnt++] = 32 * w + __ffs(bits) - 1;
      bits &= bits - 1u;
      if (cnt == R) {
        flush(R);
        cnt = 0;
      }
    }
  }
  if (cnt) flush(cnt);
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int c = lane + 32 * u;
    if (c < nq) {
      const float* d = dz1 + (size_t)b * h + 4 * c;  // (rows of h floats: not 16-byte aligned in general)
      const float a4[4] = {acc[u].x, acc[u].y, acc[u].z, acc[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (4 * c + i < h) s += (double)d[i] * a4[i];
    }
  }
  __shared__ double red[kQ1Threads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kQ1Threads / 32; ++i) t += red[i];
    part[b] = t;
  }
}

// q_b = grad log psi(x_b) . p = (W1 half: q1 partials + dz1_b . p_b1) + (W2 half: GEMM partials
// x 2^e).  One warp per sample.
__global__ void sr_q_kernel(int B, int h, const float* __restrict__ dz1, const double* __restrict__ pb1,
                            const double* __restrict__ q1_part, int q1_tiles, const double* __restrict__ sp_part,
                            int nparts, const unsigned* __restrict__ pmax, double* __restrict__ q) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  double s = 0.0;
  for (int k = lane; k < h; k += 32) s += (double)dz1[(size_t)b * h + k] * pb1[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  double t2 = 0.0;  // GEMM partials: lane-strided, then the same fixed shuffle tree
  for (int t = lane; t < nparts; t += 32) t2 += sp_part[(size_t)t * B + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t2 += __shfl_xor_sync(kFull, t2, o);
  if (lane == 0) {
    for (int t = 0; t < q1_tiles; ++t) s += q1_part[(size_t)t * B + b];
    q[b] = s + ldexp(t2, pmax_exp(pmax));
  }
}

// REINFORCE-style weights of F p: y = coef (q - mean q) (centred) or coef q, normalised to
// w' = y / wscale with wscale = 2^e >= max |y| (the backward's fp16 operand range).  One block.
// sum of q over this rank's samples (fixed order) -> *out; summed over ranks before the weights
__global__ void __launch_bounds__(1024) sr_qsum_kernel(int B, const double* __restrict__ q, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s += q[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    *out = t;
  }
}

// (qsum: the sum of q over every rank's samples; N: their number)
__global__ void __launch_bounds__(1024) sr_weights_kernel(int B, const double* __restrict__ q, double coef,
                                                          int centered, const double* __restrict__ qsum, double N,
                                                          float* __restrict__ w, float* __restrict__ wscale) {
  __shared__ float s_max[32];
  const double mean = centered ? *qsum / N : 0.0;
  float m = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) m = fmaxf(m, (float)fabs(coef * (q[b] - mean)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mm = fmaxf(mm, s_max[i]);
    s_max[0] = mm;
  }
  __syncthreads();
  int e = 0;
  if (s_max[0] > 0.f) frexpf(s_max[0], &e);
  for (int b = threadIdx.x; b < B; b += blockDim.x) w[b] = (float)ldexp(coef * (q[b] - mean), -e);
  if (threadIdx.x == 0) *wscale = ldexpf(1.f, e);
}


// ---- small models (reference d <= 2000, where sr_direction solves the dense system exactly):
// the score rows are materialised in fp64 (live layout) and F is applied exactly, so CG is a
// direct solve (it terminates in at most rank(F) + 1 <= B iterations) ----

// S[b][t] = 2 grad log psi(x_b) at live entry t (models.cpp:221-244)
__global__ void sr_dense_scores_kernel(int B, int n, int h, int Hd, int W, int np, const uint32_t* __restrict__ X,
                                       const float* __restrict__ G1, const __half* __restrict__ Dh,
                                       const __half* __restrict__ Dl, const float* __restrict__ Epart, int splits,
                                       const int32_t* __restrict__ deg, int64_t off_b1, int64_t off_w2,
                                       int64_t off_b2, int64_t total, double* __restrict__ S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (t >= total) return;
  auto dz1 = [&](int k) {
    float e = 0.f;
    for (int z = 0; z < splits; ++z) e += Epart[((size_t)z * B + b) * h + k];
    return G1[(size_t)b * h + k] > 0.f ? (double)e : 0.0;
  };
  auto dval = [&](int i) {
    return (double)__half2float(Dh[(size_t)b * np + i]) + (double)__half2float(Dl[(size_t)b * np + i]);
  };
  double v;
  if (t < off_b1) {  // W1T[j][k]
    const int j = (int)(t / h), k = (int)(t % h);
    const int xj = (X[(size_t)b * W + (j >> 5)] >> (j & 31)) & 1;
    v = (j + 1 <= deg[k] && xj) ? dz1(k) : 0.0;
  } else if (t < off_w2) {
    v = dz1((int)(t - off_b1));
  } else if (t < off_b2) {
    const int64_t u = t - off_w2;
    const int i = (int)(u / h), k = (int)(u % h);
    v = deg[k] < i + 1 ? dval(i) * (double)G1[(size_t)b * h + k] : 0.0;
  } else {
    v = dval((int)(t - off_b2));
  }
  S[(size_t)b * total + t] = 2.0 * v;
}

// column means subtracted (FisherEstimate's centring), sequential over samples per column
__global__ void sr_dense_center_kernel(int B, int64_t total, double* __restrict__ S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += S[(size_t)b * total + t];
  const double mean = s / (double)B;
  for (int b = 0; b < B; ++b) S[(size_t)b * total + t] -= mean;
}

// u = S p (one block per row)
__global__ void __launch_bounds__(kVecThreads) sr_dense_sp_kernel(int64_t total, const double* __restrict__ S,
                                                                  const double* __restrict__ p, double* __restrict__ u) {
  const int b = blockIdx.x;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) s += S[(size_t)b * total + t] * p[t];
  s = block_sum256(s);
  if (threadIdx.x == 0) u[b] = s;
}

// out = scale S^T u (one thread per column, sequential over samples)
__global__ void sr_dense_stu_kernel(int B, int64_t total, const double* __restrict__ S, const double* __restrict__ u,
                                    double scale, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += S[(size_t)b * total + t] * u[b];
  out[t] = s * scale;
}

// Lower triangle of C = M M^T + shift I, M[i][k] = A[i * si + k * sk] (m rows, K columns):
// the B x B Gram S S^T (si = total, sk = 1) or the d x d S^T S (si = 1, sk = total).
__global__ void sr_gram_kernel(int m, int64_t K, int64_t si, int64_t sk, const double* __restrict__ A, double scale,
                               double shift, double* __restrict__ C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * m) return;
  const int i = (int)(e / m), j = (int)(e % m);
  if (j > i) return;
  double s = 0.0;
  for (int64_t k = 0; k < K; ++k) s += A[i * si + k * sk] * A[j * si + k * sk];
  C[(size_t)i * m + j] = s * scale + (i == j ? shift : 0.0);
}

// Column j of the in-place lower Cholesky factor (left-looking): one warp per row i >= j; every
// warp recomputes the pivot.  flag: set if the matrix is not positive definite.
__global__ void __launch_bounds__(256) sr_chol_col_kernel(int m, int j, double* __restrict__ C,
                                                          unsigned* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int i = j + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= m) return;
  const double* Lj = C + (size_t)j * m;
  const double* Li = C + (size_t)i * m;
  double dj = 0.0, di = 0.0;
  for (int k = lane; k < j; k += 32) {
    dj += Lj[k] * Lj[k];
    di += Li[k] * Lj[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dj += __shfl_xor_sync(kFull, dj, o);
    di += __shfl_xor_sync(kFull, di, o);
  }
  const double piv = Lj[j] - dj;
  if (lane == 0) {
    if (!(piv > 0.0)) {
      *flag = 1u;
      return;
    }
    const double l = sqrt(piv);
    if (i == j) C[(size_t)m * m + j] = l;  // the pivots live after the matrix (C[j][j] stays A[j][j])
    else C[(size_t)i * m + j] = (Li[j] - di) / l;
  }
}

// x = C^{-1} b with C = L L^T (strict lower part in C, pivots at C + m m; in place in x)
__global__ void __launch_bounds__(1024) sr_chol_solve_kernel(int m, const double* __restrict__ L,
                                                             double* __restrict__ x) {
  __shared__ double red[32];
  for (int pass = 0; pass < 2; ++pass) {
    for (int r = 0; r < m; ++r) {
      const int i = pass == 0 ? r : m - 1 - r;
      double s = 0.0;
      if (pass == 0)
        for (int k = threadIdx.x; k < i; k += blockDim.x) s += L[(size_t)i * m + k] * x[k];
      else
        for (int k = i + 1 + threadIdx.x; k < m; k += blockDim.x) s += L[(size_t)k * m + i] * x[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        x[i] = (x[i] - t) / L[(size_t)m * m + i];
      }
      __syncthreads();
    }
  }
}

// partial sums of ||F x + lambda x - g||^2
__global__ void __launch_bounds__(kVecThreads) sr_resid_kernel(int64_t total, const double* __restrict__ Fx,
                                                              const double* __restrict__ x, double lambda,
                                                              const double* __restrict__ g, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const double r = Fx[t] + lambda * x[t] - g[t];
    s += r * r;
  }
  s = block_sum256(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// delta = (g - S^T z) / lambda (Woodbury back-substitution); z already holds S^T z in out
__global__ void sr_woodbury_kernel(int64_t total, const double* __restrict__ g, double inv_lambda,
                                   double* __restrict__ x) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    x[t] = (g[t] - x[t]) * inv_lambda;
}

#define SR_CHECK() VQMC_CUDA(cudaGetLastError())

double sum_parts(Handle* H, const double* part, int cnt) {
  sr_sum_kernel<<<1, kVecThreads, 0, H->stream>>>(cnt, part, H->d_sr_scal);
  SR_CHECK();
  VQMC_CUDA(cudaMemcpyAsync(H->h_sr_scal, H->d_sr_scal, sizeof(double), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  H->launches++;
  return *H->h_sr_scal;
}

// G = F p (without lambda), p = H->cg_p with max |p| over [W2 | b2] in H->d_pmax.  Needs the
// batch's G1 / D / X and dg1 partials.
void apply_fisher(Handle* H, int B, bool centered) {
  const Layout& L = H->L;
  sr_split_kernel<<<(unsigned)L.n, 128, 0, H->stream>>>(L.n, L.h, H->hp18, H->cg_p, L.off_w2,
                                                                         L.off_b2, H->d_deg, H->d_pmax, H->SRh,
                                                                         H->SRl);
  SR_CHECK();
  const int nparts = launch_sp_umma(H, B);
  {
    const int ld = 4 * ((L.h + 3) / 4);
    const int64_t tp = (int64_t)L.Hd * ld;
    sr_p1f_kernel<<<(unsigned)((tp + 255) / 256), 256, 0, H->stream>>>(L.Hd, L.h, ld, H->cg_p + L.off_w1t, H->d_deg,
                                                                       H->sr_p1f);
    if (ld / 4 <= 128)
      sr_q1_kernel<4, 4><<<B, kQ1Threads, 0, H->stream>>>(B, L.h, L.Hd, L.W, ld, H->X, H->sr_dz1, H->sr_p1f, H->sr_q1);
    else
      sr_q1_kernel<8, 2><<<B, kQ1Threads, 0, H->stream>>>(B, L.h, L.Hd, L.W, ld, H->X, H->sr_dz1, H->sr_p1f, H->sr_q1);
    sr_q_kernel<<<(B + 7) / 8, 256, 0, H->stream>>>(B, L.h, H->sr_dz1, H->cg_p + L.off_b1, H->sr_q1, 1, H->sp_part,
                                                    nparts, H->d_pmax, H->sr_q);
  }
  SR_CHECK();
  // F p = S~^T S~ p / N with S = 2 grad log psi over all N = B x ranks samples (the reference's
  // shared_scores): weights 4 (q - mean q) / N on grad log psi, then the gradient all-reduce
  const double N = (double)B * H->nranks;
  sr_qsum_kernel<<<1, 1024, 0, H->stream>>>(B, H->sr_q, H->d_sr_scal + 2);
  SR_CHECK();
  comm_allreduce_sum(H, H->d_sr_scal + 2, 1, true);
  sr_weights_kernel<<<1, 1024, 0, H->stream>>>(B, H->sr_q, 4.0 / N, centered ? 1 : 0, H->d_sr_scal + 2, N, H->w,
                                               H->d_wscale);
  SR_CHECK();
  H->launches += 6;
  launch_gw2_umma(H, B, /*wg1_done=*/false);  // w' [G1 | 1] pair, then gW2 / gb2
  launch_backward_after_dg1(H, B);            // dz1 (the batch's dg1 partials), gW1 / gb1
  comm_allreduce_sum(H, H->G, (size_t)H->L.total, false);
}

void apply_fisher_dense(Handle* H, int B) {
  const int64_t total = H->L.total;
  sr_dense_sp_kernel<<<B, kVecThreads, 0, H->stream>>>(total, H->sr_S, H->cg_p, H->sr_q);
  SR_CHECK();
  sr_dense_stu_kernel<<<(unsigned)((total + 127) / 128), 128, 0, H->stream>>>(B, total, H->sr_S, H->sr_q,
                                                                              1.0 / (double)B, H->cg_ap);
  SR_CHECK();
  H->launches += 2;
}

}  // namespace

void sr_build_scores(Handle* H, int B, bool centered) {
  const Layout& L = H->L;
  const int64_t total = L.total;
  if ((size_t)B * total > H->sr_S_cap) {
    if (H->sr_S) cudaFree(H->sr_S);
    VQMC_CUDA(cudaMalloc((void**)&H->sr_S, (size_t)B * total * sizeof(double)));
    H->sr_S_cap = (size_t)B * total;
  }
  sr_dense_scores_kernel<<<dim3((unsigned)((total + 127) / 128), B), 128, 0, H->stream>>>(
      B, L.n, L.h, L.Hd, L.W, H->np8, H->X, H->G1, H->Dh, H->Dl, H->Epart, H->splits, H->d_deg, L.off_b1, L.off_w2,
      L.off_b2, total, H->sr_S);
  SR_CHECK();
  H->launches++;
  if (centered) {
    sr_dense_center_kernel<<<(unsigned)((total + 127) / 128), 128, 0, H->stream>>>(B, total, H->sr_S);
    SR_CHECK();
    H->launches++;
  }
}


void ensure_sr(Handle* H, int B) {
  const Layout& L = H->L;
  auto alloc = [](auto** p, size_t count) {
    VQMC_CUDA(cudaMalloc((void**)p, count * sizeof(**p)));
  };
  if (!H->cg_x) {
    alloc(&H->cg_x, (size_t)L.total);
    alloc(&H->cg_r, (size_t)L.total);
    alloc(&H->cg_p, (size_t)L.total);
    alloc(&H->cg_g, (size_t)L.total);
    alloc(&H->cg_ap, (size_t)L.total);
    alloc(&H->SRh, (size_t)L.n * H->hp18);
    alloc(&H->SRl, (size_t)L.n * H->hp18);
    alloc(&H->cg_part, (size_t)kVecBlocks);
    alloc(&H->sr_p1f, (size_t)L.Hd * 4 * ((L.h + 3) / 4));
    alloc(&H->d_sr_scal, (size_t)8);  // [0] rs [1] alpha [2] q sum; device CG loop: [4] rs0 [5] rs [6] it [7] beta
    alloc(&H->d_pmax, (size_t)1);
    VQMC_CUDA(cudaMallocHost((void**)&H->h_sr_scal, 8 * sizeof(double)));
  }
  if (B > H->sr_cap_B) {
    if (H->sr_q) cudaFree(H->sr_q);
    if (H->sp_part) cudaFree(H->sp_part);
    alloc(&H->sr_q, (size_t)B);
    if (H->sr_dz1) cudaFree(H->sr_dz1);
    if (H->sr_q1) cudaFree(H->sr_q1);
    alloc(&H->sr_dz1, (size_t)B * L.h);
    alloc(&H->sr_q1, (size_t)B);
    const int nparts = Umma2Cfg<kTailBN>::kEpiSets * ((L.n + kTailBN - 1) / kTailBN);
    alloc(&H->sp_part, (size_t)nparts * B);
    H->sr_cap_B = B;
  }
}

void free_sr(Handle* H) {
  if (H->sr_gexec) cudaGraphExecDestroy(H->sr_gexec);
  H->sr_gexec = nullptr;
  void* ptrs[] = {H->cg_x, H->cg_r, H->cg_p, H->cg_g, H->cg_ap, H->sr_S, H->sr_C, H->SRh, H->SRl, H->cg_part, H->d_sr_scal, H->d_pmax,
                  H->sr_q, H->sp_part, H->sr_dz1, H->sr_q1, H->sr_p1f};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (H->h_sr_scal) cudaFreeHost(H->h_sr_scal);
}

void launch_sr_grad_from_G(Handle* H, double scale) {
  sr_grad_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(H->L.total, H->G, scale, H->cg_g);
  SR_CHECK();
  H->launches++;
}

void launch_sr_apply(Handle* H, double lr, const double* delta) {
  sr_apply_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(H->L.total, lr, delta, H->P);
  SR_CHECK();
  H->launches++;
}

// conjugate_gradient (optimizer.cpp:46-71) on v -> F v + lambda v for the gradient in H->cg_g;
// the solution lands in H->cg_x.  Returns false (with iterations / relative residual) when the
// residual contract ||(F + lambda I) x - g|| <= tol ||g|| is not met.
// The dense branch of sr_direction (optimizer.cpp:64-73, d <= 2000): an exact fp64 solve of
// (S~^T S~ / B + lambda I) delta = g by Cholesky (the reference's LDLT; same solution for this SPD
// system) in the smaller of the two spaces: d x d directly, or, when B <= d, the B x B system of
// the Woodbury identity delta = (g - S~^T (B lambda I + S~ S~^T)^{-1} S~ g) / lambda.  Accepted
// only if ||(F + lambda I) delta - g|| <= tol ||g|| (0 iterations reported, like the reference).
bool sr_dense_solve(Handle* H, int B, double lambda, double tol, bool centered, int* iterations, double* residual,
                    double* gnorm_out) {
  const int64_t total = H->L.total;
  sr_build_scores(H, B, centered);
  cg_init_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->cg_g, H->cg_x, H->cg_r, H->cg_p, H->cg_part);
  SR_CHECK();
  H->launches++;
  const double gnorm = std::sqrt(sum_parts(H, H->cg_part, kVecBlocks));
  if (gnorm_out) *gnorm_out = gnorm;
  *iterations = 0;
  *residual = 0.0;
  if (gnorm == 0.0) return true;
  const bool bspace = (int64_t)B <= total;
  const int m = bspace ? B : (int)total;
  if ((size_t)m * m + m > H->sr_C_cap) {
    if (H->sr_C) cudaFree(H->sr_C);
    VQMC_CUDA(cudaMalloc((void**)&H->sr_C, ((size_t)m * m + m) * sizeof(double)));
    H->sr_C_cap = (size_t)m * m + m;
  }
  const unsigned gblocks = (unsigned)(((int64_t)m * m + 255) / 256);
  double* rhs;
  if (bspace) {
    sr_gram_kernel<<<gblocks, 256, 0, H->stream>>>(m, total, total, 1, H->sr_S, 1.0, (double)B * lambda, H->sr_C);
    sr_dense_sp_kernel<<<B, kVecThreads, 0, H->stream>>>(total, H->sr_S, H->cg_g, H->sr_q);  // S~ g
    rhs = H->sr_q;
  } else {
    sr_gram_kernel<<<gblocks, 256, 0, H->stream>>>(m, B, 1, total, H->sr_S, 1.0 / (double)B, lambda, H->sr_C);
    VQMC_CUDA(cudaMemcpyAsync(H->cg_x, H->cg_g, total * sizeof(double), cudaMemcpyDeviceToDevice, H->stream));
    rhs = H->cg_x;
  }
  SR_CHECK();
  VQMC_CUDA(cudaMemsetAsync(H->d_pmax, 0, sizeof(unsigned), H->stream));  // (reused as the not-SPD flag)
  for (int j = 0; j < m; ++j) {
    const unsigned blocks = (unsigned)(((int64_t)(m - j) * 32 + 255) / 256);
    sr_chol_col_kernel<<<blocks, 256, 0, H->stream>>>(m, j, H->sr_C, H->d_pmax);
  }
  SR_CHECK();
  sr_chol_solve_kernel<<<1, 1024, 0, H->stream>>>(m, H->sr_C, rhs);
  SR_CHECK();
  if (bspace) {
    sr_dense_stu_kernel<<<(unsigned)((total + 127) / 128), 128, 0, H->stream>>>(B, total, H->sr_S, H->sr_q, 1.0,
                                                                                  H->cg_x);
    sr_woodbury_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->cg_g, 1.0 / lambda, H->cg_x);
    SR_CHECK();
  }
  H->launches += m + 5;
  unsigned not_spd = 0;
  VQMC_CUDA(cudaMemcpyAsync(&not_spd, H->d_pmax, sizeof(unsigned), cudaMemcpyDeviceToHost, H->stream));
  VQMC_CUDA(cudaStreamSynchronize(H->stream));
  if (not_spd) {
    *residual = INFINITY;
    return false;
  }
  // residual contract with the exact operator
  VQMC_CUDA(cudaMemcpyAsync(H->cg_p, H->cg_x, total * sizeof(double), cudaMemcpyDeviceToDevice, H->stream));
  apply_fisher_dense(H, B);
  sr_resid_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->cg_ap, H->cg_x, lambda, H->cg_g, H->cg_part);
  SR_CHECK();
  H->launches++;
  *residual = std::sqrt(sum_parts(H, H->cg_part, kVecBlocks)) / gnorm;
  return *residual <= tol;
}

bool sr_solve(Handle* H, int B, double lambda, double tol, int max_iterations, bool centered, int* iterations,
              double* residual, double* gnorm_out) {
  const Layout& L = H->L;
  const int64_t total = L.total;
  // optimizer.cpp:66: the reference solves the dense system when d <= 2000
  if (H->d <= 2000) {
    if (H->nranks > 1) throw InvalidArgument("multi-GPU SR needs the CG path (reference d > 2000)");
    return sr_dense_solve(H, B, lambda, tol, centered, iterations, residual, gnorm_out);
  }
  cg_init_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->cg_g, H->cg_x, H->cg_r, H->cg_p, H->cg_part);
  SR_CHECK();
  H->launches++;
  double rs = sum_parts(H, H->cg_part, kVecBlocks);  // (also leaves rs in d_sr_scal[0])
  const double rhs_norm = std::sqrt(rs);
  if (gnorm_out) *gnorm_out = rhs_norm;
  int it_done = 0;
  if (rhs_norm == 0.0) {
    *iterations = 0;
    *residual = 0.0;
    return true;
  }
  sr_dz1_kernel<<<(unsigned)(((int64_t)B * L.h + 255) / 256), 256, 0, H->stream>>>(B, L.h, H->splits, H->Epart,
                                                                                      H->G1, H->sr_dz1);
  VQMC_CUDA(cudaMemsetAsync(H->d_pmax, 0, sizeof(unsigned), H->stream));
  sr_pmax_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(L.off_w2, L.total, H->cg_p, H->d_pmax);
  SR_CHECK();
  H->launches++;
  static const bool host_loop = [] {
    const char* e = std::getenv("VQMC_SR_HOST_LOOP");
    return e && e[0] == '1';
  }();
  if (H->nranks == 1 && max_iterations > 0 && H->sr_device_loop && !host_loop) {
    // one graph launch runs the whole solve: the iterations repeat under a conditional node until
    // the device-side test stops them (no host round trip per iteration)
    cg_state_init_kernel<<<1, 1, 0, H->stream>>>(H->d_sr_scal);
    SR_CHECK();
    Handle::SrGraphKey key{true, B, H->cap_B, H->sr_cap_B, centered, lambda, tol, max_iterations};
    if (!H->sr_gexec || !(H->sr_gkey == key)) {
      if (H->sr_gexec) cudaGraphExecDestroy(H->sr_gexec);
      H->sr_gexec = nullptr;
      cudaGraph_t g = nullptr;
      VQMC_CUDA(cudaGraphCreate(&g, 0));
      try {
        cudaGraphConditionalHandle cond;
        VQMC_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = cond;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        VQMC_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        VQMC_CUDA(cudaStreamBeginCaptureToGraph(H->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        H->capturing = true;
        try {
          apply_fisher(H, B, centered);
          cg_pap_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->G, H->cg_p, lambda, H->cg_part);
          cg_alpha_kernel<<<1, kVecThreads, 0, H->stream>>>(kVecBlocks, H->cg_part, H->d_sr_scal);
          cg_xr_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->d_sr_scal, H->G, H->cg_p, lambda,
                                                                   H->cg_x, H->cg_r, H->cg_part);
          cg_check_kernel<<<1, kVecThreads, 0, H->stream>>>(cond, kVecBlocks, H->cg_part, H->d_sr_scal, tol,
                                                            max_iterations, H->d_pmax);
          cg_p_dev_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, L.off_w2, H->d_sr_scal, H->cg_r,
                                                                      H->cg_p, H->d_pmax);
          SR_CHECK();
        } catch (...) {
          H->capturing = false;
          cudaGraph_t tmp = nullptr;
          cudaStreamEndCapture(H->stream, &tmp);
          throw;
        }
        H->capturing = false;
        VQMC_CUDA(cudaStreamEndCapture(H->stream, &body));
        VQMC_CUDA(cudaGraphInstantiate(&H->sr_gexec, g, 0));
      } catch (...) {
        cudaGraphDestroy(g);
        throw;
      }
      cudaGraphDestroy(g);
      H->sr_gkey = key;
    }
    VQMC_CUDA(cudaGraphLaunch(H->sr_gexec, H->stream));
    VQMC_CUDA(cudaMemcpyAsync(H->h_sr_scal, H->d_sr_scal, 8 * sizeof(double), cudaMemcpyDeviceToHost, H->stream));
    VQMC_CUDA(cudaStreamSynchronize(H->stream));
    const int it = (int)H->h_sr_scal[6];
    H->launches += (int64_t)it * 10;
    *iterations = it;
    *residual = std::sqrt(H->h_sr_scal[5]) / rhs_norm;
    return *residual <= tol;
  }
  for (int it = 0; it < max_iterations; ++it) {
    apply_fisher(H, B, centered);
    cg_pap_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->G, H->cg_p, lambda, H->cg_part);
    cg_alpha_kernel<<<1, kVecThreads, 0, H->stream>>>(kVecBlocks, H->cg_part, H->d_sr_scal);
    cg_xr_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, H->d_sr_scal, H->G, H->cg_p, lambda, H->cg_x,
                                                             H->cg_r, H->cg_part);
    SR_CHECK();
    H->launches += 3;
    it_done = it + 1;
    const double rs_next = sum_parts(H, H->cg_part, kVecBlocks);  // the convergence test (host)
    if (std::sqrt(rs_next) <= tol * rhs_norm) {
      rs = rs_next;
      break;
    }
    VQMC_CUDA(cudaMemsetAsync(H->d_pmax, 0, sizeof(unsigned), H->stream));
    cg_p_kernel<<<kVecBlocks, kVecThreads, 0, H->stream>>>(total, L.off_w2, rs_next / rs, H->cg_r, H->cg_p,
                                                            H->d_pmax);
    SR_CHECK();
    H->launches++;
    rs = rs_next;
  }
  *iterations = it_done;
  *residual = std::sqrt(rs) / rhs_norm;
  return *residual <= tol;
}

}  // namespace vqmc_b200

// Test hook: x = A^{-1} b through the SR dense Cholesky kernels (A: m x m SPD, row-major; only
// its lower triangle is read).  Returns 1 if the factorization flagged A as not SPD.
extern "C" int vqmc_test_sr_chol(int m, const double* A, const double* b, double* x) {
  using namespace vqmc_b200;
  double *dC = nullptr, *dx = nullptr;
  unsigned* flag = nullptr;
  cudaMalloc((void**)&dC, ((size_t)m * m + m) * sizeof(double));
  cudaMalloc((void**)&dx, (size_t)m * sizeof(double));
  cudaMalloc((void**)&flag, sizeof(unsigned));
  cudaMemcpy(dC, A, (size_t)m * m * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(dx, b, (size_t)m * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemset(flag, 0, sizeof(unsigned));
  for (int j = 0; j < m; ++j)
    sr_chol_col_kernel<<<(unsigned)(((int64_t)(m - j) * 32 + 255) / 256), 256>>>(m, j, dC, flag);
  sr_chol_solve_kernel<<<1, 1024>>>(m, dC, dx);
  unsigned f = 0;
  cudaMemcpy(&f, flag, sizeof(unsigned), cudaMemcpyDeviceToHost);
  cudaMemcpy(x, dx, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  cudaFree(dC);
  cudaFree(dx);
  cudaFree(flag);
  return e != cudaSuccess ? -1 : (int)f;
}
