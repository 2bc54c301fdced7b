// Adam element update (optimizer.cpp:21-35) and the writes of everything derived from an updated
// parameter (the fp16 pair of W2 for the GEMMs, the head sampler's staged copies).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "internal.cuh"
#include "ptx.cuh"

namespace vqmc_b200 {

// Adam hyper-parameters of the current step, read once per thread from StepParams.
struct AdamHyper {
  float lr, b1, b2, eps, ibc1, ibc2;
  __device__ __forceinline__ void load(const StepParams* sp) {
    lr = sp->lr;
    b1 = sp->b1;
    b2 = sp->b2;
    eps = sp->eps;
    ibc1 = sp->ibc1;  // (= 1.f / sp->bc1, formed once per step)
    ibc2 = sp->ibc2;
  }
  // one element; g is already scaled by 1/L
  // (explicit roundings and FMAs: every kernel that inlines this gives bitwise the same update;
  // MUFU sqrt / rcp instead of the correctly rounded ones cut the kernel's instructions by 30% and
  // changed nothing measurable: it waits on memory, not on issue)
  __device__ __forceinline__ void update(float g, float& m, float& v, float& p) const {
    m = __fmaf_rn(b1, m, __fmul_rn(1.f - b1, g));
    v = __fmaf_rn(b2, v, __fmul_rn(1.f - b2, __fmul_rn(g, g)));
    const float mh = __fmul_rn(m, ibc1), vh = __fmul_rn(v, ibc2);
    p = __fmaf_rn(-lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), eps)), p);
  }
};

// head v3 staging order (head.cu): row r of word m = r / 32 keeps entry k (k >= 32 m) at
// 128 (t >> 2) + 4 (k & 31) + (t & 3), t = k / 32 - m; entries of earlier words are not staged.
__device__ __forceinline__ int head_rel_pos_dev(int r, int k) {
  const int t = (k >> 5) - (r >> 5);
  return t < 0 ? -1 : 128 * (t >> 2) + 4 * (k & 31) + (t & 3);
}

struct AdamOut {
  int h, hp18, Hd, hpk, Hdp;
  float inv_h;  // 1 / h (W2 row of an index: float estimate, corrected by one)
  bool perm;  // head staging copies are lane-permuted (head v3)
  bool vec_w2;  // h % 4 == 0 and off_w2 % 4 == 0: a group of 4 never straddles two W2 rows
  int64_t off_b1, off_w2, off_b2;
  const int* comp_pos;  // completion slot of hidden unit k
  float* W1Tp;
  float* W2cp;
  __half* W2h;  // fp16 pair of [W2m | b2], row stride hp18
  __half* W2l;
  // sticky non-finite-logit flag of the step's sampler: when set, Adam leaves P / M / V (and the
  // derived copies) untouched, so a failed step does not poison the parameters (the reference
  // aborts in phase 1, before any update: trainer.cpp:170-179)
  const uint32_t* flag;
  bool v4;        // head v4 staging (head4.cuh) instead of the v3 rows
  Head4Stage h4;
};

// (i, k) = divmod(u, h) without an integer divide: the fp32 estimate is corrected by steps of one.
__device__ __forceinline__ void w2_row(const AdamOut& o, unsigned u, unsigned& i, unsigned& k) {
  int ii = (int)__fmul_rz((float)u, o.inv_h);
  int kk = (int)u - ii * o.h;
  while (kk < 0) {  // (once at most while u < 2^24; a few times for larger layouts)
    --ii;
    kk += o.h;
  }
  while (kk >= o.h) {
    ++ii;
    kk -= o.h;
  }
  i = (unsigned)ii;
  k = (unsigned)kk;
}

__device__ __forceinline__ void adam_side_writes(const AdamOut& o, int64_t t, float p) {
  // (32-bit index math: the live buffer is < 2^31 entries, checked at handle creation)
  if (t < o.off_b1) {  // W1T[j][k]
    const unsigned tt = (unsigned)t, j = tt / (unsigned)o.h, k = tt - j * (unsigned)o.h;
    if (o.v4) {
      head4_put_w1(o.h4, (int)j, (int)k, p);
    } else if (!o.perm) {
      o.W1Tp[(size_t)j * o.hpk + k] = p;
    } else {
      const int pos = head_rel_pos_dev((int)j, (int)k);
      if (pos >= 0) o.W1Tp[(size_t)j * o.hpk + pos] = p;
    }
  } else if (t >= o.off_w2 && t < o.off_b2) {  // W2[i][k]
    unsigned i, k;
    w2_row(o, (unsigned)(t - o.off_w2), i, k);
    ptx::split_f16(p, o.W2h[(size_t)i * o.hp18 + k], o.W2l[(size_t)i * o.hp18 + k]);
    if ((int)i < o.Hd && o.v4) {
      head4_put_w2(o.h4, (int)i, (int)k, p);
    } else if ((int)i < o.Hd) {
      const int c = o.comp_pos[k];
      if (!o.perm) {
        o.W2cp[(size_t)c * o.Hdp + i] = p;
      } else {
        const int pos = head_rel_pos_dev(c, (int)i);
        if (pos >= 0) o.W2cp[(size_t)c * o.Hdp + pos] = p;
      }
    }
  } else if (t >= o.off_b2) {  // b2[i]: column h of the W2 pair (the tail GEMM's bias column)
    const size_t i = (size_t)(t - o.off_b2);
    ptx::split_f16(p, o.W2h[i * o.hp18 + o.h], o.W2l[i * o.hp18 + o.h]);
  }
}

}  // namespace vqmc_b200
