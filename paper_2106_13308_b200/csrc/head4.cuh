// Head sampler v4 staging layout (head4.cu): where every head-block weight lives.
//
// The sequential head bits i < Hd (fast MADE structure: bit i completes hidden unit i) are
// processed one 32-bit word m at a time.  Inside the word a warp runs the serial chain with the
// word's own 32 x 32 blocks held in registers (TRI); the contributions of word m to all LATER
// words' slots are applied once per word as tensor-core MMAs (mma.sync m16n8k16, fp16 pairs,
// fp32 accumulators: slots x the CTA's 8 samples x the word's 32 bits), whose A operands are the
// AF blocks below, pre-arranged in the m16n8k16 A-fragment order so one 16-byte shared load
// per lane gives one fragment.
//
//   TRI[m][l'][lane]      = W1[32m + lane][32m + l']   (l' <= lane, else 0)   in-word z1 updates
//   TRI[m][32 + l'][lane] = W2[32m + lane][32m + l']   (l' <  lane, else 0)   in-word z2 updates
//   AF chunk (m, r, z) = 16 KB: [w 8][ks 2][hl 2][lane 32][8 halves], tile j = 8 r + w of 16
//     slots; z = 0: A[s][k] = W1[s][32m + 16ks + k] (slot s = hidden unit), z = 1: A[s][k] =
//     W2[s][32m + 16ks + k] (slot s = head output); hl = fp16 hi / lo of the pair.
// Only slots of later words (s >= 32 (m + 1)) are stored in AF; every such weight is unmasked.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace vqmc_b200 {

struct Head4Stage {
  __half* AF;  // [nwords][KG][2][8][2][2][256] halves (16 KB per (word, round, z) chunk)
  float* TRI;  // [nwords][64][32]
  int KG;      // rounds of 8 tiles (h <= 128 KG)
};

__host__ __device__ __forceinline__ int64_t head4_af_off(int KG, int m, int r, int z, int w, int ks, int hl) {
  return ((((((int64_t)m * KG + r) * 2 + z) * 8 + w) * 2 + ks) * 2 + hl) * 256;
}
__host__ __device__ __forceinline__ int64_t head4_chunk_off(int KG, int m, int r, int z) {
  return (((int64_t)m * KG + r) * 2 + z) * 8192;  // halves
}

// A[s][b] of word m = b >> 5 (slot s in a later word), as its fp16 pair, in fragment order.
__device__ __forceinline__ void head4_put_frag(const Head4Stage& S, int s, int b, int z, float p) {
  const int m = b >> 5, jt = s >> 4, r = jt >> 3, w = jt & 7, ks = (b >> 4) & 1, kk = b & 15, row = s & 15;
  const int reg = (row >> 3) | ((kk >> 3) << 1);
  const int lane = (row & 7) * 4 + ((kk & 7) >> 1);
  const int64_t o = head4_af_off(S.KG, m, r, z, w, ks, 0) + lane * 8 + reg * 2 + (kk & 1);
  const __half hi = __float2half_rn(p);
  S.AF[o] = hi;
  S.AF[o + 256] = __float2half_rn(p - __half2float(hi));
}

// W1T[j][k] = W1[k][j]: input bit j of hidden unit k (masked, i.e. zero, for j > k).
__device__ __forceinline__ void head4_put_w1(const Head4Stage& S, int j, int k, float p) {
  const int m = j >> 5, mk = k >> 5;
  if (mk == m) {
    if (j <= k) S.TRI[((int64_t)m * 64 + (j & 31)) * 32 + (k & 31)] = p;
  } else if (mk > m) {
    head4_put_frag(S, k, j, 0, p);
  }
}
// W2[i][k]: head output i from hidden unit k (= bit k; masked for k >= i).
__device__ __forceinline__ void head4_put_w2(const Head4Stage& S, int i, int k, float p) {
  const int m = k >> 5, mi = i >> 5;
  if (mi == m) {
    if (k < i) S.TRI[((int64_t)m * 64 + 32 + (k & 31)) * 32 + (i & 31)] = p;
  } else if (mi > m) {
    head4_put_frag(S, i, k, 1, p);
  }
}

}  // namespace vqmc_b200
