// epilogue.cuh — the fused bias + softmax-statistics + k-best step, per row.
//
// PAPER.md Alg. 4 keeps, in ONE pass over p, the running max,
// the running sum of exp(p - max) rescaled whenever the max grows
// (sum = e^{x_t - max_b} + e^{Delta} * sum, Delta = max_a - max_b;
// reading G1 — the pseudocode's "Delta x sum" is a typo for e^{Delta}), and
// the best class. Observation 2: probabilities are needed only for
// the winners, so the k-best is selected on the raw biased logits and
// normalised later (merge kernel). Here the scan is blocked by 32 columns:
// one max and one rescale per chunk, then 32 exps. The k-best is a sorted
// register array; the per-chunk max gates the (rare) insertion path, so the
// common case costs one compare per 32 logits.
#pragma once
#include <cstdint>
#include <math_constants.h>
#include "ptx.cuh"

namespace amun {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNegInf = -__builtin_huge_valf();

// a ranks before b: larger logit, then smaller token id (reading G3).
__device__ __forceinline__ bool better_lv(float al, int av, float bl, int bv) {
  return (al > bl) || (al == bl && av < bv);
}

template <int KB>
struct RowState {
  float m;        // running max of biased logits
  float s;        // running sum of exp(l - m)
  float l[KB];    // k-best biased logits, descending
  int v[KB];      // their global token ids

  __device__ __forceinline__ void reset() {
    m = kNegInf;
    s = 0.f;
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      l[i] = kNegInf;
      v[i] = -1;
    }
  }

  // Insert (x, id) keeping the array sorted by (l desc, v asc); the carried
  // element uses the full key so equal logits keep their token order.
  __device__ __forceinline__ void insert(float x, int id) {
    float cx = x;
    int cv = id;
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const bool b = better_lv(cx, cv, l[i], v[i]);
      const float tl = l[i];
      const int tv = v[i];
      l[i] = b ? cx : tl;
      v[i] = b ? cv : tv;
      cx = b ? tl : cx;
      cv = b ? tv : cv;
    }
  }

  // Consume 32 biased logits x[j] with token ids vbase + j, in ascending j.
  // Masked entries must already be -inf.
  __device__ __forceinline__ void chunk32(const float (&x)[32], int vbase) {
    float t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = fmaxf(x[j], x[j + 16]);
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
      for (int j = 0; j < w; ++j) t[j] = fmaxf(t[j], t[j + w]);
    const float cm = t[0];
    if (cm == kNegInf) return;  // whole chunk masked: nothing to add (guards -inf - -inf)
    if (cm > m) {               // Alg. 4: new max -> rescale the sum by e^{Delta}
      s *= ex2((m - cm) * kLog2e);
      m = cm;
    }
    const float ms = m * kLog2e;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      a0 += ex2(fmaf(x[j + 0], kLog2e, -ms));
      a1 += ex2(fmaf(x[j + 1], kLog2e, -ms));
      a2 += ex2(fmaf(x[j + 2], kLog2e, -ms));
      a3 += ex2(fmaf(x[j + 3], kLog2e, -ms));
    }
    s += (a0 + a1) + (a2 + a3);
    if (cm > l[KB - 1]) {  // Alg. 4 "if p' > max ... best <- i", generalised to k
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (x[j] > l[KB - 1]) insert(x[j], vbase + j);
    }
  }

  // Partial record {m, s, l[0..k_max), v[0..k_max)} (see amun.h).
  __device__ __forceinline__ void emit(float* rec, int k_max) const {
    rec[0] = m;
    rec[1] = s;
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      if (i < k_max) {
        rec[2 + i] = l[i];
        rec[2 + k_max + i] = __int_as_float(v[i]);
      }
    }
  }
};

// Static persistent schedule shared by the fused kernels and the merge.
// The flattened column space [0, n_mt * Vp) (Vp = V_local rounded up to 16)
// is cut into equal ranges of C columns (C % 16 == 0), one per CTA; a CTA
// walks its range in tiles of <= 256 columns; a range may span two M-tiles
// (segments). CTA c's partial for M-tile mt goes to slot c + mt (unique).
struct Schedule {
  long long Vp, C, total;
  __device__ __forceinline__ long long first_cta(int mt) const { return (mt * Vp) / C; }
  __device__ __forceinline__ long long last_cta(int mt) const { return ((mt + 1) * Vp - 1) / C; }
};

struct TileIter {
  long long pos, end, Vp;
  __device__ __forceinline__ bool next(int& mt, int& v0, int& width, bool& last) {
    if (pos >= end) return false;
    mt = (int)(pos / Vp);
    const long long base = (long long)mt * Vp;
    v0 = (int)(pos - base);
    const long long seg_end = min(base + Vp, end) - base;
    width = (int)min(256LL, seg_end - v0);
    last = (v0 + width == seg_end);
    pos += width;
    return true;
  }
};

}  // namespace amun
