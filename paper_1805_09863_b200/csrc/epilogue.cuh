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

#ifndef AMUN_EXP
#define AMUN_EXP 0
#endif
namespace amun {
#if AMUN_EXP == 4
// instrumentation build only: [0] row-chunks, [1] row-chunks with a candidate,
// [2] insertions, [3] insertions into a filling list, [4] warp-chunks with a candidate
__device__ unsigned long long amun_dbg[8];
#define AMUN_DBG(i, n) atomicAdd(&amun_dbg[i], (unsigned long long)(n))
#endif

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

  // Insert a NEW element whose token id is larger than every id already in
  // the list (true inside one ascending scan): ties keep the older entries
  // ahead. All compares are independent and each slot is one select pair,
  // so the dependency depth is short (no carried compare-swap chain).
  __device__ __forceinline__ void insert_new(float x, int id) {
    bool b[KB];   // b[i]: entry i stays ahead of x; a prefix, since l is sorted
#pragma unroll
    for (int i = 0; i < KB; ++i) b[i] = l[i] >= x;
    shift_in(b, x, id);
  }

  // Slot i keeps its entry if it ranks ahead of the new one, else takes the
  // new one (first slot behind it) or its predecessor's entry.
  __device__ __forceinline__ void shift_in(const bool (&b)[KB], float x, int id) {
#pragma unroll
    for (int i = KB - 1; i >= 1; --i) {
      l[i] = b[i] ? l[i] : (b[i - 1] ? x : l[i - 1]);
      v[i] = b[i] ? v[i] : (b[i - 1] ? id : v[i - 1]);
    }
    l[0] = b[0] ? l[0] : x;
    v[0] = b[0] ? v[0] : id;
  }

  // Insert (x, id) ranking before the current KB-th entry, ids in any order:
  // entries ranking ahead of it under the full key (l desc, v asc) stay.
  __device__ __forceinline__ void insert_pos(float x, int id) {
#if AMUN_EXP == 1
    l[KB - 1] = x; v[KB - 1] = id; return;
#endif
#if AMUN_EXP == 4
    AMUN_DBG(2, 1);
    if (l[KB - 1] == kNegInf) AMUN_DBG(3, 1);
#endif
    bool b[KB];
#pragma unroll
    for (int i = 0; i < KB; ++i) b[i] = better_lv(l[i], v[i], x, id);
    shift_in(b, x, id);
  }

  // Register-only variant of chunk32 (no shared-memory staging): the same
  // statistics and gate; a candidate group's four values (x[g], x[g+8],
  // x[g+16], x[g+24]) are selected from registers by a 3-level select tree
  // and offered with the full tie key (ids arrive out of order).
  // group maxima g[j] = max(x[j], x[j+8], x[j+16], x[j+24]) and the chunk max
  __device__ __forceinline__ static float groups32(const float (&x)[32], float (&g)[8]) {
    float t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = fmaxf(x[j], x[j + 16]);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = fmaxf(t[j], t[j + 8]);
    return fmaxf(fmaxf(fmaxf(g[0], g[4]), fmaxf(g[1], g[5])),
                 fmaxf(fmaxf(g[2], g[6]), fmaxf(g[3], g[7])));
  }
  // Alg. 4's online update for a block whose maximum is cm: one rescale by
  // e^{m_old - m_new}, then sum exp(x - m) over the block.
  __device__ __forceinline__ void rescale(float cm) {
    if (cm > m) {
      s *= ex2((m - cm) * kLog2e);
      m = cm;
    }
  }
  // exp2 arguments and 8 running sums on packed fp32 pairs:
  // a[u] += e[u] + e[u+8] + e[u+16] + e[u+24] (in that order)
  __device__ __forceinline__ void expsum32(const float (&x)[32], float ms, float (&a)[8], bool first) {
    float e[32];
#pragma unroll
    for (int u = 0; u < 32; u += 2)
      ffma2(e[u], e[u + 1], x[u], x[u + 1], kLog2e, kLog2e, -ms, -ms);
#pragma unroll
    for (int u = 0; u < 32; ++u) e[u] = ex2(e[u]);
    if (first) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = e[u];
    } else {
#pragma unroll
      for (int u = 0; u < 8; u += 2) fadd2(a[u], a[u + 1], a[u], a[u + 1], e[u], e[u + 1]);
    }
#pragma unroll
    for (int j = 8; j < 32; j += 8)
#pragma unroll
      for (int u = 0; u < 8; u += 2) fadd2(a[u], a[u + 1], a[u], a[u + 1], e[j + u], e[j + u + 1]);
  }

  template <bool TOPK = true, bool STATS = true>
  __device__ __forceinline__ void chunk32r(const float (&x)[32], int vbase, float hint) {
    float g[8];
    const float cm = groups32(x, g);
    if (STATS && cm != kNegInf) {   // (STATS = false: Alg. 5 argmax only, no exp)
      rescale(cm);
      float a[8];
      expsum32(x, m * kLog2e, a, true);
      s += ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    if constexpr (TOPK) kbest32(x, g, cm, vbase, hint);
  }

  // The k-best step for one 32-column chunk with group maxima g and max cm.
  __device__ __forceinline__ void kbest32(const float (&x)[32], const float (&g)[8], float cm,
                                          int vbase, float hint) {
    if constexpr (KB == 1) {
      // Alg. 4 / Alg. 5 "if p' > max: best <- i", per chunk: only the chunk
      // maximum can replace the best; its token is the lowest index holding
      // it. Entries below the hint (a proven lower bound) are not offered.
      if (cm != kNegInf && cm >= hint && cm >= l[0]) {
        uint32_t msk = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) msk |= (x[j] == cm) ? (1u << j) : 0u;
        const int id = vbase + __ffs(msk) - 1;
        if (better_lv(cm, id, l[0], v[0])) {
          l[0] = cm;
          v[0] = id;
        }
      }
      return;
    }
    const float thr = l[KB - 1];
    float tg = (hint > thr) ? hint : thr;     // candidates: x >= tg (full key decides ties)
    if constexpr (KB <= 8) {
      if (__any_sync(0xffffffffu, thr == kNegInf)) {   // list filling: KB-th group maximum
        float q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = g[j];
#define AMUN_CS(a, b) { const float hi = fmaxf(q[a], q[b]); q[b] = fminf(q[a], q[b]); q[a] = hi; }
        AMUN_CS(0, 1) AMUN_CS(2, 3) AMUN_CS(4, 5) AMUN_CS(6, 7)
        AMUN_CS(0, 2) AMUN_CS(1, 3) AMUN_CS(4, 6) AMUN_CS(5, 7)
        AMUN_CS(1, 2) AMUN_CS(5, 6) AMUN_CS(0, 4) AMUN_CS(3, 7)
        AMUN_CS(1, 5) AMUN_CS(2, 6)
        AMUN_CS(1, 4) AMUN_CS(3, 6)
        AMUN_CS(2, 4) AMUN_CS(3, 5)
        AMUN_CS(3, 4)
#undef AMUN_CS
        if (q[KB - 1] > tg) tg = q[KB - 1];
      }
    }
    const bool need = cm >= tg && cm != kNegInf;
#if AMUN_EXP == 4
    if ((threadIdx.x & 31) == 0) {
      AMUN_DBG(0, __popc(__ballot_sync(0xffffffffu, cm != kNegInf)));
      AMUN_DBG(1, __popc(__ballot_sync(0xffffffffu, need)));
      if (__any_sync(0xffffffffu, need)) AMUN_DBG(4, 1);
    } else {
      __ballot_sync(0xffffffffu, cm != kNegInf); __ballot_sync(0xffffffffu, need); __any_sync(0xffffffffu, need);
    }
#endif
#if AMUN_EXP == 2
    if (__any_sync(0xffffffffu, need)) { if (need) { l[KB - 1] = cm; v[KB - 1] = vbase; } return; }
#endif
    if (__any_sync(0xffffffffu, need)) {
      uint32_t gm = 0;
      if (need) {
#pragma unroll
        for (int j = 0; j < 8; ++j) gm |= (g[j] >= tg) ? (1u << j) : 0u;
      }
      while (gm) {
        const int gi = __ffs(gm) - 1;
        gm &= gm - 1;
        float q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int b = 8 * u;
          const float s01 = (gi & 1) ? x[b + 1] : x[b + 0];
          const float s23 = (gi & 1) ? x[b + 3] : x[b + 2];
          const float s45 = (gi & 1) ? x[b + 5] : x[b + 4];
          const float s67 = (gi & 1) ? x[b + 7] : x[b + 6];
          const float s03 = (gi & 2) ? s23 : s01;
          const float s47 = (gi & 2) ? s67 : s45;
          q[u] = (gi & 4) ? s47 : s03;
        }
        // pre-check the 4 values; only qualifying ones (usually 1) are offered
        uint32_t em = (q[0] >= tg ? 1u : 0u) | (q[1] >= tg ? 2u : 0u) | (q[2] >= tg ? 4u : 0u) |
                      (q[3] >= tg ? 8u : 0u);
        while (em) {
          const int u = __ffs(em) - 1;
          em &= em - 1;
          const float xv = (u & 2) ? ((u & 1) ? q[3] : q[2]) : ((u & 1) ? q[1] : q[0]);
          const int id = vbase + gi + 8 * u;
          if (xv >= hint && better_lv(xv, id, l[KB - 1], v[KB - 1])) insert_pos(xv, id);
        }
      }
    }
  }

  // Consume 32 biased logits x[j] with token ids vbase + j, in ascending j.
  // Masked entries must already be -inf. `xs` is this thread's 32-float
  // shared-memory scratch row (128-byte aligned); its 16-byte chunks are
  // XOR-swizzled by `sw` (= row & 7) so a warp's stores are conflict-free.
  // `hint` is a proven lower bound for the row's k-th best logit (k entries
  // >= hint exist elsewhere in the row), so entries below it cannot be in
  // the row's top-k and are not offered (-inf when unknown).
  // Must be called by all 32 lanes of the warp together (warp-uniform gate).
  template <bool TOPK = true>
  __device__ __forceinline__ void chunk32(const float (&x)[32], int vbase, float* xs, int sw,
                                          float hint = kNegInf) {
    // max tree; g[j] = max(x[j], x[j+8], x[j+16], x[j+24]) (the group maxima)
    float t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = fmaxf(x[j], x[j + 16]);
    float g[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = fmaxf(t[j], t[j + 8]);
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = fmaxf(g[j], g[j + 4]);
    t[0] = fmaxf(fmaxf(t[0], t[2]), fmaxf(t[1], t[3]));
    const float cm = t[0];
    if (cm != kNegInf) {        // whole chunk masked: nothing to add (guards -inf - -inf)
      if (cm > m) {             // Alg. 4: new max -> rescale the sum by e^{Delta}
        s *= ex2((m - cm) * kLog2e);
        m = cm;
      }
      const float ms = m * kLog2e;
      // 8 independent chains so MUFU latency overlaps (one warp per SMSP
      // per group cannot hide it with other warps alone)
      float a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = ex2(fmaf(x[u], kLog2e, -ms));
#pragma unroll
      for (int j = 8; j < 32; j += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += ex2(fmaf(x[j + u], kLog2e, -ms));
      s += ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    // k-best (Alg. 4 "if p' > max ... best <- i", generalised to k): only
    // elements above the current k-th best can enter. The chunk max gates
    // the whole path; candidates are found with one bitmask and visited in
    // ascending j, each read back from shared memory.
    if constexpr (!TOPK) return;
    // single-compare gate: x >= tg  <=>  x > l[KB-1] && x >= hint
    const float thr = l[KB - 1];
    float tg = (hint > thr) ? hint : nextafterf(thr, __int_as_float(0x7f800000));
    if constexpr (KB <= 8) {
      // list still filling (start of a CTA range): the KB-th largest group
      // maximum is a lower bound on the chunk's KB-th best (KB distinct
      // elements reach it), so nothing below it can enter the row's top-KB
      if (__any_sync(0xffffffffu, thr == kNegInf)) {
        float q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = g[j];
        // sorting network for 8 (19 comparators), descending
#define AMUN_CS(a, b) { const float hi = fmaxf(q[a], q[b]); q[b] = fminf(q[a], q[b]); q[a] = hi; }
        AMUN_CS(0, 1) AMUN_CS(2, 3) AMUN_CS(4, 5) AMUN_CS(6, 7)
        AMUN_CS(0, 2) AMUN_CS(1, 3) AMUN_CS(4, 6) AMUN_CS(5, 7)
        AMUN_CS(1, 2) AMUN_CS(5, 6) AMUN_CS(0, 4) AMUN_CS(3, 7)
        AMUN_CS(1, 5) AMUN_CS(2, 6)
        AMUN_CS(1, 4) AMUN_CS(3, 6)
        AMUN_CS(2, 4) AMUN_CS(3, 5)
        AMUN_CS(3, 4)
#undef AMUN_CS
        if (q[KB - 1] > tg) tg = q[KB - 1];
      }
    }
    const bool need = cm >= tg;
    if (__any_sync(0xffffffffu, need)) {
      if (need) {
        // stage the chunk group-transposed: slot j holds (x[j], x[j+8], x[j+16],
        // x[j+24]), 16-byte slots XOR-swizzled by `sw`
        float4* xs4 = reinterpret_cast<float4*>(xs);
#pragma unroll
        for (int j = 0; j < 8; ++j) xs4[j ^ sw] = make_float4(x[j], x[j + 8], x[j + 16], x[j + 24]);
        // candidate groups first (8 compares), then only their 4 values
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (g[j] >= tg) {
            const float4 q = xs4[j ^ sw];
            mask |= (q.x >= tg ? (1u << j) : 0u) | (q.y >= tg ? (1u << (j + 8)) : 0u) |
                    (q.z >= tg ? (1u << (j + 16)) : 0u) | (q.w >= tg ? (1u << (j + 24)) : 0u);
          }
        }
        while (mask) {   // ascending token id, so ties keep the earlier entries ahead
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          const float xv = xs[(((j & 7) ^ sw) << 2) | (j >> 3)];
          if (xv > l[KB - 1]) insert_new(xv, vbase + j);
        }
      }
      __syncwarp();
    }
  }

  // Monoid combine with another partial state over a disjoint column set
  // (the rescale of P:195-197 and a k-best union with the full tie key).
  __device__ __forceinline__ void combine(float m2, float s2, const float* l2, const int* v2) {
    const float mn = fmaxf(m, m2);
    if (mn != kNegInf) {
      s = (m == kNegInf ? 0.f : s * ex2((m - mn) * kLog2e)) +
          (m2 == kNegInf ? 0.f : s2 * ex2((m2 - mn) * kLog2e));
      m = mn;
    }
#pragma unroll
    for (int i = 0; i < KB; ++i)
      if (v2[i] >= 0 && better_lv(l2[i], v2[i], l[KB - 1], v[KB - 1])) insert(l2[i], v2[i]);
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

// Cross-CTA k-th-best hints: a per-row 64-bit word {generation, ordered float}
// updated with atomicMax. Any CTA's local k-th best value is a lower bound on
// the row's global k-th best, so every CTA may skip entries below the largest
// one published so far. The generation tag makes stale words from earlier
// launches read as "no hint" without a reset.
__device__ __forceinline__ uint32_t f2o(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t o) {
  return (o & 0x80000000u) ? __uint_as_float(o & 0x7fffffffu) : __uint_as_float(~o);
}
__device__ __forceinline__ float hint_decode(unsigned long long h, uint32_t gen) {
  return ((uint32_t)(h >> 32) == gen) ? o2f((uint32_t)h) : kNegInf;
}
__device__ __forceinline__ unsigned long long hint_encode(float x, uint32_t gen) {
  return ((unsigned long long)gen << 32) | f2o(x);
}

// Static persistent schedule shared by the fused kernels and the merge.
// The flattened column space has one band of `band` columns per M-tile, of
// which the first Vp (= V_local rounded up to 16) are real; CTA c owns the
// flat range [c*C, (c+1)*C) (C % 16 == 0) and walks its real columns in
// tiles of <= 256 columns; a range may span two M-tiles (segments). CTA c's
// partial for M-tile mt goes to slot c + mt (unique).
//   aligned mode: band = s*C with s splits per M-tile, so the CTAs of all
//     M-tiles start at the same vocab offsets and stream each W tile at the
//     same time (one HBM read, the other M-tiles hit in L2);
//   flattened mode: band = Vp, C = total / #SMs (many M-tiles).
struct Schedule {
  long long band, Vp, C, total;
  __device__ __forceinline__ long long first_cta(int mt) const { return (mt * band) / C; }
  __device__ __forceinline__ long long last_cta(int mt) const { return (mt * band + Vp - 1) / C; }
};

// The persistent schedule over n_mt row units x Vp vocab columns for G CTAs
// (or CTA pairs): aligned vocab splits (every unit cut at the same
// boundaries, so concurrent CTAs share W tiles in L2) when they fill >= 90%
// of G, else an equal flattened split. Shared by the host (plan) and the
// device (amun_output_layer_dev, where N is only known on the device).
// `align` (16, or 128 for MXFP4 plans, whose scale atoms cover 128 W rows):
// Vp and every CTA range start are multiples of it, so every tile starts on
// an aligned column.
__host__ __device__ inline Schedule schedule_for(long long n_mt, long long Vp, long long G,
                                                 long long align = 16) {
  Schedule s;
  s.Vp = Vp;
  const long long splits = G / n_mt;
  if (splits >= 1 && n_mt * splits * 10 >= G * 9) {
    s.C = ((Vp + splits - 1) / splits + align - 1) / align * align;
    s.band = (Vp + s.C - 1) / s.C * s.C;
  } else {
    s.C = ((n_mt * Vp + G - 1) / G + align - 1) / align * align;
    s.band = Vp;
  }
  s.total = n_mt * s.band;
  return s;
}

// Tile widths of a CTA range: 256 columns, except that with `taper` the
// range's final segment ends in narrower tiles (<= 64, and <= 128 before
// it), so the epilogue of the last tile — the drain after the last MMA,
// when nothing overlaps it — is short. All roles of a CTA (producer, MMA,
// epilogue) walk the same iterator, so they agree on every tile.
__device__ __forceinline__ int taper_width(long long rem) {
  if (rem <= 64) return (int)rem;
  if (rem <= 192) return (int)(rem - 64);
  if (rem <= 384) return (int)(rem - 128);
  return 256;
}

struct TileIter {
  long long pos, end;
  Schedule sch;
  int taper = 0;
  int wmax = 256;   // widest tile (224 for MXFP4: TMEM columns for the scale factors)
  __device__ __forceinline__ bool next(int& mt, int& v0, int& width, bool& last) {
    for (;;) {
      if (pos >= end) return false;
      mt = (int)(pos / sch.band);
      const long long base = (long long)mt * sch.band;
      if (pos - base >= sch.Vp) {  // padding of an aligned band: skip to the next band
        pos = base + sch.band;
        continue;
      }
      v0 = (int)(pos - base);
      const long long seg_end = min(base + sch.Vp, end) - base;
#ifdef TC_BN_OVERRIDE
      width = (int)min((long long)TC_BN_OVERRIDE, seg_end - v0);
#else
      width = (taper && base + sch.Vp >= end) ? taper_width(seg_end - v0)
                                              : (int)min((long long)wmax, seg_end - v0);
#endif
      last = (v0 + width == seg_end);
      pos += width;
      return true;
    }
  }
};

}  // namespace amun
