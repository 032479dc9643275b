// merge.cuh — exact merge of partial states and per-sentence beam k-best.
//
// Row phase (the reduce step of Alg. 6, for (max, sum, k-best)
// states): for row r, over its partial records j in fixed order,
//   M = max_j m_j,  Z = sum_j s_j * exp(m_j - M)  (rescale of P:195-197),
//   lse_r = M + log Z,  row k-best = best k of the union (l desc, v asc).
// Sentence phase ("k-best ... simple extension", P:29 beam search;
// readings G4/G5): only the winners are normalised (observation 2):
//   cost = prev_cost[r] + (l - lse_r)
// and the top-k_s over the sentence's rows is selected by
// (cost desc, r asc, l desc, v asc). Per-row k-best with k >= k_s contains
// the sentence's top-k_s, so the selection is exact.
//
// mode ROW: writes one merged partial record per row (vocab-shard output).
// mode SENT: CTA per sentence, writes out_idx / out_cost.
#pragma once
#include "epilogue.cuh"

namespace amun {

struct MergeParams {
  // partial locator: layout 0 = fused-kernel slots [slot][128][stride] with
  // the Schedule; layout 2 = the same for CTA pairs; layout 1 = external
  // [G][N][stride]
  const float* __restrict__ part;
  int stride, k_max, layout, G;
  Schedule sch;
  int N, S;
  const float* __restrict__ prev_cost;
  const int* __restrict__ offsets;
  const int* __restrict__ k_s;
  int k;
  long long V_total;
  long long* __restrict__ out_idx;
  float* __restrict__ out_cost;
  float* __restrict__ out_part;  // ROW mode: [N][stride]
};

__device__ __forceinline__ void row_splits(const MergeParams& p, int r, const float*& base,
                                           long long& jstride, int& n) {
  if (p.layout == 0) {
    const int mt = r >> 7;
    const long long c0 = p.sch.first_cta(mt), c1 = p.sch.last_cta(mt);
    base = p.part + ((c0 + mt) * 128 + (r & 127)) * (long long)p.stride;
    jstride = 128LL * p.stride;
    n = (int)(c1 - c0 + 1);
  } else if (p.layout == 2) {
    // CTA pairs: slot (pair + mp) * 2 + rank holds M-tile 2 mp + rank
    const int mt = r >> 7, mp = mt >> 1, rk = mt & 1;
    const long long c0 = p.sch.first_cta(mp), c1 = p.sch.last_cta(mp);
    base = p.part + (((c0 + mp) * 2 + rk) * 128 + (r & 127)) * (long long)p.stride;
    jstride = 2LL * 128 * p.stride;
    n = (int)(c1 - c0 + 1);
  } else {
    base = p.part + (long long)r * p.stride;
    jstride = (long long)p.N * p.stride;
    n = p.G;
  }
}

struct Cand {
  float cost, l;
  int r, v;
};
// a ranks before b in a sentence
__device__ __forceinline__ bool better_cand(const Cand& a, const Cand& b) {
  if (a.cost != b.cost) return a.cost > b.cost;
  if (a.r != b.r) return a.r < b.r;
  if (a.l != b.l) return a.l > b.l;
  return a.v < b.v;
}
__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src_xor) {
  Cand o;
  o.cost = __shfl_xor_sync(0xffffffffu, c.cost, src_xor);
  o.l = __shfl_xor_sync(0xffffffffu, c.l, src_xor);
  o.r = __shfl_xor_sync(0xffffffffu, c.r, src_xor);
  o.v = __shfl_xor_sync(0xffffffffu, c.v, src_xor);
  return o;
}

template <int KB>
struct CandList {  // sorted by better_cand, capacity KB
  Cand c[KB];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int i = 0; i < KB; ++i) c[i] = Cand{kNegInf, kNegInf, 0x7fffffff, 0x7fffffff};
  }
  __device__ __forceinline__ void insert(Cand x) {
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const bool b = better_cand(x, c[i]);
      const Cand t = c[i];
      c[i] = b ? x : t;
      x = b ? t : x;
    }
  }
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int i = 0; i + 1 < KB; ++i) c[i] = c[i + 1];
    c[KB - 1] = Cand{kNegInf, kNegInf, 0x7fffffff, 0x7fffffff};
  }
};

// Row phase for row r, executed by one full warp. Returns lse (all lanes);
// lane i < k_max receives the i-th best (l, v) of the row in (ol, ov).
// Lane j takes record j (already sorted by the producer, so it IS the lane's
// list); records j + 32, j + 64, ... (only with > 32 splits) are inserted.
template <int KB>
__device__ __forceinline__ void merge_row(const MergeParams& p, int r, int lane, float& M_out,
                                          float& Z_out, float& ol, int& ov) {
  const float* base;
  long long js;
  int n;
  row_splits(p, r, base, js, n);
  RowState<KB> lst;
  lst.reset();
  float m0 = kNegInf, s0 = 0.f;
  if (lane < n) {
    const float* rec = base + lane * js;
    m0 = rec[0];
    s0 = rec[1];
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      if (i < p.k_max) {
        lst.l[i] = rec[2 + i];
        lst.v[i] = __float_as_int(rec[2 + p.k_max + i]);
      }
    }
  }
  float M = m0;
  for (int j = lane + 32; j < n; j += 32) {
    const float* rec = base + j * js;
    M = fmaxf(M, rec[0]);
    for (int i = 0; i < p.k_max; ++i) {
      const float li = rec[2 + i];
      const int vi = __float_as_int(rec[2 + p.k_max + i]);
      if (vi >= 0 && better_lv(li, vi, lst.l[KB - 1], lst.v[KB - 1])) lst.insert(li, vi);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float Z = (m0 != kNegInf) ? s0 * expf(m0 - M) : 0.f;
  for (int j = lane + 32; j < n; j += 32) {
    const float* rec = base + j * js;
    const float mj = rec[0];
    if (mj != kNegInf) Z += rec[1] * expf(mj - M);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
  M_out = M;
  Z_out = Z;
  ol = kNegInf;
  ov = -1;
  for (int i = 0; i < p.k_max; ++i) {
    float bl = lst.l[0];
    int bv = lst.v[0];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const float tl = __shfl_xor_sync(0xffffffffu, bl, o);
      const int tv = __shfl_xor_sync(0xffffffffu, bv, o);
      if (tv >= 0 && (bv < 0 || better_lv(tl, tv, bl, bv))) {
        bl = tl;
        bv = tv;
      }
    }
    if (bv < 0) break;  // warp-uniform: no more candidates
    if (lst.v[0] == bv) {  // owner pops (token ids are unique within a row)
#pragma unroll
      for (int t = 0; t + 1 < KB; ++t) {
        lst.l[t] = lst.l[t + 1];
        lst.v[t] = lst.v[t + 1];
      }
      lst.l[KB - 1] = kNegInf;
      lst.v[KB - 1] = -1;
    }
    if (lane == i) {
      ol = bl;
      ov = bv;
    }
  }
}

constexpr int MG_WARPS = 8;

template <int KB>
__global__ void __launch_bounds__(MG_WARPS * 32) merge_rows_kernel(const MergeParams p) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * MG_WARPS + warp;
  if (r >= p.N) return;
  float M, Z, l;
  int v;
  merge_row<KB>(p, r, lane, M, Z, l, v);
  float* rec = p.out_part + (long long)r * p.stride;
  if (lane == 0) {
    rec[0] = M;
    rec[1] = Z;
  }
  if (lane < p.k_max) {
    rec[2 + lane] = l;
    rec[2 + p.k_max + lane] = __int_as_float(v);
  }
}

__device__ __forceinline__ Cand shfl_cand_idx(const Cand& c, int src) {
  Cand o;
  o.cost = __shfl_sync(0xffffffffu, c.cost, src);
  o.l = __shfl_sync(0xffffffffu, c.l, src);
  o.r = __shfl_sync(0xffffffffu, c.r, src);
  o.v = __shfl_sync(0xffffffffu, c.v, src);
  return o;
}

// Sentence phase. CTA = one sentence, warp w takes rows r0+w, r0+w+8, ...
// Per row: lse from a warp max/sum over the row's partial records, then every
// lane offers the (l, v) entries of its records, scored
// cost = prev_cost[r] + (l - lse), to a lane-local sorted list. Each warp
// extracts its top-KB (KB rounds of warp argmax) into shared memory; after ONE
// barrier, warp 0 ranks the <= 8*KB survivors by counting better ones and
// writes rank i to output slot i (ranks are unique: (r, v) pairs are).
constexpr int MS_WARPS = 8;

template <int KB>
__global__ void __launch_bounds__(MS_WARPS * 32) merge_sentences_kernel(const MergeParams p) {
  __shared__ Cand pool[MS_WARPS * KB];
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // inputs that do not come from the fused kernel are read before the
  // programmatic-dependent-launch wait, so their latency overlaps its tail
  const int r0 = p.offsets[s], r1 = p.offsets[s + 1];
  const int ks = p.k_s ? min(p.k_s[s], p.k) : p.k;
  float pc = 0.f;
  if (r0 + warp < r1) pc = p.prev_cost[r0 + warp];
  pdl_wait();
  CandList<KB> cl;
  cl.reset();
  for (int r = r0 + warp; r < r1; r += MS_WARPS) {
    if (r != r0 + warp) pc = p.prev_cost[r];
    const float* base;
    long long js;
    int n;
    row_splits(p, r, base, js, n);
    float M = kNegInf;
    for (int j = lane; j < n; j += 32) M = fmaxf(M, base[j * js]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float Z = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float* rec = base + j * js;
      const float mj = rec[0];
      if (mj != kNegInf) Z += rec[1] * expf(mj - M);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
    const float lse = M + logf(Z);
    for (int j = lane; j < n; j += 32) {
      const float* rec = base + j * js;
      for (int i = 0; i < p.k_max; ++i) {
        const int vi = __float_as_int(rec[2 + p.k_max + i]);
        if (vi < 0) break;
        const float li = rec[2 + i];
        const Cand c{pc + (li - lse), li, r, vi};
        if (!better_cand(c, cl.c[KB - 1])) break;   // entries are sorted: the rest lose too
        cl.insert(c);
      }
    }
  }
  // warp top-KB -> shared pool
  for (int i = 0; i < KB; ++i) {
    Cand b = cl.c[0];
    int src = lane;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const Cand t = shfl_cand(b, o);
      const int ts = __shfl_xor_sync(0xffffffffu, src, o);
      if (better_cand(t, b) || (!better_cand(b, t) && ts < src)) {
        b = t;
        src = ts;
      }
    }
    if (lane == src) cl.pop();
    if (lane == 0) pool[warp * KB + i] = b;
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int NP = MS_WARPS * KB;
    int nvalid = 0;
    for (int e = lane; e < NP; e += 32) {
      const Cand c = pool[e];
      const bool valid = (c.v >= 0) && (c.v != 0x7fffffff);
      nvalid += valid;
      if (!valid) continue;
      int rank = 0;
      for (int f = 0; f < NP; ++f) rank += better_cand(pool[f], c) ? 1 : 0;
      if (rank < ks) {
        p.out_idx[(long long)s * p.k + rank] = (long long)c.r * p.V_total + c.v;
        p.out_cost[(long long)s * p.k + rank] = c.cost;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
    const int filled = min(ks, nvalid);
    for (int i = filled + lane; i < p.k; i += 32) {
      p.out_idx[(long long)s * p.k + i] = -1LL;
      p.out_cost[(long long)s * p.k + i] = kNegInf;
    }
  }
}

}  // namespace amun
