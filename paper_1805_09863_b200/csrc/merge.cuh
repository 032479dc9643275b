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
  long long part_floats;          // capacity of part (checked builds; 0 = unchecked)
  const int* __restrict__ N_dev; // amun_output_layer_dev: N on the device (layout 0), else NULL
  int num_sms;
};

// amun_output_layer_dev: the row count and the fused kernel's schedule are
// resolved on the device (the same schedule_for as the fused kernel).
__device__ __forceinline__ MergeParams merge_dyn(const MergeParams& p) {
  MergeParams q = p;
  if (p.N_dev) {
    q.N = max(0, min(*p.N_dev, p.N));
    const int unit = p.layout == 2 ? 256 : 128;   // layout 2: CTA-pair units
    q.sch = schedule_for((max(q.N, 1) + unit - 1) / unit, p.sch.Vp,
                         p.layout == 2 ? p.num_sms / 2 : p.num_sms);
  }
  return q;
}

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
  // every record of the row inside the partial buffer
  AMUN_DCHECK(r >= 0 && r < p.N && n >= 1 && base >= p.part &&
              (p.part_floats == 0 ||
               (base - p.part) + (n - 1) * jstride + p.stride <= p.part_floats));
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

// ---------------------------------------------------------------- row phase v3
// 64-bit sort key of a row entry: ordered logit in the high word, inverted
// token id in the low word, so a plain max picks (l desc, v asc); 0 = empty.
__device__ __forceinline__ unsigned long long lv_key(float l, int v) {
  return v < 0 ? 0ull : (((unsigned long long)f2o(l) << 32) | (uint32_t)(0x7fffffff - v));
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y > x ? y : x;
  }
  return x;
}

// One partial record {m, s, l[k_max], v[k_max]} into registers. With
// k_max == KB the layout is static and the record (2 + 2 KB floats, 8-byte
// aligned) is read as float2 pairs: half the load instructions, which matters
// when one SM reads a row's ~148 scattered records (small batches).
template <int KB>
__device__ __forceinline__ void load_record(const MergeParams& p, const float* rec, bool ok,
                                            float& m, float& s, float (&l)[KB], int (&v)[KB]) {
  m = kNegInf;
  s = 0.f;
#pragma unroll
  for (int i = 0; i < KB; ++i) {
    l[i] = kNegInf;
    v[i] = -1;
  }
  if (!ok) return;
  if (p.k_max == KB) {
    float f[2 + 2 * KB];
    if constexpr ((2 + 2 * KB) % 4 == 0) {   // odd KB: whole 16-byte units when aligned
      if ((reinterpret_cast<uintptr_t>(rec) & 15) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(rec);
#pragma unroll
        for (int t = 0; t < (2 + 2 * KB) / 4; ++t) {
          const float4 q = r4[t];
          f[4 * t] = q.x;
          f[4 * t + 1] = q.y;
          f[4 * t + 2] = q.z;
          f[4 * t + 3] = q.w;
        }
      } else {
        const float2* r2 = reinterpret_cast<const float2*>(rec);
#pragma unroll
        for (int t = 0; t < 1 + KB; ++t) {
          const float2 q = r2[t];
          f[2 * t] = q.x;
          f[2 * t + 1] = q.y;
        }
      }
    } else {
      const float2* r2 = reinterpret_cast<const float2*>(rec);
#pragma unroll
      for (int t = 0; t < 1 + KB; ++t) {
        const float2 q = r2[t];
        f[2 * t] = q.x;
        f[2 * t + 1] = q.y;
      }
    }
    m = f[0];
    s = f[1];
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      l[i] = f[2 + i];
      v[i] = __float_as_int(f[2 + KB + i]);
    }
  } else {
    m = rec[0];
    s = rec[1];
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      if (i < p.k_max) {
        l[i] = rec[2 + i];
        v[i] = __float_as_int(rec[2 + p.k_max + i]);
      }
    }
  }
}

// One full warp over n partial records at base + j * js, j = lane, lane +
// step, ... (step = 32: all of a row's records; a multiple of 32: one warp's
// share when a row's records are split over several warps): M + log Z and the
// top-k_max (l, v) of their union. Lane i < k_max receives entry i (v = -1 if none).
template <int KB>
__device__ __forceinline__ void records_topk(const MergeParams& p, const float* base, long long js,
                                             int n, int step, int lane, float& lse, float& M_out,
                                             float& Z_out, float& ol, int& ov) {
  RowState<KB> lst;      // lane-local sorted list (l desc, v asc)
  lst.reset();
  float m0, s0;           // record `lane` is already sorted: it is the lane's list
  load_record<KB>(p, base + (lane < n ? lane : 0) * js, lane < n, m0, s0, lst.l, lst.v);
  // Lower bound on the row's k-th best: some lane holds k_max entries >= its
  // own k-th (one record's sorted top-k), so entries of further records below
  // the warp maximum of those can be skipped (ties are kept: the full key
  // decides them). Most of a row's ~148 records (one M-tile over all CTAs)
  // then contribute no insertion at all.
  auto kth_bound = [&]() {
    float T = (p.k_max == KB) ? lst.l[KB - 1] : kNegInf;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) T = fmaxf(T, __shfl_xor_sync(0xffffffffu, T, o));
    return T;
  };
  float M = m0, Z;
  constexpr int RMAX = (KB <= 6) ? 4 : 1;   // further records per lane held in registers
  if (KB <= 6 && n <= (RMAX + 1) * step) {
    // every further record of this lane loaded in ONE round of independent
    // loads (the merge is latency-bound: each dependent round costs ~1 us)
    float xm[RMAX], xs[RMAX], xl[RMAX][KB];
    int xv[RMAX][KB];
#pragma unroll
    for (int t = 0; t < RMAX; ++t) {
      const int j = lane + (t + 1) * step;
      load_record<KB>(p, base + (j < n ? j : 0) * js, j < n, xm[t], xs[t], xl[t], xv[t]);
    }
    const float T = (n > step) ? kth_bound() : kNegInf;
#pragma unroll
    for (int t = 0; t < RMAX; ++t) {
      M = fmaxf(M, xm[t]);
#pragma unroll
      for (int i = 0; i < KB; ++i) {   // a record is sorted: stop at its first loser
        if (xv[t][i] < 0 || xl[t][i] < T ||
            !better_lv(xl[t][i], xv[t][i], lst.l[KB - 1], lst.v[KB - 1]))
          break;
        lst.insert(xl[t][i], xv[t][i]);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    Z = (m0 != kNegInf) ? s0 * expf(m0 - M) : 0.f;
#pragma unroll
    for (int t = 0; t < RMAX; ++t)
      if (xm[t] != kNegInf) Z += xs[t] * expf(xm[t] - M);
  } else {
    // more records per lane: loop, all of a record's fields loaded before its
    // entries are offered (no data-dependent exit between the loads)
    const float T = (n > step) ? kth_bound() : kNegInf;
#pragma unroll 2
    for (int j = lane + step; j < n; j += step) {
      const float* rec = base + j * js;
      M = fmaxf(M, rec[0]);
      float rl[KB];
      int rv[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        rl[i] = i < p.k_max ? rec[2 + i] : kNegInf;
        rv[i] = i < p.k_max ? __float_as_int(rec[2 + p.k_max + i]) : -1;
      }
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        if (rv[i] < 0 || rl[i] < T || !better_lv(rl[i], rv[i], lst.l[KB - 1], lst.v[KB - 1])) break;
        lst.insert(rl[i], rv[i]);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    Z = (m0 != kNegInf) ? s0 * expf(m0 - M) : 0.f;
#pragma unroll 4
    for (int j = lane + step; j < n; j += step) {
      const float* rec = base + j * js;
      const float mj = rec[0];
      const float sj = rec[1];
      if (mj != kNegInf) Z += sj * expf(mj - M);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
  M_out = M;
  Z_out = Z;
  lse = M + logf(Z);
  ol = kNegInf;
  ov = -1;
  for (int i = 0; i < p.k_max; ++i) {
    // the max of the 64-bit key (ordered logit, inverted id) in two 32-bit
    // warp reductions (one REDUX each): the best logit, then the lowest id
    // among the lanes holding it; an empty head has key 0
    const uint32_t hi = lst.v[0] < 0 ? 0u : f2o(lst.l[0]);
    const uint32_t bhi = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t lo = (hi == bhi && lst.v[0] >= 0) ? (uint32_t)(0x7fffffff - lst.v[0]) : 0u;
    const uint32_t blo = __reduce_max_sync(0xffffffffu, lo);
    const unsigned long long best = ((unsigned long long)bhi << 32) | blo;
    const unsigned long long head = lst.v[0] < 0 ? 0ull
                                                 : (((unsigned long long)hi << 32) | (uint32_t)(0x7fffffff - lst.v[0]));
    if (best == 0ull) break;                  // warp-uniform: no more entries
    if (head == best) {                       // unique (token ids are unique in a row)
#pragma unroll
      for (int t = 0; t + 1 < KB; ++t) {
        lst.l[t] = lst.l[t + 1];
        lst.v[t] = lst.v[t + 1];
      }
      lst.l[KB - 1] = kNegInf;
      lst.v[KB - 1] = -1;
    }
    if (lane == i) {                          // the key carries the winner exactly
      ov = 0x7fffffff - (int)(uint32_t)best;
      ol = o2f((uint32_t)(best >> 32));
    }
  }
}

// Row r, one full warp: lse_r = M + log Z over the row's partial records and
// the row's top-k_max (l, v).
template <int KB>
__device__ __forceinline__ void row_topk(const MergeParams& p, int r, int lane, float& lse,
                                         float& M_out, float& Z_out, float& ol, int& ov) {
  const float* base;
  long long js;
  int n;
  row_splits(p, r, base, js, n);
  records_topk<KB>(p, base, js, n, 32, lane, lse, M_out, Z_out, ol, ov);
}

constexpr int MS_WARPS = 8;
constexpr int MS_CAP = 256;   // candidates ranked per batch of rows

// Row r (one full warp): the merged record {M, Z, top-k_max} over the row's
// partial records, written to out_part (ROW mode; the vocab-shard output).
template <int KB>
__device__ __forceinline__ void merged_row_record(const MergeParams& p, int r, int lane) {
  float lse, M, Z, l;
  int v;
  row_topk<KB>(p, r, lane, lse, M, Z, l, v);
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

template <int KB>
__global__ void __launch_bounds__(MS_WARPS * 32) merge_rows_kernel(const MergeParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * MS_WARPS + warp;
  if (r >= p.N) return;
  merged_row_record<KB>(p, r, lane);
}

// Alg. 5 reduce (P:244-251 with k = 1, no normalisation), row r, one full
// warp: the best (l desc, v asc) entry 0 over the row's vocab-split records,
// written to tok[r] / logit[r].
__device__ __forceinline__ void argmax_row(const MergeParams& p, int r, int lane,
                                           long long* __restrict__ tok, float* __restrict__ logit) {
  const float* base;
  long long js;
  int n;
  row_splits(p, r, base, js, n);
  // up to 8 records per lane are loaded before any is reduced (independent
  // loads in flight; the row's records are 128 * stride floats apart)
  unsigned long long best = 0ull;
  for (int j0 = 0; j0 < n; j0 += 8 * 32) {
    float l[8];
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * 32 + lane;
      l[u] = kNegInf;
      v[u] = -1;
      if (j < n) {
        const float* rec = base + j * js;
        l[u] = __ldcg(rec + 2);
        v[u] = __float_as_int(__ldcg(rec + 2 + p.k_max));
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned long long key = lv_key(l[u], v[u]);
      best = key > best ? key : best;
    }
  }
  best = warp_max_u64(best);
  if (lane == 0) {
    tok[r] = best ? (long long)(0x7fffffff - (int)(uint32_t)best) : -1LL;
    logit[r] = best ? o2f((uint32_t)(best >> 32)) : kNegInf;
  }
}

#ifndef AMUN_TC_DEFINE   // (non-template kernel: defined once, in amun.cu's unit)
__global__ void __launch_bounds__(32) argmax_rows_kernel(const MergeParams p,
                                                         long long* __restrict__ tok,
                                                         float* __restrict__ logit) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= p.N) return;
  argmax_row(p, r, lane, tok, logit);
}
#endif

// Sentence phase. CTA = one sentence. Warps take rows; each row's top-k_max
// (already scored cost = prev_cost + l - lse: only the winners are
// normalised) goes to shared memory; the carried best-k plus a batch of
// rows' candidates are ranked by counting better ones (ranks are unique), and
// the best k stay at the front for the next batch.
// `sync` is the barrier of the MS_WARPS warps doing the merge (threads
// 0 .. MS_WARPS*32-1 of the CTA): __syncthreads in the merge kernels, a named
// barrier in the fused kernel's tail (tail.cuh), where other warps exist.
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct MergeWarpsSync {   // named barrier 10 over the MS_WARPS merge warps
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync 10, %0;" ::"n"(MS_WARPS * 32) : "memory");
  }
};

template <int KB, class Sync = CtaSync>
__device__ __forceinline__ void merge_sentence(const MergeParams& p, int s, Cand* pool, Cand* best,
                                               int& s_valid, Sync sync = Sync()) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = p.offsets[s], r1 = p.offsets[s + 1];
  const int ks = p.k_s ? min(p.k_s[s], p.k) : p.k;
  float pc = 0.f;
  if (r0 + warp < r1) pc = p.prev_cost[r0 + warp];
  const int nrows = r1 - r0;
  const int rows_per_batch = max(1, MS_CAP / p.k_max);
  int keep = 0;
  for (int rb = 0; rb < nrows || (rb == 0 && nrows == 0); rb += rows_per_batch) {
    const int re = min(nrows, rb + rows_per_batch);
    for (int rr = rb + warp; rr < re; rr += MS_WARPS) {
      const int r = r0 + rr;
      if (rr != warp) pc = p.prev_cost[r];
      float lse, M, Z, l;
      int v;
      row_topk<KB>(p, r, lane, lse, M, Z, l, v);
      if (lane < p.k_max) {
        Cand c = (v >= 0) ? Cand{pc + (l - lse), l, r, v}
                          : Cand{kNegInf, kNegInf, 0x7fffffff, 0x7fffffff};
        pool[keep + (rr - rb) * p.k_max + lane] = c;
      }
    }
    if (threadIdx.x == 0) s_valid = 0;
    sync();
    const int n = keep + (re - rb) * p.k_max;
    int valid = 0;
    for (int e = threadIdx.x; e < n; e += MS_WARPS * 32) {
      const Cand c = pool[e];
      if (c.v == 0x7fffffff) continue;
      ++valid;
      int rank = 0;
      for (int f = 0; f < n; ++f) rank += better_cand(pool[f], c) ? 1 : 0;
      if (rank < p.k) best[rank] = c;
    }
    if (valid) atomicAdd(&s_valid, valid);
    sync();
    keep = min(s_valid, p.k);
    if (threadIdx.x < keep) pool[threadIdx.x] = best[threadIdx.x];
    sync();
    if (nrows == 0) break;
  }
  if (threadIdx.x < p.k) {
    const int i = threadIdx.x;
    AMUN_DCHECK(s >= 0 && s < p.S && r0 >= 0 && r0 <= r1 && r1 <= p.N);
    const bool ok = i < keep && i < ks;
    p.out_idx[(long long)s * p.k + i] = ok ? (long long)pool[i].r * p.V_total + pool[i].v : -1LL;
    p.out_cost[(long long)s * p.k + i] = ok ? pool[i].cost : kNegInf;
  }
}

// Sentence s with k_max = 1 (greedy, beam 1 / k 1), ONE warp, no shared
// memory or barriers: the sentence's best is the best (better_cand order) of
// its rows' single candidates pc + (l - lse) — exactly what merge_sentence
// selects for k = 1 (the same expression, so the same bits), so warps can
// take sentences independently.
// r0 / r1 / pc0: the sentence's row range and its first row's prev_cost when
// the caller loaded them already (the fused tail does, before its grid-wide
// wait: they are inputs, not other CTAs' results); r0 < 0: load them here.
__device__ __forceinline__ void merge_sentence_k1(const MergeParams& p, int s, int lane, int r0 = -1,
                                                  int r1 = 0, float pc0 = 0.f) {
  if (r0 < 0) {
    r0 = p.offsets[s];
    r1 = p.offsets[s + 1];
    pc0 = r1 > r0 ? p.prev_cost[r0] : 0.f;
  }
  const int ks = p.k_s ? min(p.k_s[s], p.k) : p.k;
  Cand best{kNegInf, kNegInf, 0x7fffffff, 0x7fffffff};
  for (int r = r0; r < r1; ++r) {
    const float pc = r == r0 ? pc0 : p.prev_cost[r];
    float lse, M, Z, l;
    int v;
    row_topk<1>(p, r, lane, lse, M, Z, l, v);   // lane 0 holds the row's best
    if (lane == 0 && v >= 0) {
      const Cand c{pc + (l - lse), l, r, v};
      if (better_cand(c, best)) best = c;
    }
  }
  if (lane == 0 && p.k >= 1) {
    AMUN_DCHECK(s >= 0 && s < p.S && r0 >= 0 && r0 <= r1 && r1 <= p.N);
    const bool ok = best.v != 0x7fffffff && ks >= 1;
    p.out_idx[(long long)s * p.k] = ok ? (long long)best.r * p.V_total + best.v : -1LL;
    p.out_cost[(long long)s * p.k] = ok ? best.cost : kNegInf;
  }
}

template <int KB>
__global__ void __launch_bounds__(MS_WARPS * 32) merge_sentences_kernel(const MergeParams p0) {
  const MergeParams p = merge_dyn(p0);
  if constexpr (KB == 1) {   // a warp per sentence (grid = S / MS_WARPS, launch_merge)
    const int s = blockIdx.x * MS_WARPS + (threadIdx.x >> 5);
    if (s < p.S) merge_sentence_k1(p, s, threadIdx.x & 31);
  } else {
    __shared__ Cand pool[KB + MS_CAP];
    __shared__ Cand best[KB];
    __shared__ int s_valid;
    merge_sentence<KB>(p, blockIdx.x, pool, best, s_valid);
  }
}

}  // namespace amun
