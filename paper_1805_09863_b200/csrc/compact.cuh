// compact.cuh — mini-batching (Alg. 2): after each decode
// step "Remove h from b" for every finished hypothesis, so the next
// step's GEMM only sees live rows. Stable stream compaction (reading G8):
//   j = #alive rows before r;  dst[j] = src[r] for every registered column.
//
// One launch, no memset, no inter-CTA communication. Every CTA redundantly
// counts the N alive flags per 64-flag block (16-byte loads) and scans the
// block counts into a shared-memory prefix table, so a prefix query (alive
// rows before row r) is one table read plus four independent 16-byte loads.
// CTA b then
//   * owns output rows [b N'/G, (b+1) N'/G) (so all CTAs stay busy however
//     few rows survive; G capped at one wave) and gathers them with 16-byte
//     vector copies, CP_UNROLL loads in flight per thread; writes src_row
//     for those rows;
//   * computes new_beam_offsets[s] for s = b*256 + t, ... (prefix queries);
//   * (CTA 0 only) counts the sentences with a live row -> counts[1].
// The same kernel advances a beam (amun_beam_advance): the flags are the
// sentences' selected winner slots (offsets s * k), and each surviving slot
// gathers its PARENT row's state (SPEC S:324-331 expand_beam + Alg. 2).
#pragma once
#include <cstdint>

#include "ptx.cuh"   // AMUN_DCHECK


namespace amun {

constexpr int CP_THREADS = 256;
#ifdef CP_ROWS_OVERRIDE
constexpr int CP_ROWS = CP_ROWS_OVERRIDE;
#else
constexpr int CP_ROWS = 8;       // output rows per CTA below one wave (compact_bench sweep: 4/8/16/32)
#endif
#ifdef CP_UNROLL_OVERRIDE
constexpr int CP_UNROLL = CP_UNROLL_OVERRIDE;
#else
constexpr int CP_UNROLL = 4;     // independent 16-byte loads in flight per thread
#endif
constexpr int CP_MAXCOLS = 16;
constexpr int CP_MAXR = 128;     // output rows one CTA may own (grid capped at one wave)
constexpr int CP_CTAS_PER_SM = 6;
constexpr int CP_MAXBLK = 4096;  // prefix blocks held in shared memory
constexpr int CP_SFLAGS = 16384; // flags cached in shared memory up to this N (6 CTAs / SM)
constexpr int CP_CNTPRE = 4097;  // CTA 0's sentence offsets in shared memory up to S + 1 = this

struct CompactCol {
  const uint8_t* src;
  uint8_t* dst;
  long long row_bytes;
};

struct CompactParams {
  CompactCol col[CP_MAXCOLS];
  int n_cols, N, S, blk_log2;    // 2^blk_log2 = flags per prefix block (>= 64, <= CP_MAXBLK blocks)
  int flags_in_smem;             // N <= CP_SFLAGS: the flags are cached in shared memory
  int dyn_off_at;                // byte offset of CTA 0's sentence offsets in dynamic smem
  int cnt_pre;                   // CTA 0's sentence offsets are prefetched into shared memory
  const uint8_t* __restrict__ alive;
  const int* __restrict__ offsets;   // [S+1]; unused when off_stride > 0
  int off_stride;                    // > 0: offsets[s] = s * off_stride (beam advance)
  int* __restrict__ new_offsets;
  int* __restrict__ src_row;
  int* __restrict__ counts;      // {N', S_alive}, written by CTA 0
  // beam advance (amun_beam_advance): flag i is winner slot i of a sentence;
  // the state columns are gathered from parent[i], and the winner's token
  // and cost are written too. All NULL for plain compaction.
  const int* __restrict__ parent;
  const int* __restrict__ vtok;
  const float* __restrict__ vcost;
  int* __restrict__ tok_out;
  float* __restrict__ cost_out;
  int exp;                           // experiments (env AMUN_CP_EXP): 1 no sentence count,
                                     // 2 + no new offsets, 3 scan only, 9 CTA 0 phase times
};

// Beam advance, step 1: classify every selected winner i (one thread each):
// live = valid and not EOS, parent row r and token v of idx = r * V_total + v.
__global__ void beam_classify_kernel(const long long* __restrict__ idx, int n, long long V_total,
                                     int eos, uint8_t* __restrict__ live, int* __restrict__ parent,
                                     int* __restrict__ tok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long e = idx[i];
  int r = 0, v = -1;
  if (e >= 0) {
    r = (int)(e / V_total);
    v = (int)(e - (long long)r * V_total);
  }
  live[i] = (e >= 0 && v != eos) ? 1 : 0;
  parent[i] = r;
  tok[i] = v;
}

__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < CP_THREADS / 32) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < CP_THREADS / 32) warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  total = warp_sums[CP_THREADS / 32 - 1];
  const int before = warp ? warp_sums[warp - 1] : 0;
  return before + x - v;
}

// 0x80 in every nonzero byte of x, 0 elsewhere (3 integer ops; __vcmpne4 is
// emulated and cost ~20x more in the prefix queries).
__device__ __forceinline__ uint32_t nz_bytes(uint32_t x) {
  return (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
}
// Nonzero-byte mask of 16 flags (one uint4): bit i = flag i != 0.
__device__ __forceinline__ uint32_t flag_mask16(uint4 w) {
  const uint32_t v[4] = {nz_bytes(w.x) >> 7, nz_bytes(w.y) >> 7, nz_bytes(w.z) >> 7,
                         nz_bytes(w.w) >> 7};   // bits 0, 8, 16, 24
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    m |= ((v[k] | (v[k] >> 7) | (v[k] >> 14) | (v[k] >> 21)) & 0xFu) << (4 * k);
  return m;
}
// Number of nonzero flags among 16.
__device__ __forceinline__ int flag_count16(uint4 w) {
  return __popc(nz_bytes(w.x)) + __popc(nz_bytes(w.y)) + __popc(nz_bytes(w.z)) +
         __popc(nz_bytes(w.w));
}

// The flags as the kernel reads them: a shared-memory copy (N <= CP_SFLAGS,
// zero-padded to 64-flag blocks) or the global array.
struct Flags {
  const uint8_t* __restrict__ g;   // global, n bytes
  const uint8_t* s;                // shared copy or NULL
  int n;
  // bit mask of the nonzero flags in [lo, hi), lo % 64 == 0, hi - lo <= 64
  __device__ __forceinline__ unsigned long long mask64(int lo, int hi) const {
    unsigned long long m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int base = lo + 16 * k;
      if (base >= hi) break;
      uint32_t mk;
      if (s) {
        mk = flag_mask16(*reinterpret_cast<const uint4*>(s + base));
      } else if ((reinterpret_cast<uintptr_t>(g) & 15) == 0 && base + 16 <= n) {
        mk = flag_mask16(__ldg(reinterpret_cast<const uint4*>(g + base)));
      } else {
        mk = 0;
        for (int i = 0; i < 16 && base + i < n; ++i) mk |= (__ldg(g + base + i) != 0 ? 1u : 0u) << i;
      }
      const int valid = hi - base;   // >= 1
      if (valid < 16) mk &= (1u << valid) - 1u;
      m |= (unsigned long long)mk << (16 * k);
    }
    return m;
  }
  // alive flags in [lo, hi), lo a multiple of 64
  __device__ __forceinline__ int count(int lo, int hi) const {
    int c = 0;
    for (int a = lo; a < hi; a += 64) c += __popcll(mask64(a, min(hi, a + 64)));
    return c;
  }
};

// Every CTA: per-block alive counts of the N flags (blocks of 2^blk_log2
// flags, <= CP_MAXBLK blocks, strided over the threads: coalesced 16-byte
// loads; for N <= CP_SFLAGS the flags are kept in shared memory), then the
// blocks' exclusive prefix in shared memory. prefix(row) = #alive rows before
// `row` is a table read plus a popcount of at most one block — shared memory
// only for N <= CP_SFLAGS, so the sentence boundaries and the gather's
// source rows cost no global round trips after the scan.
// 6 CTAs/SM: the grid is capped at one wave (CP_CTAS_PER_SM x #SMs, the
// host's launch_compact), so the redundant scans cost O(N x min(N / 8, one
// wave)) bytes of L2 reads, not O(N^2 / 8), and no launch has a second wave.
__global__ void __launch_bounds__(CP_THREADS, CP_CTAS_PER_SM) compact_kernel(const CompactParams p) {
  __shared__ int warp_sums[CP_THREADS / 32];
  __shared__ int map[CP_MAXR];
  __shared__ int gsrc[CP_MAXR];      // gather source row of output row d0 + t
  __shared__ int s_b0;
  extern __shared__ __align__(16) uint8_t cp_dyn[];   // cntb[nblk + 1] ints, then the flags
  const int tid = threadIdx.x;
  const int N = p.N, blk = 1 << p.blk_log2;
  const int nblk = (N + blk - 1) / blk;
  int* cntb = reinterpret_cast<int*>(cp_dyn);
  uint8_t* sfl = p.flags_in_smem ? cp_dyn + ((nblk + 1) * 4 + 15) / 16 * 16 : nullptr;
  const Flags fl{p.alive, sfl, N};
  // CTA 0: the sentence boundaries of its alive count, copied in while the
  // flags are scanned (cp.async: no registers held, one round trip)
  int* s_off = (blockIdx.x == 0 && p.off_stride == 0 && p.S + 1 <= CP_CNTPRE && p.cnt_pre)
                   ? reinterpret_cast<int*>(cp_dyn + p.dyn_off_at) : nullptr;
  if (s_off) {
    for (int i = tid; i <= p.S; i += CP_THREADS)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(s_off + i)),
                   "l"(p.offsets + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // (experiment 9: CTA 0's phase times in ns into src_row[1..7]; N' must be 0)
  unsigned long long dbg_t0 = 0;
  auto dbg = [&](int i) {
    if (p.exp >= 9 && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (i == 0) dbg_t0 = t; else p.src_row[i] = (int)(t - dbg_t0);
    }
  };
  dbg(0);
  auto off_at = [&](int s) { return p.off_stride > 0 ? s * p.off_stride : __ldg(p.offsets + s); };
  // this thread's new_offsets boundary, requested before the scan
  const int s_mine = blockIdx.x * CP_THREADS + tid;
  const int off_mine = (s_mine <= p.S) ? off_at(s_mine) : 0;

  // 1. per-block counts (and the shared-memory copy of the flags)
  for (int i = tid; i < nblk; i += CP_THREADS) {
    if (sfl) {   // blk = 64: copy the block, zero-padded past N
      const int lo = i * 64;
      uint4 w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int base = lo + 16 * k;
        if ((reinterpret_cast<uintptr_t>(p.alive) & 15) == 0 && base + 16 <= N) {
          w[k] = __ldg(reinterpret_cast<const uint4*>(p.alive + base));
        } else {   // the array's tail (or an unaligned array): bytes, zero past N
          uint32_t x0 = 0u, x1 = 0u, x2 = 0u, x3 = 0u;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t byte = base + j < N ? (uint32_t)__ldg(p.alive + base + j) : 0u;
            const uint32_t sh = byte << (8 * (j & 3));
            if (j < 4) x0 |= sh; else if (j < 8) x1 |= sh; else if (j < 12) x2 |= sh; else x3 |= sh;
          }
          w[k] = make_uint4(x0, x1, x2, x3);
        }
      }
      int c = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        *reinterpret_cast<uint4*>(sfl + lo + 16 * k) = w[k];
        c += flag_count16(w[k]);
      }
      cntb[i] = c;
    } else {
      cntb[i] = fl.count(i * blk, min(i * blk + blk, N));
    }
  }
  if (s_off) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // 2. exclusive prefix over the blocks (thread t: a contiguous run of them)
  const int per = (nblk + CP_THREADS - 1) / CP_THREADS;
  const int c0 = min(tid * per, nblk), c1 = min(c0 + per, nblk);
  int run = 0;
  for (int i = c0; i < c1; ++i) run += cntb[i];
  int total;
  int excl = block_excl_scan(run, warp_sums, total);
  for (int i = c0; i < c1; ++i) {
    const int v = cntb[i];
    cntb[i] = excl;
    excl += v;
  }
  if (tid == 0) cntb[nblk] = total;
  AMUN_DCHECK(nblk <= CP_MAXBLK && total >= 0 && total <= N);
  __syncthreads();
  dbg(1);
  if (p.exp >= 3 && p.exp < 9) {
    if (blockIdx.x == 0 && tid == 0) p.counts[0] = total;
    return;
  }
  auto prefix = [&](int row) {       // alive rows before `row`
    if (row >= N) return total;
    const int i = row >> p.blk_log2;
    return cntb[i] + fl.count(i << p.blk_log2, row);
  };

  // 3. This CTA owns output rows [d0, d1) = [b R, b R + R), R = ceil(N' / G)
  // <= CP_MAXR: blocks of up to 8 rows while N fits one wave, more per CTA
  // for larger N, about one row per CTA when few survive. Their source rows:
  // from the prefix block holding rank d0 on, one block per thread and round.
  // (CTA 0 owns none when G > 1: it counts the sentences, step 4)
  const int G = gridDim.x > 1 ? gridDim.x - 1 : 1, b = gridDim.x > 1 ? blockIdx.x - 1 : 0;
  const int R = (total + G - 1) / G;
  const int d0 = b < 0 ? total : min(b * R, total);
  const int d1 = min(d0 + R, total);
  const int nrows = d1 - d0;
  if (nrows > 0) {
    if (tid == 0) {   // last block i with cntb[i] <= d0 (it holds rank d0)
      int lo = 0, hi = nblk - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cntb[mid] <= d0) lo = mid; else hi = mid - 1;
      }
      s_b0 = lo;
    }
    __syncthreads();
    for (int i = s_b0 + tid; i < nblk && cntb[i] < d1; i += CP_THREADS) {
      int j = cntb[i];
      for (int a = i * blk; a < min(i * blk + blk, N) && j < d1; a += 64) {
        unsigned long long m = fl.mask64(a, min(a + 64, N));
        const int c = __popcll(m);
        if (j + c <= d0) {   // none of these ranks is ours
          j += c;
          continue;
        }
        while (m && j < d1) {
          const int r = a + __ffsll((long long)m) - 1;
          m &= m - 1;
          if (j >= d0) map[j - d0] = r;
          ++j;
        }
      }
    }
  }
  __syncthreads();
  dbg(2);

  // 4. new beam offsets, spread over all CTAs (one prefix query per thread);
  // CTA 0 — which owns no output rows, so this does not delay a gather —
  // counts the sentences still alive: sentence s is alive iff
  // prefix(offsets[s+1]) > prefix(offsets[s]). Its offsets were copied into
  // shared memory by cp.async during the scan (S + 1 <= CP_CNTPRE), so the
  // count is shared-memory reads only for N <= CP_SFLAGS. No cross-CTA
  // atomics, so nothing needs zeroing.
  if (p.exp < 2 || p.exp >= 9) {
    if (s_mine <= p.S) p.new_offsets[s_mine] = prefix(off_mine);
    for (int s = s_mine + gridDim.x * CP_THREADS; s <= p.S; s += gridDim.x * CP_THREADS)
      p.new_offsets[s] = prefix(off_at(s));
  }
  dbg(3);
  if (blockIdx.x == 0 && (p.exp < 1 || p.exp >= 9)) {
    int local_alive = 0;
    if (s_off && sfl) {
      // shared memory only, and no prefix queries: sentence s is alive iff
      // some flag in [offsets[s], offsets[s+1]) is nonzero (a beam spans one
      // or two 16-byte words)
      const uint32_t fbase = (uint32_t)__cvta_generic_to_shared(sfl);
#pragma unroll 1
      for (int s = tid; s < p.S; s += CP_THREADS) {
        const int lo = s_off[s], hi = min(s_off[s + 1], N);
        uint32_t any = 0;
        for (int w = lo & ~15; w < hi; w += 16) {
          uint4 q;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(fbase + (uint32_t)w));
          const uint32_t x[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {   // bytes of word j inside [lo, hi)
            const int b0 = w + 4 * j;
            const int from = max(lo - b0, 0), to = min(hi - b0, 4);
            const uint32_t keep = from >= to ? 0u
                                : ((to >= 4 ? 0xFFFFFFFFu : (1u << (8 * to)) - 1u) &
                                   ~((1u << (8 * from)) - 1u));
            any |= nz_bytes(x[j]) & keep;
          }
        }
        local_alive += any ? 1 : 0;
      }
    } else {
      auto off_c = [&](int s) { return s_off ? s_off[s] : off_at(s); };
      for (int s = tid; s < p.S; s += CP_THREADS)
        local_alive += prefix(off_c(s + 1)) > prefix(off_c(s)) ? 1 : 0;
    }
    dbg(4);
    int n_alive;
    block_excl_scan(local_alive, warp_sums, n_alive);
    if (tid == 0) {
      p.counts[0] = total;
      p.counts[1] = n_alive;
    }
    dbg(5);
  }

  if (nrows <= 0) return;
  if (tid < nrows) {
    const int v = map[tid];
    AMUN_DCHECK(nrows <= CP_MAXR && v >= 0 && v < N && d0 + tid < total && total <= N);
    const int src = p.parent ? p.parent[v] : v;
    gsrc[tid] = src;
    p.src_row[d0 + tid] = src;
    if (p.tok_out) p.tok_out[d0 + tid] = p.vtok[v];
    if (p.cost_out) p.cost_out[d0 + tid] = p.vcost[v];
  }
  __syncthreads();

  // 5. Gather: the CTA's nrows x n4 16-byte units of each column (unit u ->
  // row d0 + u / n4, word u % n4), CP_UNROLL independent loads in flight per
  // thread before the stores.
  for (int c = 0; c < p.n_cols; ++c) {
    const CompactCol col = p.col[c];
    const bool vec = ((col.row_bytes & 15) == 0) &&
                     (((reinterpret_cast<uintptr_t>(col.src) |
                        reinterpret_cast<uintptr_t>(col.dst)) & 15) == 0);
    if (vec) {
      const int n4 = (int)(col.row_bytes >> 4);
      const long long base = (long long)d0 * n4;
      const int lo = 0, hi = nrows * n4;
      const int4* src = reinterpret_cast<const int4*>(col.src);
      int4* dst = reinterpret_cast<int4*>(col.dst) + base;
      for (int u = lo + tid; u < hi; u += CP_UNROLL * CP_THREADS) {
        int4 t[CP_UNROLL];
#pragma unroll
        for (int q = 0; q < CP_UNROLL; ++q) {
          const int uu = u + q * CP_THREADS;
          if (uu < hi) {
            const int j = uu / n4;
            t[q] = __ldg(src + (long long)gsrc[j] * n4 + (uu - j * n4));
          }
        }
#pragma unroll
        for (int q = 0; q < CP_UNROLL; ++q)
          if (u + q * CP_THREADS < hi) dst[u + q * CP_THREADS] = t[q];
      }
    } else {
      const int n1 = (int)(col.row_bytes >> 2);
      const long long base = (long long)d0 * n1;
      const int lo = 0, hi = nrows * n1;
      const int* src = reinterpret_cast<const int*>(col.src);
      int* dst = reinterpret_cast<int*>(col.dst) + base;
      for (int u = lo + tid; u < hi; u += CP_THREADS) {
        const int j = u / n1;
        dst[u] = __ldg(src + (long long)gsrc[j] * n1 + (u - j * n1));
      }
    }
  }
}

// Sentence-level state (encoder context, source lengths: one entry per
// sentence, not per hypothesis) follows its sentence: a sentence stays while
// at least one of its rows survived the row compaction (P:61-65 removes
// hypotheses; a sentence without hypotheses is finished). alive_s[s] =
// new_offsets[s+1] > new_offsets[s]; unit_offsets = 0..S (one "row" per
// sentence) so amun_compact gathers the sentence columns.
__global__ void sentence_alive_kernel(const int* __restrict__ new_offsets, int S,
                                      unsigned char* __restrict__ alive_s,
                                      int* __restrict__ unit_offsets) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= S; s += gridDim.x * blockDim.x) {
    unit_offsets[s] = s;
    if (s < S) alive_s[s] = new_offsets[s + 1] > new_offsets[s] ? 1 : 0;
  }
}

}  // namespace amun
