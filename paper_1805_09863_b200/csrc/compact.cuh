// compact.cuh — mini-batching (Alg. 2): after each decode
// step "Remove h from b" for every finished hypothesis, so the next
// step's GEMM only sees live rows. Stable stream compaction (reading G8):
//   j = #alive rows before r;  dst[j] = src[r] for every registered column.
//
// One launch. Every CTA redundantly scans
// the N alive flags with 16-byte loads (N is a few tens of KB at most; each
// thread counts a contiguous run, then a warp-shuffle block scan), so no
// inter-CTA communication is needed. CTA b then
//   * owns output rows [b N'/G, (b+1) N'/G) (so all CTAs stay busy however
//     few rows survive) and gathers them with 16-byte vector copies,
//     CP_UNROLL loads in flight per thread; writes src_row for those rows;
//   * computes new_beam_offsets[s] for s = b*256 + t, ... (a prefix query is
//     the thread-run prefix + a vectorised count inside one run);
//   * (CTA 0 only) counts the sentences with a live row -> counts[1].
// The same kernel advances a beam (amun_beam_advance): the flags are the
// sentences' selected winner slots (offsets s * k), and each surviving slot
// gathers its PARENT row's state (SPEC S:324-331 expand_beam + Alg. 2).
#pragma once
#include <cstdint>

namespace amun {

constexpr int CP_THREADS = 256;
#ifdef CP_ROWS_OVERRIDE
constexpr int CP_ROWS = CP_ROWS_OVERRIDE;
#else
constexpr int CP_ROWS = 8;       // output rows per CTA (tools/compact_bench.py sweep: 4/8/16/32)
#endif
#ifdef CP_UNROLL_OVERRIDE
constexpr int CP_UNROLL = CP_UNROLL_OVERRIDE;
#else
constexpr int CP_UNROLL = 4;     // independent 16-byte loads in flight per thread
#endif
constexpr int CP_MAXCOLS = 16;

struct CompactCol {
  const uint8_t* src;
  uint8_t* dst;
  long long row_bytes;
};

struct CompactParams {
  CompactCol col[CP_MAXCOLS];
  int n_cols, N, S, per;         // per = flags per thread run (multiple of 16)
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

// number of nonzero bytes in [a, b) of the flag array (a % 16 == 0); the
// partial last word is read whole when it lies inside [0, n) and masked
__device__ __forceinline__ int popc_flags(uint4 w) {
  return (__popc(__vcmpne4(w.x, 0u)) + __popc(__vcmpne4(w.y, 0u)) + __popc(__vcmpne4(w.z, 0u)) +
          __popc(__vcmpne4(w.w, 0u))) >> 3;
}
__device__ __forceinline__ int count_alive(const uint8_t* __restrict__ alive, int a, int b, int n) {
  int c = 0;
  if ((reinterpret_cast<uintptr_t>(alive) & 15) != 0) {   // unaligned buffer: bytes only
    for (int r = a; r < b; ++r) c += (alive[r] != 0);
    return c;
  }
  int r = a;
  for (; r + 16 <= b; r += 16) c += popc_flags(*reinterpret_cast<const uint4*>(alive + r));
  if (r < b) {
    if (r + 16 <= n) {
      uint4 w = *reinterpret_cast<const uint4*>(alive + r);
      const int k = b - r;                  // 1..15 valid bytes
      auto keep = [](int bytes) { return bytes >= 4 ? 0xffffffffu : bytes <= 0 ? 0u : (1u << (8 * bytes)) - 1u; };
      w.x &= keep(k);
      w.y &= keep(k - 4);
      w.z &= keep(k - 8);
      w.w &= keep(k - 12);
      c += popc_flags(w);
    } else {
      for (; r < b; ++r) c += (alive[r] != 0);
    }
  }
  return c;
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

// 6 CTAs/SM (40 regs, no spills): 888 resident CTAs cover the cfg4 N = 6400
// grid (800) in one wave; 44 regs gave 5/SM and a second partial wave.
__global__ void __launch_bounds__(CP_THREADS, 6) compact_kernel(const CompactParams p) {
  __shared__ int warp_sums[CP_THREADS / 32];
  __shared__ int map[CP_ROWS];
  __shared__ int gsrc[CP_ROWS];      // gather source row of output row d0 + t
  __shared__ int thr_excl[CP_THREADS];
  const int tid = threadIdx.x;
  const int per = p.per;
  const int a0 = min(tid * per, p.N), a1 = min(a0 + per, p.N);
  const int cnt = count_alive(p.alive, a0, a1, p.N);
  int total;
  const int excl = block_excl_scan(cnt, warp_sums, total);
  thr_excl[tid] = excl;

  // This CTA owns output rows [d0, d1) = [b R, b R + R) with R = ceil(N' / G)
  // <= CP_ROWS (G >= N / CP_ROWS): full blocks of CP_ROWS rows when most rows
  // survive, about one row per CTA when few do (tools/compact_bench.py).
  const int G = gridDim.x, b = blockIdx.x;
  const int R = (total + G - 1) / G;
  const int d0 = min(b * R, total);
  const int d1 = min(d0 + R, total);
  if (excl < d0 + CP_ROWS && excl + cnt > d0) {
    // walk this thread's flags 16 at a time from registers
    int j = excl;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(p.alive) & 15) == 0;
    for (int r = a0; r < a1 && j < d0 + CP_ROWS; r += 16) {
      uint32_t w[4];
      if (vec_ok && r + 16 <= p.N) {
        const uint4 v = *reinterpret_cast<const uint4*>(p.alive + r);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          w[k] = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (r + 4 * k + i < a1) w[k] |= (uint32_t)p.alive[r + 4 * k + i] << (8 * i);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (((w[i >> 2] >> (8 * (i & 3))) & 0xffu) && r + i < a1) {
          if (j >= d0 && j < d0 + CP_ROWS) map[j - d0] = r + i;
          ++j;
        }
      }
    }
  }
  __syncthreads();

  // new beam offsets, spread over all CTAs; CTA 0 alone also counts the
  // sentences still alive (no cross-CTA atomics, so no counts reset needed)
  auto off_at = [&](int s) { return p.off_stride > 0 ? s * p.off_stride : p.offsets[s]; };
  auto prefix = [&](int row) {
    if (row >= p.N) return total;
    const int t0 = row / per;
    return thr_excl[t0] + count_alive(p.alive, t0 * per, row, p.N);
  };
  for (int s = blockIdx.x * CP_THREADS + tid; s <= p.S; s += gridDim.x * CP_THREADS)
    p.new_offsets[s] = prefix(off_at(s));
  if (blockIdx.x == 0) {
    // thread t owns sentences [t q, t q + q); boundaries are evaluated eight
    // at a time so their loads are independent (the count is one CTA's job)
    const int q = (p.S + CP_THREADS - 1) / CP_THREADS;
    const int s_end = min(tid * q + q, p.S);
    int local_alive = 0;
    for (int base = tid * q; base < s_end; base += 8) {
      int v[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) v[i] = (base + i <= s_end) ? prefix(off_at(base + i)) : 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) local_alive += (base + i < s_end) && (v[i + 1] > v[i]);
    }
    int n_alive;
    __syncthreads();   // warp_sums reuse
    block_excl_scan(local_alive, warp_sums, n_alive);
    if (tid == 0) {
      p.counts[0] = total;
      p.counts[1] = n_alive;
    }
  }

  const int nrows = d1 - d0;
  if (nrows <= 0) return;
  if (tid < nrows) {
    const int v = map[tid];
    const int src = p.parent ? p.parent[v] : v;
    gsrc[tid] = src;
    p.src_row[d0 + tid] = src;
    if (p.tok_out) p.tok_out[d0 + tid] = p.vtok[v];
    if (p.cost_out) p.cost_out[d0 + tid] = p.vcost[v];
  }
  __syncthreads();

  // Gather: the CTA's nrows x n4 16-byte units of each column (unit u -> row
  // d0 + u / n4, word u % n4), CP_UNROLL independent loads in flight per
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
