// compact.cuh — mini-batching (Alg. 2): after each decode
// step "Remove h from b" for every finished hypothesis, so the next
// step's GEMM only sees live rows. Stable stream compaction (reading G8):
//   j = #alive rows before r;  dst[j] = src[r] for every registered column.
//
// One launch. Every CTA redundantly scans the N alive flags (N is at most a
// few tens of thousands of bytes; each thread sums a contiguous run, then a
// warp-shuffle block scan) so no inter-CTA communication is needed; CTA b
// then owns output rows [b*R, b*R + R) and gathers them with 16-byte vector
// copies, one warp per row. CTA 0 also writes new_beam_offsets and counts.
#pragma once
#include <cstdint>

namespace amun {

constexpr int CP_THREADS = 256;
constexpr int CP_ROWS = 32;      // output rows per CTA
constexpr int CP_MAXCOLS = 16;

struct CompactCol {
  const uint8_t* src;
  uint8_t* dst;
  long long row_bytes;
};

struct CompactParams {
  CompactCol col[CP_MAXCOLS];
  int n_cols, N, S;
  const uint8_t* __restrict__ alive;
  const int* __restrict__ offsets;
  int* __restrict__ new_offsets;
  int* __restrict__ src_row;
  int* __restrict__ counts;
};

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

__global__ void __launch_bounds__(CP_THREADS) compact_kernel(const CompactParams p) {
  __shared__ int warp_sums[CP_THREADS / 32];
  __shared__ int map[CP_ROWS];
  __shared__ int s_alive_cnt;
  __shared__ int thr_excl[CP_THREADS];
  const int tid = threadIdx.x;
  const int per = (p.N + CP_THREADS - 1) / CP_THREADS;
  const int a0 = min(tid * per, p.N), a1 = min(a0 + per, p.N);
  int cnt = 0;
  for (int r = a0; r < a1; ++r) cnt += (p.alive[r] != 0);
  int total;
  const int excl = block_excl_scan(cnt, warp_sums, total);
  thr_excl[tid] = excl;

  const int d0 = blockIdx.x * CP_ROWS;
  // which source rows land in [d0, d0 + CP_ROWS)
  if (excl < d0 + CP_ROWS && excl + cnt > d0) {
    int j = excl;
    for (int r = a0; r < a1; ++r) {
      if (p.alive[r]) {
        if (j >= d0 && j < d0 + CP_ROWS) map[j - d0] = r;
        ++j;
      }
    }
  }

  if (blockIdx.x == 0) {
    if (tid == 0) s_alive_cnt = 0;
    __syncthreads();
    int local_alive = 0;
    for (int s = tid; s <= p.S; s += CP_THREADS) {
      // number of alive rows before o_s: thread t0 = owner of row o_s
      const int o = p.offsets[s];
      auto prefix = [&](int row) {
        if (row >= p.N) return total;
        const int t0 = row / per;   // per >= 1 here since row < N
        int c = thr_excl[t0];
        for (int rr = t0 * per; rr < row; ++rr) c += (p.alive[rr] != 0);
        return c;
      };
      const int no = prefix(o);
      p.new_offsets[s] = no;
      if (s < p.S) local_alive += (prefix(p.offsets[s + 1]) > no);
    }
    if (local_alive) atomicAdd(&s_alive_cnt, local_alive);
    __syncthreads();
    if (tid == 0) {
      p.counts[0] = total;
      p.counts[1] = s_alive_cnt;
    }
  }
  __syncthreads();

  const int nrows = min(CP_ROWS, total - d0);
  if (nrows <= 0) return;
  if (tid < nrows) p.src_row[d0 + tid] = map[tid];

  const int warp = tid >> 5, lane = tid & 31;
  for (int i = warp; i < nrows; i += CP_THREADS / 32) {
    const long long r = map[i];
    const long long d = d0 + i;
    for (int c = 0; c < p.n_cols; ++c) {
      const CompactCol col = p.col[c];
      const uint8_t* src = col.src + r * col.row_bytes;
      uint8_t* dst = col.dst + d * col.row_bytes;
      const bool vec = ((col.row_bytes & 15) == 0) &&
                       (((reinterpret_cast<uintptr_t>(col.src) | reinterpret_cast<uintptr_t>(col.dst)) & 15) == 0);
      if (vec) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        const int n4 = (int)(col.row_bytes >> 4);
        int e = lane;
        for (; e + 96 < n4; e += 128) {
          const int4 t0 = __ldg(s4 + e), t1 = __ldg(s4 + e + 32), t2 = __ldg(s4 + e + 64),
                     t3 = __ldg(s4 + e + 96);
          d4[e] = t0;
          d4[e + 32] = t1;
          d4[e + 64] = t2;
          d4[e + 96] = t3;
        }
        for (; e < n4; e += 32) d4[e] = __ldg(s4 + e);
      } else {
        const int* s1 = reinterpret_cast<const int*>(src);
        int* d1 = reinterpret_cast<int*>(dst);
        const int n1 = (int)(col.row_bytes >> 2);
        for (int e = lane; e < n1; e += 32) d1[e] = __ldg(s1 + e);
      }
    }
  }
}

}  // namespace amun
