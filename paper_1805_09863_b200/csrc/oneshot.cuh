// oneshot.cuh — NVLink one-shot exchange + merge.
//
// The vocab-sharded output layer (Alg. 6: each GPU holds a vocab
// shard, computes its (max, sum, k-best) partial state, and the states are
// reduced exactly) without a collective library call. After this rank's fused
// kernel, ONE kernel:
//   1. row phase: combines this rank's per-CTA partial records into one
//      record per row (the monoid combine of merge.cuh) and stores it
//      directly into slot [me] of EVERY rank's receive buffer (peer memory
//      mapped through CUDA IPC: NVLink stores);
//   2. signals: the rank's last CTA to finish step 1 adds 1 to counter [me]
//      in every rank's control block (red.release.sys) and advances the
//      rank's epoch;
//   3. waits until every source rank's counter reaches epoch + 1
//      (ld.acquire.sys), then
//   4. sentence phase: the per-sentence top-k_s over the G records per row
//      (merge.cuh merge_sentence, layout 1), written by every rank.
//
// Buffer of one rank (one cudaMalloc, exported by IPC handle):
//   control: u32 cnt[8] (calls signalled per source rank, monotonic),
//            u32 epoch (calls of this rank), u32 done (CTAs of the current
//            call past step 1), padded to OS_CTRL_BYTES;
//   recv:    fp32 [2][G][max_rows][stride], double-buffered by epoch parity.
// Counters only grow, so no reset is needed between calls (CUDA-graph
// replays included). Parity double-buffering is sufficient: a peer can be
// at most one call ahead (its call e+1 waits for this rank's call e+1
// signals, which are sent after this rank's call e has finished reading).
//
// Deadlock freedom: a CTA only waits after its own stores and signals; all
// CTAs of the grid are co-resident (cooperative launch), so every rank's
// signals are eventually sent. One-GPU emulation of G ranks (the only
// multi-rank execution possible on one GPU, B200_PROFILING.md "kernels that
// wait on one another"): gridDim.y = G, me = blockIdx.y, all buffers local,
// one cooperative launch.
#pragma once
#include "tail.cuh"   // (atomics / acquire-release helpers)

namespace amun {

constexpr int OS_MAX_G = 8;
constexpr int OS_CTRL_BYTES = 256;

struct OneShotParams {
  MergeParams src[OS_MAX_G];     // row phase: rank's fused-kernel slots (layout 0 / 2)
  MergeParams dst;               // sentence phase template (layout 1, G, N, S, ...)
  char* buf[OS_MAX_G];           // every rank's one-shot buffer as mapped here
  long long* out_idx[OS_MAX_G];  // per emulated rank (real mode: [0])
  float* out_cost[OS_MAX_G];
  int G, rank, emulate, nb;      // nb: CTAs per rank in this call
  long long recv_elems;          // floats per parity half: G * max_rows * stride
};

__device__ __forceinline__ void red_release_sys_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}


template <int KB>
__global__ void __launch_bounds__(MS_WARPS * 32) oneshot_kernel(const OneShotParams q) {
  __shared__ Cand pool[KB + MS_CAP];
  __shared__ Cand best[KB];
  __shared__ int s_valid;
  __shared__ unsigned int s_epoch;
  const int me = q.emulate ? (int)blockIdx.y : q.rank;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned int* ctrl = reinterpret_cast<unsigned int*>(q.buf[me]);
  // the epoch word is written only by this rank's previous launch (stream
  // order makes it visible): a plain volatile load
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned int*>(ctrl + OS_MAX_G);
  __syncthreads();
  const unsigned int epoch = s_epoch;
  const long long half = (long long)(epoch & 1u) * q.recv_elems;
  const MergeParams& sp = q.src[q.emulate ? me : 0];
  const int N = q.dst.N, stride = q.dst.stride, k_max = q.dst.k_max;

  // 1. row phase: one warp per row; consecutive rows go to different CTAs
  //    (at small N every row gets its own SM's load bandwidth)
  for (int r = b + warp * q.nb; r < N; r += q.nb * MS_WARPS) {
    float lse, M, Z, l;
    int v;
    row_topk<KB>(sp, r, lane, lse, M, Z, l, v);
    const long long off = half + ((long long)me * N + r) * stride;
    for (int p = 0; p < q.G; ++p) {
      float* rec = reinterpret_cast<float*>(q.buf[p] + OS_CTRL_BYTES) + off;
      if (lane == 0) *reinterpret_cast<float2*>(rec) = make_float2(M, Z);
      if (lane < k_max) {
        rec[2 + lane] = l;
        rec[2 + k_max + lane] = __int_as_float(v);
      }
    }
  }
  // 2. signal: the last of this rank's CTAs to finish its rows advances the
  //    epoch and signals every rank ONCE (one system-scope release per peer
  //    per call). Ordering chain: each CTA's stores -> barrier -> its thread
  //    0's acq_rel RMW on `done` (gpu scope, a release sequence) -> the last
  //    CTA's RMW -> its red.release.sys -> the peer's ld.acquire.sys.
  //    (A __threadfence_system() per CTA measured ~3 us per launch.)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atom_add_acq_rel_gpu(ctrl + OS_MAX_G + 1, 1u) == (unsigned int)q.nb - 1u) {
      ctrl[OS_MAX_G + 1] = 0u;        // next launch (stream order) starts from 0
      ctrl[OS_MAX_G] = epoch + 1u;
      for (int p = 0; p < q.G; ++p)
        red_release_sys_add(reinterpret_cast<unsigned int*>(q.buf[p]) + me, 1u);
    }
  }
  // 3. wait (acquire) until every source rank has signalled this call
  if (threadIdx.x < q.G) {
    const unsigned int* c = ctrl + threadIdx.x;
    while ((int)(ld_acquire_sys(c) - (epoch + 1u)) < 0) __nanosleep(32);
  }
  __syncthreads();
  // 4. sentence phase over [G][N][stride] in this rank's receive half
  MergeParams dp = q.dst;
  dp.part = reinterpret_cast<const float*>(q.buf[me] + OS_CTRL_BYTES) + half;
  dp.out_idx = q.out_idx[q.emulate ? me : 0];
  dp.out_cost = q.out_cost[q.emulate ? me : 0];
  for (int s = b; s < dp.S; s += q.nb) {
    merge_sentence<KB>(dp, s, pool, best, s_valid);
    __syncthreads();
  }
}

}  // namespace amun
