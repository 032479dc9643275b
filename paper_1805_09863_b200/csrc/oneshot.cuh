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
// Buffer layout, counters and the signal / wait protocol: peer.cuh (shared
// with the fused kernel's tail, the real multi-GPU path).
//
// Deadlock freedom: a CTA only waits after its own stores and signals; all
// CTAs of the grid are co-resident (cooperative launch), so every rank's
// signals are eventually sent. One-GPU emulation of G ranks (the only
// multi-rank execution possible on one GPU, B200_PROFILING.md "kernels that
// wait on one another"): gridDim.y = G, me = blockIdx.y, all buffers local,
// one cooperative launch.
#pragma once
#include "tail.cuh"   // (merge.cuh, peer.cuh)

namespace amun {

struct OneShotParams {
  MergeParams src[OS_MAX_G];     // row phase: rank's fused-kernel slots (layout 0 / 2)
  MergeParams dst;               // sentence phase template (layout 1, G, N, S, ...)
  char* buf[OS_MAX_G];           // every rank's one-shot buffer as mapped here
  long long* out_idx[OS_MAX_G];  // per emulated rank (real mode: [0])
  float* out_cost[OS_MAX_G];
  int G, rank, emulate, nb;      // nb: CTAs per rank in this call
  long long recv_elems;          // floats per parity half: G * max_rows * stride
};

template <int KB>
__global__ void __launch_bounds__(MS_WARPS * 32) oneshot_kernel(const OneShotParams q) {
  __shared__ Cand pool[KB + MS_CAP];
  __shared__ Cand best[KB];
  __shared__ int s_valid;
  __shared__ unsigned int s_epoch;
  const int me = q.emulate ? (int)blockIdx.y : q.rank;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_fail;
  // the epoch word is written only by this rank's previous launch
  if (threadIdx.x == 0) {
    s_epoch = os_epoch(q.buf[me]);
    s_fail = 0;
  }
  __syncthreads();
  const unsigned int epoch = s_epoch;
  const MergeParams& sp = q.src[q.emulate ? me : 0];
  const int N = q.dst.N, stride = q.dst.stride, k_max = q.dst.k_max;

  // 1. row phase: one warp per row; consecutive rows go to different CTAs
  //    (at small N every row gets its own SM's load bandwidth)
  for (int r = b + warp * q.nb; r < N; r += q.nb * MS_WARPS) {
    float lse, M, Z, l;
    int v;
    row_topk<KB>(sp, r, lane, lse, M, Z, l, v);
    os_store_record(q.buf, q.G, os_record_off(epoch, q.recv_elems, me, N, r, stride), k_max, lane,
                    M, Z, l, v);
  }
  // 2. signal (the rank's last CTA, once per peer), 3. wait (bounded)
  __syncthreads();
  if (threadIdx.x == 0) os_signal(q.buf, q.G, me, q.nb, epoch);
  if (!os_wait(q.buf[me], q.G, epoch)) s_fail = 1;
  __syncthreads();
  if (s_fail) return;
  // 4. sentence phase over [G][N][stride] in this rank's receive half
  MergeParams dp = q.dst;
  dp.part = reinterpret_cast<const float*>(q.buf[me] + OS_CTRL_BYTES) +
            (long long)(epoch & 1u) * q.recv_elems;
  dp.part_floats = q.recv_elems;
  dp.out_idx = q.out_idx[q.emulate ? me : 0];
  dp.out_cost = q.out_cost[q.emulate ? me : 0];
  for (int s = b; s < dp.S; s += q.nb) {
    merge_sentence<KB>(dp, s, pool, best, s_valid);
    __syncthreads();
  }
}

}  // namespace amun
