// tail.cuh — the fused kernels' grid-wide tail: the merge (a6) inside the
// same launch as steps 1-4.
//
// Tail. Every CTA's partial records {m, s, top-k} (Alg. 6's per-shard state,
// P:232-242) must be complete before any row can be merged (the reduce step
// of Alg. 6, generalised to (max, sum, k-best) states). Instead of
// a second kernel, each CTA, after its epilogue, arrives on this launch's
// counter (one acq_rel atomic); the last arrival proceeds at once, the others
// poll the counter (one thread, acquire loads with backoff). Then the
// MS_WARPS epilogue warps of every CTA run the merge on a share of the work:
//   TAIL_SENT   sentences s = cta, cta + grid, ...: the per-sentence top-k_s
//               of prev_cost + l - lse (merge.cuh merge_sentence);
//   TAIL_ROWS   rows: one merged record per row (vocab-shard output);
//   TAIL_ARGMAX rows: Alg. 5's argmax over the row's records;
//   TAIL_ONESHOT the vocab-sharded exchange (peer.cuh):
//               rows as TAIL_ROWS, each merged record stored into slot
//               [rank] of every rank's receive buffer (NVLink stores), one
//               system-scope signal per peer from the rank's last CTA, a
//               bounded wait for every rank's signal, then sentences as
//               TAIL_SENT over the G records of each row.
// Waiting on other CTAs is safe because the launch is cooperative (every CTA
// of the <= #SM grid co-resident, launch_tc.cuh launch_kernel); a count that
// overshoots or a wait longer than 10 s traps (loud failure, never a silent
// hang).
//
// Counters. Launch tag t (= 1 + the generation word every CTA reads at its
// start; also the hint tag, tc_epi.cuh) counts arrivals in arrive[t & 1].
// CTA 0 of launch t zeroes arrive[(t + 1) & 1] at its start: the counter of
// the NEXT launch, last used by launch t - 1, which has completed (stream
// order). Every generation-advancing launch (tail or not) does so, so no
// per-call reset is needed — CUDA-graph replays and a changing grid size
// included. The last arrival advances the generation to t.
#pragma once
#include "tc_epi.cuh"

namespace amun {

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned int atom_add_acq_rel_gpu(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Called by every thread of the CTA after the kernel's final barrier (all
// partial records of this CTA are written). Threads >= MS_WARPS*32 (the
// control warps) return at once.
template <int KB>
__device__ __forceinline__ void grid_tail(const TcParams& p, const TcDyn& dyn, uint8_t* scratch,
                                          uint32_t tag) {
  const int tid = threadIdx.x;
  if (tid >= MS_WARPS * 32) return;
  // k_max = 1 sentences: their row range and prev_cost are inputs (not other
  // CTAs' results), so each warp requests its first sentence's now and the
  // loads overlap the grid-wide wait below
  int pre_r0 = -1, pre_r1 = 0;
  float pre_pc = 0.f;
  if (KB == 1 && (p.tail & 15) == TAIL_SENT && !(p.tail & TAIL_X_NOWORK)) {
    const int s = blockIdx.x + gridDim.x * (tid >> 5);
    if (s < p.mp.S) {
      pre_r0 = p.mp.offsets[s];
      pre_r1 = p.mp.offsets[s + 1];
      pre_pc = pre_r1 > pre_r0 ? p.mp.prev_cost[pre_r0] : 0.f;
    }
  }
  if (tid == 0) {
    // arrival: acq_rel RMW on this launch's counter (release: the CTA's
    // records, ordered before it by the barrier; acquire: every earlier
    // arrival's records, through the RMW chain)
    unsigned int* ctr = p.arrive + (tag & 1u);
    const unsigned int prev = atom_add_acq_rel_gpu(ctr, 1u);
    if (prev + 1u == gridDim.x || (p.tail & TAIL_X_NOWORK && p.tail & TAIL_X_FENCE)) {
      p.gen_ctr[0] = tag;   // last arrival: every CTA has read the generation
    } else {
      // one poller per CTA, with backoff: polling must not steal L2 request
      // slots from the CTAs still streaming W (measured: 256 tight pollers
      // per CTA cost the HBM-bound greedy config ~1.5 us)
      const unsigned long long t0 = globaltimer_ns();
      unsigned int v;
      while ((v = ld_acquire_gpu(ctr)) != gridDim.x) {
        if (v > gridDim.x || globaltimer_ns() - t0 > 10000000000ull) {
          printf("AMUN: fused tail of CTA %d: arrival count %u of %u after %llu ns: the "
                 "workspace was not initialised (amun_ol_workspace_init) or CTAs are not "
                 "co-resident\n", (int)blockIdx.x, v, gridDim.x, globaltimer_ns() - t0);
          __trap();
        }
        __nanosleep(p.tail & TAIL_X_SLEEP ? 32 : 128);
      }
    }
  }
  MergeWarpsSync()();
  if (tid == 0) tl_mark(p.tl, TL_RELEASED);

  MergeParams mp = p.mp;
  mp.N = dyn.N;
  mp.sch = dyn.sch;
  const int G = gridDim.x, c = blockIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kind = p.tail & 15;
  if (p.tail & TAIL_X_NOWORK) return;   // (experiment: the arrival / wait alone)
  if (kind == TAIL_SENT && KB == 1) {   // k_max = 1: a warp per sentence (merge_sentence_k1)
    for (int s = c + G * warp; s < mp.S; s += G * MS_WARPS) {
      merge_sentence_k1(mp, s, lane, pre_r0, pre_r1, pre_pc);
      pre_r0 = -1;   // later sentences load their own
    }
  } else if (kind == TAIL_SENT) {
    Cand* pool = reinterpret_cast<Cand*>(scratch);
    Cand* best = pool + KB + MS_CAP;
    int* s_valid = reinterpret_cast<int*>(best + KB);
    for (int s = c; s < mp.S; s += G) {
      merge_sentence<KB, MergeWarpsSync>(mp, s, pool, best, *s_valid);
      MergeWarpsSync()();
    }
  } else if (kind == TAIL_ROWS) {
    for (int r = c + G * warp; r < mp.N; r += G * MS_WARPS) merged_row_record<KB>(mp, r, lane);
  } else if (kind == TAIL_ARGMAX) {
    for (int r = c + G * warp; r < mp.N; r += G * MS_WARPS)
      argmax_row(mp, r, lane, mp.out_idx, mp.out_cost);
  } else if (kind == TAIL_ONESHOT) {
    Cand* pool = reinterpret_cast<Cand*>(scratch);
    Cand* best = pool + KB + MS_CAP;
    int* s_valid = reinterpret_cast<int*>(best + KB);
    int* s_os = s_valid + 1;          // {failed wait, epoch}
    const OneShotTail& os = p.os;
    // the epoch: read before this CTA's done-arrival (os_signal), which the
    // rank's last CTA waits for before it advances the epoch
    if (tid == 0) {
      s_os[0] = 0;
      s_os[1] = (int)os_epoch(os.buf[os.rank]);
    }
    MergeWarpsSync()();
    const unsigned int epoch = (unsigned int)s_os[1];
    for (int r = c + G * warp; r < mp.N; r += G * MS_WARPS) {
      float lse, M, Z, l;
      int v;
      row_topk<KB>(mp, r, lane, lse, M, Z, l, v);
      os_store_record(os.buf, os.G, os_record_off(epoch, os.recv_elems, os.rank, mp.N, r, mp.stride),
                      mp.k_max, lane, M, Z, l, v);
    }
    MergeWarpsSync()();
    if (tid == 0) os_signal(os.buf, os.G, os.rank, G, epoch);
    if (!os_wait(os.buf[os.rank], os.G, epoch)) s_os[0] = 1;
    MergeWarpsSync()();
    if (s_os[0]) return;
    MergeParams dp = mp;              // sentence phase over [G][N][stride]
    dp.layout = 1;
    dp.G = os.G;
    dp.part_floats = os.recv_elems;
    dp.part = reinterpret_cast<const float*>(os.buf[os.rank] + OS_CTRL_BYTES) +
              (long long)(epoch & 1u) * os.recv_elems;
    for (int s = c; s < dp.S; s += G) {
      merge_sentence<KB, MergeWarpsSync>(dp, s, pool, best, *s_valid);
      MergeWarpsSync()();
    }
  }
  if (p.tl) {
    MergeWarpsSync()();
    if (tid == 0) tl_mark(p.tl, TL_TAIL_END);
  }
}

}  // namespace amun
