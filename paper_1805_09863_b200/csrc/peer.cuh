// peer.cuh — the NVLink one-shot exchange protocol,
// shared by the standalone one-shot kernel (oneshot.cuh; the one-GPU
// emulation of G ranks) and the fused kernel's tail (tail.cuh TAIL_ONESHOT;
// the real multi-GPU path).
//
// Alg. 6 reduces the per-shard states (max^j, best^j) in a
// serial step after every shard is done. Across GPUs the shard states are
// per-row records {M, Z, l[k], v[k]} (the monoid of merge.cuh). Each rank
// stores its rows' records straight into slot [me] of EVERY rank's receive
// buffer (CUDA-IPC mappings: NVLink stores), signals, waits for every rank's
// signal, then reduces the G records of each row in rank order — the same
// reduce as all-gather + merge (reading G18).
//
// Buffer of one rank (one cudaMalloc, exported by IPC handle):
//   control: u32 cnt[8] (calls signalled per source rank, monotonic),
//            u32 epoch (calls of this rank), u32 done (CTAs of the current
//            call past the row phase), u32 err (1 after a timed-out wait),
//            padded to OS_CTRL_BYTES;
//   recv:    fp32 [2][G][max_rows][stride], double-buffered by epoch parity.
// Counters only grow, so no reset is needed between calls (CUDA-graph
// replays included). Parity double-buffering is sufficient: a peer can be
// at most one call ahead (its call e+1 waits for this rank's call e+1
// signals, which are sent after this rank's call e has finished reading).
#pragma once
#include <cstdint>

namespace amun {

constexpr int OS_MAX_G = 8;
constexpr int OS_CTRL_BYTES = 256;
constexpr int OS_EPOCH = OS_MAX_G;       // control word indices
constexpr int OS_DONE = OS_MAX_G + 1;
constexpr int OS_ERR = OS_MAX_G + 2;
constexpr unsigned long long OS_TIMEOUT_NS = 4000000000ull;   // 4 s

// The one-shot exchange as the fused kernel's tail sees it (TcParams::os).
struct OneShotTail {
  char* buf[OS_MAX_G];   // every rank's one-shot buffer as mapped in this process
  int G, rank;
  long long recv_elems;  // floats per parity half: G * max_rows * stride
};

__device__ __forceinline__ void red_release_sys_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int atom_add_acq_rel_gpu_u32(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long os_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The epoch (calls of this rank so far). Written only by this rank's
// previous call (stream order makes it visible): a plain volatile load.
__device__ __forceinline__ unsigned int os_epoch(const char* own_buf) {
  return *reinterpret_cast<const volatile unsigned int*>(
      reinterpret_cast<const unsigned int*>(own_buf) + OS_EPOCH);
}

// Float offset of rank `me`'s record of row r in the receive half of `epoch`.
__device__ __forceinline__ long long os_record_off(unsigned int epoch, long long recv_elems, int me,
                                                   int N, int r, int stride) {
  return (long long)(epoch & 1u) * recv_elems + ((long long)me * N + r) * stride;
}

// Row phase, one full warp (lane l holds entry l of the merged top-k, as
// records_topk leaves it): the record {M, Z, l[k_max], v[k_max]} into slot
// `off` of every rank's receive buffer.
__device__ __forceinline__ void os_store_record(char* const* buf, int G, long long off, int k_max,
                                                int lane, float M, float Z, float l, int v) {
  for (int p = 0; p < G; ++p) {
    float* rec = reinterpret_cast<float*>(buf[p] + OS_CTRL_BYTES) + off;
    if (lane == 0) *reinterpret_cast<float2*>(rec) = make_float2(M, Z);
    if (lane < k_max) {
      rec[2 + lane] = l;
      rec[2 + k_max + lane] = __int_as_float(v);
    }
  }
}

// Signal, thread 0 of each of the nb CTAs of this rank's call, after a CTA
// barrier that follows the CTA's record stores: the LAST CTA advances the
// epoch and adds 1 to counter [me] of every rank (one system-scope release
// per peer per call). Ordering chain: each CTA's stores -> barrier -> its
// thread 0's acq_rel RMW on `done` (gpu scope, a release sequence) -> the
// last CTA's RMW -> its red.release.sys -> the peer's ld.acquire.sys.
// (A __threadfence_system() per CTA measured ~3 us per launch.)
__device__ __forceinline__ void os_signal(char* const* buf, int G, int me, int nb,
                                          unsigned int epoch) {
  unsigned int* ctrl = reinterpret_cast<unsigned int*>(buf[me]);
  if (atom_add_acq_rel_gpu_u32(ctrl + OS_DONE, 1u) == (unsigned int)nb - 1u) {
    ctrl[OS_DONE] = 0u;               // next call (stream order) starts from 0
    ctrl[OS_EPOCH] = epoch + 1u;
    for (int p = 0; p < G; ++p)
      red_release_sys_add(reinterpret_cast<unsigned int*>(buf[p]) + me, 1u);
  }
}

// Wait (acquire), threads 0..G-1 of a CTA: until every source rank has
// signalled call `epoch`. Bounded: a rank that never signals (it failed
// host validation, passed another N, or never called) sets the error word
// after OS_TIMEOUT_NS and the wait returns false — no hung GPU; the host
// reads the word with amun_oneshot_error. Follow with a CTA barrier.
__device__ __forceinline__ bool os_wait(const char* own_buf, int G, unsigned int epoch) {
  if ((int)threadIdx.x >= G) return true;
  const unsigned int* c = reinterpret_cast<const unsigned int*>(own_buf) + threadIdx.x;
  unsigned long long t0 = 0;
  int spins = 0;
  while ((int)(ld_acquire_sys(c) - (epoch + 1u)) < 0) {
    if (++spins == 64) t0 = os_globaltimer();
    if (spins > 64 && (spins & 255) == 0 && os_globaltimer() - t0 > OS_TIMEOUT_NS) {
      atomicExch(const_cast<unsigned int*>(reinterpret_cast<const unsigned int*>(own_buf)) + OS_ERR,
                 1u);
      printf("AMUN one-shot: rank slot %d never signalled call %u (timeout); outputs of this "
             "call are not written\n", (int)threadIdx.x, epoch);
      return false;
    }
    __nanosleep(32);
  }
  return true;
}

}  // namespace amun
