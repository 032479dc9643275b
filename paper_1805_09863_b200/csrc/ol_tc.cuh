// ol_tc.cuh — fused output layer on the 5th-gen tensor cores (sm_100a).
//
// Steps 1-4 of PAPER.md P:81-87 in one persistent, warp-specialised kernel:
//   warp 0  TMA producer: X tile [128 rows x 64 K] and W tile [256 vocab x 64 K]
//           per stage (128B swizzle), STAGES-deep mbarrier ring.
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer:
//           D[128 x width] (fp32, TMEM) += X_tile * W_tile^T, K = 16 per MMA.
//           Two TMEM accumulators (2 x 256 columns = all 512) so the epilogue
//           of tile t overlaps the MMAs of tile t+1.
//   warps 2-3  idle (the control warpgroup 0-3 gives its registers away)
//   warps 4-11 epilogue, two warpgroups of four warps (one warp per TMEM lane
//           quadrant in each group; group g takes the 32-column chunks
//           c = g, g+2, ... of every tile, so two warps per SM sub-partition
//           hide each other's latency). Thread = hypothesis row. Per chunk:
//           tcgen05.ld of 32 columns, + bias (step 2), online max/sum-of-exp
//           (step 3, Alg. 4 with the exp(Delta) rescale of P:193-200) and a
//           register k-best (step 4). The N x V logits never reach
//           HBM. At the end of a CTA's range in an M-tile the two groups'
//           states are combined (same monoid as the merge) and one partial
//           record {m, s, top-k} per (row, CTA range) is written (Alg. 6's
//           per-shard state).
// MODE 1 (test hook) writes the biased logits instead of statistics.
// MODE 2 / 3 (benchmark hooks, the analogue of the paper's Table 4 split):
// 2 = bare GEMM (the epilogue only drains TMEM), 3 = GEMM + bias + online
// softmax statistics without the k-best.
#pragma once
#include "epilogue.cuh"

namespace amun {

struct TcParams {
  int N, V_local, v_offset, n_kblk;
  Schedule sch;
  const float* __restrict__ bias;
  float* __restrict__ part;   // [slots][128][stride]
  int stride, k_max;
  float* __restrict__ logits; // MODE 1: [N][V_local]
  unsigned long long* __restrict__ hint;   // [N] cross-CTA k-th-best hints
  unsigned int* __restrict__ gen_ctr;      // {generation, CTAs done}: device-side, so every
                                           // launch (graph replays too) gets a fresh tag
};

// Read the launch generation (all CTAs, before any of them finishes).
__device__ __forceinline__ uint32_t read_generation(const unsigned int* gen_ctr) {
  return 1u + *reinterpret_cast<const volatile unsigned int*>(gen_ctr);
}
// Called once per CTA after all its work: the last CTA advances the generation.
__device__ __forceinline__ void finish_generation(unsigned int* gen_ctr) {
  __threadfence();
  const unsigned int prev = atomicAdd(gen_ctr + 1, 1u);
  if (prev == gridDim.x - 1) {   // every CTA has read the generation and finished
    gen_ctr[1] = 0u;
    atomicAdd(gen_ctr, 1u);
    __threadfence();
  }
}

constexpr int TC_BM = 128;
#ifndef TC_BN_OVERRIDE
constexpr int TC_BN = 256;
#else
constexpr int TC_BN = TC_BN_OVERRIDE;
#endif
constexpr int TC_BK = 64;
#ifdef TC_STAGES_OVERRIDE
constexpr int TC_STAGES = TC_STAGES_OVERRIDE;
#else
constexpr int TC_STAGES = 4;
#endif
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;   // 16 KB
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;   // 32 KB
constexpr int TC_EPI_GROUPS = 2;
constexpr int TC_EPI_THREADS = TC_EPI_GROUPS * 128;
constexpr int TC_THREADS = 128 + TC_EPI_THREADS;  // control warpgroup + epilogue warpgroups
// setmaxnreg budgets. They only redistribute the CTA's launch pool
// (TC_LAUNCH_REGS per thread): a warpgroup can grow only into what the
// others released, else setmaxnreg.inc blocks forever.
constexpr int TC_LAUNCH_REGS = 65536 / TC_THREADS / 8 * 8;   // 168
constexpr int TC_CTRL_REGS = 56;
constexpr int TC_EPI_REGS = 224;
static_assert(128 * TC_CTRL_REGS + TC_EPI_THREADS * TC_EPI_REGS <= TC_LAUNCH_REGS * TC_THREADS,
              "setmaxnreg budget exceeds the launch register pool");
constexpr int TC_XS_BYTES = TC_EPI_GROUPS * 128 * 32 * 4;   // candidate scratch, 16 KB/group
constexpr int TC_MS_BYTES = 128 * 2 * 4;                    // group-exchange (m, s)
constexpr int TC_SMEM = TC_STAGES * (TC_A_BYTES + TC_B_BYTES) + TC_XS_BYTES + TC_MS_BYTES +
                        1024 /*align*/ + 256 /*barriers*/;

// Bias of columns [v0 + c0, v0 + c0 + 32) (zero past `limit`): eight 16-byte
// loads whose address is the same for every lane of the warp (broadcast).
__device__ __forceinline__ void load_bias32(const float* __restrict__ bias, int v0, int c0,
                                            int limit, float (&bb)[32]) {
  const int nv = limit - c0;
  if (nv >= 32) {
    const float4* b4 = reinterpret_cast<const float4*>(bias + v0 + c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 t = __ldg(b4 + j);
      bb[4 * j + 0] = t.x;
      bb[4 * j + 1] = t.y;
      bb[4 * j + 2] = t.z;
      bb[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) bb[j] = (j < nv) ? __ldg(bias + v0 + c0 + j) : 0.f;
  }
}

// Step 2 (+ bias) and the per-row statistics for one 32-column chunk.
template <int KB, int MODE>
__device__ __forceinline__ void consume_chunk(const TcParams& p, RowState<KB>& st,
                                              const uint32_t (&r)[32], const float (&bb)[32],
                                              int row, int v0, int c0, int limit, float* xs,
                                              int sw, float hint) {
  const int nv = limit - c0;
  float x[32];
  if (nv >= 32) {   // full chunk (all but the vocabulary tail): no masking
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]) + bb[j];
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = (j < nv) ? __uint_as_float(r[j]) + bb[j] : kNegInf;
  }
  if constexpr (MODE == 1) {
    if (row < p.N) {
      float* out = p.logits + (long long)row * p.V_local + v0 + c0;
      for (int j = 0; j < 32 && j < nv; ++j) out[j] = x[j];
    }
  } else if constexpr (MODE == 2) {
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= r[j];
    st.s += __uint_as_float(acc & 0x007fffffu);   // keep the loads alive
  } else if constexpr (MODE == 3) {
    st.template chunk32<false>(x, p.v_offset + v0 + c0, xs, sw, hint);
  } else {
    st.chunk32(x, p.v_offset + v0 + c0, xs, sw, hint);
  }
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int KB, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1)
    ol_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                 const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + TC_STAGES * TC_A_BYTES;
  float* xs_all = reinterpret_cast<float*>(sB + TC_STAGES * TC_B_BYTES);
  float* ms_x = reinterpret_cast<float*>(sB + TC_STAGES * TC_B_BYTES + TC_XS_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + TC_STAGES * TC_B_BYTES + TC_XS_BYTES +
                                               TC_MS_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* gen_smem = tmem_holder + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], TC_EPI_THREADS);
    }
    fence_barrier_init();
    *gen_smem = (MODE == 0) ? read_generation(p.gen_ctr) : 0u;
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t gen = *gen_smem;   // this launch's hint tag
  pdl_trigger();   // let the dependent merge grid get scheduled early (it waits for us)

  const long long start = (long long)blockIdx.x * p.sch.C;
  const long long stop = min(start + p.sch.C, p.sch.total);

  if (warp < 4) {
  reg_dealloc<TC_CTRL_REGS>();
  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    // The whole warp walks the schedule (keeps it converged); lane 0 issues.
    const uint64_t pol_x = policy_evict_last();     // X is re-read by every CTA
    TileIter it{start, stop, p.sch};
    int mt, v0, width;
    bool last;
    int stage = 0;
    uint32_t phase = 0;
    while (it.next(mt, v0, width, last)) {
      for (int kb = 0; kb < p.n_kblk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[stage], TC_A_BYTES + TC_B_BYTES);
          tma_load_2d(&tmX, &full[stage], sA + stage * TC_A_BYTES, kb * TC_BK, mt * TC_BM, pol_x);
          tma_load_2d(&tmW, &full[stage], sB + stage * TC_B_BYTES, kb * TC_BK, v0, 0ull);
        }
        __syncwarp();
        if (++stage == TC_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // The whole warp waits; lane 0 issues tcgen05.mma and the commits (a
    // commit tracks the MMAs issued by the same thread).
    TileIter it{start, stop, p.sch};
    int mt, v0, width;
    bool last;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    while (it.next(mt, v0, width, last)) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * TC_BN;
      const uint32_t idesc = idesc_bf16_f32(TC_BM, width);
      for (int kb = 0; kb < p.n_kblk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint64_t ad = sdesc_k_sw128(smem_u32(sA + stage * TC_A_BYTES));
          const uint64_t bd = sdesc_k_sw128(smem_u32(sB + stage * TC_B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)   // +32 bytes of K per MMA (>>4 = 2)
            mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);              // smem slot free once these MMAs finish
        }
        __syncwarp();
        if (++stage == TC_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) mma_commit(&tfull[acc]);     // accumulator ready for the epilogue
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  } else {
    reg_alloc<TC_EPI_REGS>();
    // ------------------------------------------------ epilogue (warps 4..11)
    const int e = warp - 4;
    const int grp = e >> 2;                        // 0 or 1: which chunks
    const int q = warp & 3;                        // TMEM lane quadrant of this warp
    const int row_local = q * 32 + lane;
    const int sw = row_local & 7;
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    float* xs = xs_all + (grp * 128 + row_local) * 32;
    RowState<KB> st;
    st.reset();
    TileIter it{start, stop, p.sch};
    int mt, v0, width;
    bool last;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t ra[32], rb[32];
    float ba[32], bn[32];
    float hintv = kNegInf, published = kNegInf;
    while (it.next(mt, v0, width, last)) {
      const int row = mt * TC_BM + row_local;
      const int limit = min(width, p.V_local - v0);
      const int nch = (width + 31) >> 5;
      // newest cross-CTA hint for this row (L2, not L1: other SMs update it)
      // bias of this group's first chunk requested before the accumulator wait
      if (grp < nch) load_bias32(p.bias, v0, grp * 32, limit, ba);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + t_lane + acc * TC_BN;
      if (grp < nch) tmem_ld32(tbase + grp * 32, ra);
      // software pipeline: TMEM + bias loads of chunk c+2 fly while c is consumed
      for (int c = grp; c < nch; c += 4) {
        tmem_ld_wait(ra);
        if (c + 2 < nch) {
          tmem_ld32(tbase + (c + 2) * 32, rb);
          load_bias32(p.bias, v0, (c + 2) * 32, limit, bn);
        }
        consume_chunk<KB, MODE>(p, st, ra, ba, row, v0, c * 32, limit, xs, sw, hintv);
        if (c + 2 >= nch) break;
        tmem_ld_wait(rb);
        if (c + 4 < nch) {
          tmem_ld32(tbase + (c + 4) * 32, ra);
          load_bias32(p.bias, v0, (c + 4) * 32, limit, ba);
        }
        consume_chunk<KB, MODE>(p, st, rb, bn, row, v0, (c + 2) * 32, limit, xs, sw, hintv);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (MODE == 0 && row < p.N) {
        if (st.l[KB - 1] > published) {   // publish our k-th best
          published = st.l[KB - 1];
          atomicMax(p.hint + row, hint_encode(published, gen));
        }
        // newest cross-CTA hint for the next tile (L2, not L1: other SMs
        // update it); its latency overlaps the next accumulator wait
        hintv = fmaxf(hintv, hint_decode(__ldcg(p.hint + row), gen));
      }
      if (last) {
        hintv = kNegInf;   // next segment is a different M-tile (other rows)
        published = kNegInf;
        if constexpr (MODE != 1) {
          // combine the two groups' states for this row, then emit
          if (grp == 1) {
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              xs[i] = st.l[i];
              xs[16 + i] = __int_as_float(st.v[i]);
            }
            ms_x[2 * row_local] = st.m;
            ms_x[2 * row_local + 1] = st.s;
          }
          named_bar_sync(1 + q, 64);
          if (grp == 0) {
            const float* o = xs + 128 * 32;        // the same row of group 1
            float l2[KB];
            int v2[KB];
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              l2[i] = o[i];
              v2[i] = __float_as_int(o[16 + i]);
            }
            st.combine(ms_x[2 * row_local], ms_x[2 * row_local + 1], l2, v2);
            if (row < p.N) {
              const long long slot = (long long)blockIdx.x + mt;
              st.emit(p.part + (slot * TC_BM + row_local) * p.stride, p.k_max);
            }
          }
          named_bar_sync(5 + q, 64);   // group 1 may reuse its scratch row after this
        }
        st.reset();
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if (MODE == 0 && threadIdx.x == 0) finish_generation(p.gen_ctr);
}

}  // namespace amun
