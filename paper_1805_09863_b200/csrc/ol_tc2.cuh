// ol_tc2.cuh — the fused output layer on CTA pairs (tcgen05.mma.cta_group::2).
//
// Same steps, epilogue (tc_epi.cuh) and partial records as ol_tc.cuh; the
// mainloop runs on a pair of CTAs of one cluster (the two SMs of a TPC):
//   * the pair computes a 256-row x N-vocab tile (N <= 256) per MMA:
//     CTA rank r holds rows [128 r, 128 r + 128) of the pair's A tile (X of
//     M-tile 2 mp + r) and vocab rows [r N/2, (r+1) N/2) of the B tile (W),
//     so each SM's shared memory carries 32 KB per 64-deep K step instead of
//     48 KB (64 + 64 B/clk of TMA writes + tensor-core reads at full MMA
//     rate; the 1-CTA 128x256 tile needs 96 + 96 B/clk);
//   * only the leader (rank 0) issues tcgen05.mma; both CTAs' TMA loads
//     complete on the leader's `full` barrier; the leader's commits arrive on
//     `empty`/`tfull` of both CTAs (multicast); both CTAs' epilogue warps
//     arrive on the leader's `tempty`;
//   * each CTA's TMEM holds its own 128 rows x N columns, so the epilogue is
//     the single-CTA one.
#pragma once
#include "tail.cuh"

namespace amun {

#ifdef TC2_STAGES_OVERRIDE
constexpr int TC2_STAGES = TC2_STAGES_OVERRIDE;
#else
constexpr int TC2_STAGES = 6;
#endif
constexpr int TC2_A_BYTES = TC_BM * TC_BK * 2;          // 16 KB: this CTA's 128 rows of X
constexpr int TC2_B_BYTES = (TC_BN / 2) * TC_BK * 2;    // 16 KB: this CTA's half of the W tile
constexpr int TC2_SMEM = TC2_STAGES * (TC2_A_BYTES + TC2_B_BYTES) + TC_BIAS_BYTES + TC_XCH_BYTES +
                         TC_THRX_BYTES + 1024 /*align*/ + 512 /*barriers*/;
static_assert(TC_NBIAS >= 2 + TC2_STAGES, "bias ring too small for the producer's lead");

template <int KB, int MODE, int NG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TcCfg<NG>::kThreads, 1)
    ol_tc2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap /*tmWn: single-CTA kernel only*/,
                  const TcParams p) {
  using Cfg = TcCfg<NG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + TC2_STAGES * TC2_A_BYTES;
  float* sbias = reinterpret_cast<float*>(sB + TC2_STAGES * TC2_B_BYTES);
  float* xch = sbias + TC_NBIAS * TC_BN;
  unsigned long long* thr_x = reinterpret_cast<unsigned long long*>(xch + 128 * TC_XCH_FLOATS);
  uint64_t* full = reinterpret_cast<uint64_t*>(thr_x + TC_THRX_BYTES / 8);
  uint64_t* empty = full + TC2_STAGES;
  uint64_t* tfull = empty + TC2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bfull + TC_NBIAS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Warp roles: the epilogue warpgroups take the LOW warp ids and the control
  // warpgroup (TMA producer, MMA issuer, 2 idle) the highest ones: the warp
  // scheduler favours higher warp ids, so the single-thread producer/issuer
  // are not starved by the busy epilogue warps sharing their sub-partition.
  constexpr int kCtrl = 4 * NG;                    // first control warp
  const int role = warp - kCtrl;                   // 0 = TMA, 1 = MMA, 2-3 idle, < 0 epilogue
  const uint32_t rank = cluster_ctarank();          // 0 = leader, 1 = peer
  const int pair = blockIdx.x >> 1;

  for (int i = threadIdx.x; i < TC_THRX_BYTES / 8; i += blockDim.x)   // no stale tags
    sts_u64(smem_u32(thr_x + i), 0ull);
  if (role == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int i = 0; i < TC2_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * NG * 4);     // one arrival per epilogue warp of the pair
    }
    for (int i = 0; i < TC_NBIAS; ++i) mbar_init(&bfull[i], 1);
    fence_barrier_init();
  }
  if (role == 1) {
    tmem_alloc_2sm(tmem_holder, 512);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  cluster_sync();      // barriers of both CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // this launch's tag (hints, tail counters): read by the epilogue threads
  // (the only users), off the TMA producer's path to its first load
  uint32_t gen = 0u;

  const TcDyn dyn = tc_dyn<true>(p);       // N (and the schedule) from the device in _dev mode
  const long long start = (long long)pair * dyn.sch.C;
  const long long stop = min(start + dyn.sch.C, dyn.sch.total);

  if (role >= 0) {
    reg_dealloc<Cfg::kCtrlRegs>();
    if (role == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_x = policy_evict_last();
      TileIter it{start, stop, dyn.sch};
      int mp, v0, width;
      bool last;
      int stage = 0, tile = 0;
      uint32_t phase = 0;
      while (it.next(mp, v0, width, last)) {
        const int mt = 2 * mp + (int)rank;
        const int vb = v0 + (int)rank * (width >> 1);   // this CTA's half of the B tile
        if (lane == 0) bias_ring_load(p, sbias, bfull, tile, v0, width);
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait_spin(&empty[stage], phase ^ 1);
          if (lane == 0) {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (TC2_A_BYTES + TC2_B_BYTES));
            const uint32_t lb = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_2d_2sm(&tmX, lb, sA + stage * TC2_A_BYTES, kb * TC_BK, mt * TC_BM, pol_x);
            tma_load_2d_2sm(&tmW, lb, sB + stage * TC2_B_BYTES, kb * TC_BK, vb, 0ull);
          }
          __syncwarp();
          if (++stage == TC2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ++tile;
      }
    } else if (role == 1 && rank == 0) {
      // ------------------------------------------------ MMA issuer (leader only)
      TileIter it{start, stop, dyn.sch};
      int mp, v0, width;
      bool last;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      while (it.next(mp, v0, width, last)) {
        mbar_wait_spin(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * TC_BN;
        const uint32_t idesc = idesc_bf16_f32(2 * TC_BM, width);
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait_spin(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t ad = sdesc_k_sw128(smem_u32(sA + stage * TC2_A_BYTES));
            const uint64_t bd = sdesc_k_sw128(smem_u32(sB + stage * TC2_B_BYTES));
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k)
              mma_bf16_2sm(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            mma_commit_2sm_mc(&empty[stage], 0x3);   // both CTAs' slots free
          }
          __syncwarp();
          if (++stage == TC2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) mma_commit_2sm_mc(&tfull[acc], 0x3);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    reg_alloc<Cfg::kEpiRegs>();
    if constexpr (MODE == 0 || MODE == 4) {
      gen = read_generation(p.gen_ctr);
      // the next launch's tail counter (tail.cuh "Counters")
      if (blockIdx.x == 0 && threadIdx.x == 0) p.arrive[(gen + 1u) & 1u] = 0u;
    }
    tc_epilogue<KB, MODE, NG, true>(p, tmem_base, start, stop, tfull, tempty, bfull, sbias, xch,
                                    thr_x, gen, warp, lane, rank, (long long)pair, dyn);
    if constexpr (MODE == 0 || MODE == 4) {
      // the merge in this launch, inside the epilogue branch (see ol_tc.cuh)
      if (p.tail) {
        tc_fence_before();
        named_bar_sync(11, Cfg::kEpiThreads);
        grid_tail<KB>(p, dyn, reinterpret_cast<uint8_t*>(xch), gen);
      }
    }
  }

  tc_fence_before();
  cluster_sync();      // the leader's last commits/arrivals into the peer are done
  if (role == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
  if constexpr (MODE == 0 || MODE == 4) {
    if (!p.tail && threadIdx.x == 0) finish_generation(p.gen_ctr);
  }
}

}  // namespace amun
