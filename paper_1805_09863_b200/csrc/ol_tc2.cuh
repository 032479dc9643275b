// ol_tc2.cuh — the fused output layer on CTA pairs (tcgen05.mma.cta_group::2).
//
// Same steps, epilogue and partial records as ol_tc.cuh (read that first);
// the mainloop runs on a pair of CTAs of one cluster (the two SMs of a TPC):
//   * the pair computes a 256-row x N-vocab tile (N <= 256) per MMA:
//     CTA rank r holds rows [128 r, 128 r + 128) of the pair's A tile (X of
//     M-tile 2 mp + r) and vocab rows [r N/2, (r+1) N/2) of the B tile (W),
//     so each SM's shared memory carries 32 KB per 64-deep K step instead of
//     48 KB: 64 + 64 B/clk of TMA writes + tensor-core reads at full MMA rate,
//     within the SM's shared-memory bandwidth (the 1-CTA 128x256 tile needs
//     96 + 96 B/clk and measured shared-memory bound);
//   * only the leader (rank 0) issues tcgen05.mma; both CTAs' TMA loads
//     complete on the leader's `full` barrier; the leader's commits arrive on
//     `empty`/`tfull` of both CTAs (multicast); both CTAs' epilogue warps
//     arrive on the leader's `tempty`;
//   * each CTA's TMEM holds its own 128 rows x N columns, so the epilogue is
//     the single-CTA one unchanged.
#pragma once
#include "ol_tc.cuh"

namespace amun {

#ifdef TC2_STAGES_OVERRIDE
constexpr int TC2_STAGES = TC2_STAGES_OVERRIDE;
#else
constexpr int TC2_STAGES = 6;
#endif
constexpr int TC2_A_BYTES = TC_BM * TC_BK * 2;          // 16 KB: this CTA's 128 rows of X
constexpr int TC2_B_BYTES = (TC_BN / 2) * TC_BK * 2;    // 16 KB: this CTA's half of the W tile
constexpr int TC2_SMEM = TC2_STAGES * (TC2_A_BYTES + TC2_B_BYTES) + TC_XS_BYTES + TC_MS_BYTES +
                         1024 /*align*/ + 256 /*barriers*/;
constexpr int TC2_EPI_WARPS = TC_EPI_THREADS / 32;

template <int KB, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    ol_tc2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + TC2_STAGES * TC2_A_BYTES;
  float* xs_all = reinterpret_cast<float*>(sB + TC2_STAGES * TC2_B_BYTES);
  float* ms_x = reinterpret_cast<float*>(sB + TC2_STAGES * TC2_B_BYTES + TC_XS_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + TC2_STAGES * TC2_B_BYTES + TC_XS_BYTES +
                                               TC_MS_BYTES);
  uint64_t* empty = full + TC2_STAGES;
  uint64_t* tfull = empty + TC2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* gen_smem = tmem_holder + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();          // 0 = leader, 1 = peer
  const int pair = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int i = 0; i < TC2_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * TC2_EPI_WARPS);   // one arrival per epilogue warp of the pair
    }
    fence_barrier_init();
    *gen_smem = (MODE == 0) ? read_generation(p.gen_ctr) : 0u;
  }
  if (warp == 1) {
    tmem_alloc_2sm(tmem_holder, 512);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  cluster_sync();      // barriers of both CTAs initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t gen = *gen_smem;   // this launch's hint tag
  pdl_trigger();

  const long long start = (long long)pair * p.sch.C;
  const long long stop = min(start + p.sch.C, p.sch.total);

  if (warp < 4) {
    reg_dealloc<TC_CTRL_REGS>();
    if (warp == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_x = policy_evict_last();
      TileIter it{start, stop, p.sch};
      int mp, v0, width;
      bool last;
      int stage = 0;
      uint32_t phase = 0;
      while (it.next(mp, v0, width, last)) {
        const int mt = 2 * mp + (int)rank;
        const int vb = v0 + (int)rank * (width >> 1);   // this CTA's half of the B tile
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
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
      }
    } else if (warp == 1 && rank == 0) {
      // ------------------------------------------------ MMA issuer (leader only)
      TileIter it{start, stop, p.sch};
      int mp, v0, width;
      bool last;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      while (it.next(mp, v0, width, last)) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * TC_BN;
        const uint32_t idesc = idesc_bf16_f32(2 * TC_BM, width);
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait(&full[stage], phase);
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
    reg_alloc<TC_EPI_REGS>();
    // ------------------------------------------------ epilogue (warps 4..11, both CTAs)
    const int e = warp - 4;
    const int grp = e >> 2;
    const int q = warp & 3;
    const int row_local = q * 32 + lane;
    const int sw = row_local & 7;
    const uint32_t t_lane = (uint32_t)(q * 32) << 16;
    float* xs = xs_all + (grp * 128 + row_local) * 32;
    const uint32_t tempty_leader[2] = {mapa_shared(smem_u32(&tempty[0]), 0),
                                       mapa_shared(smem_u32(&tempty[1]), 0)};
    RowState<KB> st;
    st.reset();
    TileIter it{start, stop, p.sch};
    int mp, v0, width;
    bool last;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t ra[32], rb[32];
    float ba[32], bn[32];
    float hintv = kNegInf, published = kNegInf;
    while (it.next(mp, v0, width, last)) {
      const int mt = 2 * mp + (int)rank;
      const int row = mt * TC_BM + row_local;
      const bool live = mt * TC_BM < p.N;            // warp-uniform: padding M-tile of a pair
      const int limit = min(width, p.V_local - v0);
      const int nch = (width + 31) >> 5;
      if (live && grp < nch) load_bias32(p.bias, v0, grp * 32, limit, ba);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + t_lane + acc * TC_BN;
      if (live) {
        if (grp < nch) tmem_ld32(tbase + grp * 32, ra);
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
      if (MODE == 0 && row < p.N) {
        if (st.l[KB - 1] > published) {
          published = st.l[KB - 1];
          atomicMax(p.hint + row, hint_encode(published, gen));
        }
        hintv = fmaxf(hintv, hint_decode(__ldcg(p.hint + row), gen));
      }
      if (last) {
        hintv = kNegInf;
        published = kNegInf;
        if constexpr (MODE != 1) {
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
            const float* o = xs + 128 * 32;
            float l2[KB];
            int v2[KB];
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              l2[i] = o[i];
              v2[i] = __float_as_int(o[16 + i]);
            }
            st.combine(ms_x[2 * row_local], ms_x[2 * row_local + 1], l2, v2);
            if (row < p.N) {
              // pair layout: slot (pair + mp) * 2 + rank holds M-tile 2 mp + rank
              const long long slot = ((long long)pair + mp) * 2 + rank;
              st.emit(p.part + (slot * TC_BM + row_local) * p.stride, p.k_max);
            }
          }
          named_bar_sync(5 + q, 64);
        }
        st.reset();
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync();      // the leader's last commits/arrivals into the peer are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
  if (MODE == 0 && threadIdx.x == 0) finish_generation(p.gen_ctr);
}

}  // namespace amun
