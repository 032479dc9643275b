// ol_tc.cuh — fused output layer on the 5th-gen tensor cores (sm_100a),
// single-CTA version (tcgen05.mma.cta_group::1).
//
// Steps 1-4 of PAPER.md P:81-87 in one persistent, warp-specialised kernel
// (epilogue warpgroups on the low warp ids, the control warpgroup on the
// highest four):
//   warps 0 .. 4NG-1  epilogue, NG warpgroups (tc_epi.cuh): + bias (step 2),
//           online softmax statistics (step 3), register k-best (step 4);
//           the N x V logits never reach HBM; one partial record
//           {m, s, top-k} per (row, CTA range) (Alg. 6's per-shard state,
//           P:232-242); then the merge in the launch's tail (tail.cuh).
//   warp 4NG    TMA producer: X tile [128 rows x 128 bytes of K] and W tile
//           [256 vocab rows x 128 bytes of K] per stage (128B swizzle),
//           STAGES-deep mbarrier ring; with each tile a 1-D bulk copy of its
//           bias slice into the bias ring. A range's narrow remainder tile
//           reads W in 64-row boxes (tmWn).
//   warp 4NG+1  TMEM allocator + single-thread tcgen05.mma issuer:
//           D[128 x width] (fp32, TMEM) += X_tile * W_tile^T, 32 bytes of K
//           per MMA. Two TMEM accumulators (2 x 256 columns = all 512) so the
//           epilogue of tile t overlaps the MMAs of tile t+1.
//   warp 4NG+2  mxfp4 plans: re-bases each stage's W scale atoms; else idle
//   warp 4NG+3  idle (the control warpgroup gives its registers away)
// MODE 1 (test hook) writes the biased logits instead of statistics.
// MODE 2 / 3 (benchmark hooks, the analogue of the paper's Table 4 split):
// 2 = bare GEMM (the epilogue only drains TMEM), 3 = GEMM + bias + online
// softmax statistics without the k-best.
#pragma once
#include "tail.cuh"

namespace amun {

// Pipeline geometry of the single-CTA kernel: stages of TC_KBYTES bytes of
// K per row (128: SWIZZLE_128B, 4 stages of 16 KB A + 32 KB B; 64:
// SWIZZLE_64B, 8 stages of 8 + 16 KB). The same 192 KB of stages; 64-byte
// blocks keep 7 of 8 stages in flight instead of 3 of 4 but measured 1.3x
// SLOWER per tile (9.2-9.9 vs 7.0 us at cfg beam, tools/timeline.py): twice
// the barrier round trips and MMA issues per byte. An L2-resident W (V =
// 45k, one copy) runs at the same 7.0 us per tile, so DRAM is not the bound.
#ifdef TC_STAGES_OVERRIDE
constexpr int TC_STAGES = TC_STAGES_OVERRIDE;
#else
constexpr int TC_STAGES = TC_KBYTES == 64 ? 8 : 4;
#endif
constexpr int TC_A_BYTES = TC_BM * TC_KBYTES;   // 8 KB (16 KB)
constexpr int TC_B_BYTES = TC_BN * TC_KBYTES;   // 16 KB (32 KB)
constexpr int TC_SMEM = TC_STAGES * (TC_A_BYTES + TC_B_BYTES) + TC_BIAS_BYTES + TC_XCH_BYTES +
                        TC_THRX_BYTES + 1024 /*align*/ + 512 /*barriers*/;
constexpr int TC_SMEM_F8 = TC_SMEM + TC_SCALE_BYTES;   // + the e4m3 column-scale ring
// MXFP4 (ELT 3): W stages of 224 rows (28 KB unpacked); per stage the raw
// scale atoms (up to 3) and the 2 atoms re-based to the tile's first row;
// A's constant atom.
constexpr int TC_B_BYTES_F4 = TC_BN_F4 * TC_KBYTES;
constexpr int TC_SMEM_F4 = TC_STAGES * (TC_A_BYTES + TC_B_BYTES_F4) + TC_BIAS_BYTES +
                           TC_XCH_BYTES + TC_THRX_BYTES + 1024 + 512 +
                           (1 + TC_STAGES * (TC_SF_RAW + 2)) * TC_SF_ATOM;
#if !defined(AMUN_WITH_NG3) && !defined(AMUN_WITH_NG4)
// (the NG3 / NG4 experiment builds' larger thr_x area leaves no room for the
// e4m3 / mxfp4 rings: those plans then fail at launch in such builds)
static_assert(TC_SMEM_F8 <= 227 * 1024 && TC_SMEM_F4 <= 227 * 1024, "shared memory budget");
#endif
static_assert(TC_B_BYTES_F4 % 1024 == 0, "SW128 tiles are 1024-byte aligned");
static_assert(TC_SFA_COL >= TC_BN_F4 && tc_sfb_col(2) + 8 <= 256 &&
              tc_sfb_col(3) >= 256 + TC_BN_F4 && tc_sfb_col(TC_STAGES - 1) + 8 <= 512,
              "mxfp4 scale columns overlap an accumulator");
static_assert(TC_NBIAS >= 2 + TC_STAGES, "bias ring too small for the producer's lead");

// ELT = 0: bf16 X, W (kind::f16, 64 elements per 128-byte K block);
// ELT = 1: e4m3 X, W with per-row scales (kind::f8f6f4, 128 elements per
// block; NEXT f4, the modern analogue of the paper's 16-bit storage P:264-268);
// ELT = 2: fp32 as 3xTF32 (kind::tf32, 32 elements per block): rows stored
// as [X_hi | X_hi | X_lo] and [W_hi | W_lo | W_hi], so the K = 3H product is
// X_hi W_hi + X_hi W_lo + X_lo W_hi (NEXT f2).
// ELT = 3: e4m3 X with per-row scales, MXFP4 W (E2M1 codes + one E8M0 scale
// per 32 K elements) on kind::mxf8f6f4.block_scale; 224-column tiles (TMEM
// holds the scales beside the accumulators, tc_epi.cuh). Each stage also
// carries the K block's W scale atoms covering the tile's rows (one bulk
// copy of up to 3 contiguous 128-row atoms); warp 10 (a control warp that
// was idle) re-bases them to the tile's first row (2 atoms, the layout
// tcgen05.cp reads), and the MMA thread copies those to TMEM before the
// stage's MMAs (NEXT f4).
template <int KB, int MODE, int NG, int ELT = 0>
__global__ void __launch_bounds__(TcCfg<NG>::kThreads, 1)
    ol_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                 const __grid_constant__ CUtensorMap tmWn, const TcParams p) {
  using Cfg = TcCfg<NG>;
  constexpr int kBBytes = ELT == 3 ? TC_B_BYTES_F4 : TC_B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + TC_STAGES * TC_A_BYTES;
  float* sbias = reinterpret_cast<float*>(sB + TC_STAGES * kBBytes);
  float* xch = sbias + TC_NBIAS * TC_BN;
  unsigned long long* thr_x = reinterpret_cast<unsigned long long*>(xch + 128 * TC_XCH_FLOATS);
  uint64_t* full = reinterpret_cast<uint64_t*>(thr_x + TC_THRX_BYTES / 8);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bfull + TC_NBIAS);
  // e4m3 column-scale ring, after the 512-byte barrier area (TC_SMEM_F8)
  float* sscale = (ELT == 1 && scale_ring_ok(p, TC_STAGES))
                      ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512)
                      : nullptr;
  // mxfp4 (TC_SMEM_F4): A's constant atom, the raw scale atoms
  // [TC_STAGES][TC_SF_RAW][512], the re-based ones [TC_STAGES][2][512]; the
  // re-based stages' barriers after the others in the barrier area
  uint8_t* ssfa = reinterpret_cast<uint8_t*>(full) + 512;
  uint8_t* ssf_raw = ssfa + TC_SF_ATOM;
  uint8_t* ssf = ssf_raw + TC_STAGES * TC_SF_RAW * TC_SF_ATOM;
  uint64_t* sfready = full + 40;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Warp roles: the epilogue warpgroups take the LOW warp ids and the control
  // warpgroup (TMA producer, MMA issuer, 2 idle) the highest ones: the warp
  // scheduler favours higher warp ids, so the single-thread producer/issuer
  // are not starved by the busy epilogue warps sharing their sub-partition.
  constexpr int kCtrl = 4 * NG;                    // first control warp
  const int role = warp - kCtrl;                   // 0 = TMA, 1 = MMA, 2-3 idle, < 0 epilogue

  // Programmatic dependent launch: the next launch in the stream may be
  // scheduled now (its CTAs still need this kernel's SMs to free up).
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && !p.pdl) tl_mark(p.tl, TL_ENTRY);
  for (int i = threadIdx.x; i < TC_THRX_BYTES / 8; i += blockDim.x)   // no stale tags
    sts_u64(smem_u32(thr_x + i), 0ull);
  if constexpr (ELT == 3) {
    // A's scales: 2^0 (E8M0 code 127) for every row and K block; X keeps its
    // per-row fp32 scale, applied in the epilogue. Written by the generic
    // proxy, read by tcgen05.cp (async proxy): fence before the barrier.
    for (int i = threadIdx.x; i < TC_SF_ATOM / 4; i += blockDim.x)
      reinterpret_cast<uint32_t*>(ssfa)[i] = 0x7F7F7F7Fu;
    fence_proxy_async_smem();
  }
  if (role == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    if (p.wnarrow) prefetch_tmap(&tmWn);
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], p.mc > 1 ? p.mc : 1);   // W multicast: every cluster CTA's MMAs
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], NG * 4);        // one arrival per epilogue warp
    }
    for (int i = 0; i < TC_NBIAS; ++i) mbar_init(&bfull[i], 1);
    if constexpr (ELT == 3)
      for (int i = 0; i < TC_STAGES; ++i) mbar_init(&sfready[i], 1);
    fence_barrier_init();
  }
  if (role == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if (p.mc > 1) cluster_sync();   // peers' barriers initialised before any multicast
  tc_fence_after();
  // (PDL) everything above touched only shared memory / TMEM / the kernel
  // parameters; wait for the previous grid in the stream (completion and
  // memory visibility) before any global memory access. (Issuing the first
  // W loads before this wait — W is read-only — gained 1.4 us for the fused
  // kernel alone at cfg greedy but nothing with the fused tail, and its code
  // in the producer cost the tail path 2.5 us at cfg beam even when off at
  // run time; removed.)
  if (p.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) tl_mark(p.tl, TL_ENTRY);
  }
  const uint32_t tmem_base = *tmem_holder;
  if constexpr (ELT == 3) {
    if (role == 1 && lane == 0) tmem_cp_sf(tmem_base + TC_SFA_COL, sdesc_rows16(smem_u32(ssfa)));
  }
  // this launch's tag (hints, tail counters): read by the epilogue threads
  // (the only users), off the TMA producer's path to its first load
  uint32_t gen = 0u;
  if (threadIdx.x == 0) tl_mark(p.tl, TL_SETUP);

  const TcDyn dyn = tc_dyn<false>(p);      // N (and the schedule) from the device in _dev mode
  // W multicast clusters (p.mc > 1): the mc CTAs of a cluster are the mc
  // M-tiles of ONE vocab split (aligned schedule), so they stream the same W
  // tiles in lockstep; the logical CTA index (ranges, record slots) is
  // M-tile * splits + split
  const uint32_t mc_rank = p.mc > 1 ? cluster_ctarank() : 0u;
  const long long cta = p.mc > 1 ? (long long)mc_rank * (dyn.sch.band / dyn.sch.C) + blockIdx.x / p.mc
                                 : (long long)blockIdx.x;
  const long long start = cta * dyn.sch.C;
  const long long stop = min(start + dyn.sch.C, dyn.sch.total);

  if (role >= 0) {
    reg_dealloc<Cfg::kCtrlRegs>();
    if (role == 0) {
      // ------------------------------------------------ TMA producer
      // The whole warp walks the schedule (keeps it converged); lane 0 issues.
      const uint64_t pol_x = policy_evict_last();     // X is re-read by every CTA
      TileIter it{start, stop, dyn.sch};
      it.taper = p.taper;
      if constexpr (ELT == 3) it.wmax = TC_BN_F4;
      int mt, v0, width;
      bool last;
      int stage = 0, tile = 0;
      uint32_t phase = 0;
      // TC_KBYTES of K per block: bf16 / e4m3 / fp32 (tf32x3) elements
      constexpr int kBlockElems = ELT == 1 || ELT == 3 ? TC_KBYTES : ELT == 2 ? TC_KBYTES / 4
                                                                               : TC_KBYTES / 2;
      int loads = 0;
      while (it.next(mt, v0, width, last)) {
        if (lane == 0) bias_ring_load(p, sbias, bfull, tile, v0, width, sscale);
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait_spin(&empty[stage], phase ^ 1);
          // (experiment p.mma_only, MODE 2: only the first TC_STAGES blocks are
          // loaded; later stages are marked full without a copy, so the MMAs
          // re-read stale data: the pipeline without TMA traffic)
          // (mma_only 2: only X is copied again, 3: only W; stale otherwise)
          const bool warm = MODE == 2 && p.mma_only && loads++ >= TC_STAGES;
          if (warm && p.mma_only == 1) {
            if (lane == 0) mbar_arrive(&full[stage]);
            __syncwarp();
            if (++stage == TC_STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          const bool load_x = !warm || p.mma_only == 2, load_w = !warm || p.mma_only == 3;
          if (lane == 0) {
            if (tile == 0 && kb == 0) tl_mark(p.tl, TL_TMA0);
            // W in boxes of p.wbox rows (256, or 64 so narrow tapered tiles
            // do not drag 256 rows through L2 -> SMEM); the boxes land
            // contiguously, i.e. the same SW128 K-major tile
            // a narrow tile (a range's remainder, <= 192 columns) loads only
            // the 64-row boxes it needs (tmWn), not a full 256-row box
            const bool narrow = p.wnarrow && width <= 192;
            const int wbox = narrow ? 64 : p.wbox;
            const int nbox = (width + wbox - 1) / wbox;
            const CUtensorMap* tw = narrow ? &tmWn : &tmW;
            // (mxfp4 W: the transaction counts the packed global bytes, half
            // the unpacked shared-memory box)
            constexpr int kWDiv = ELT == 3 ? 2 : 1;
            // mxfp4: this K block's 128-row scale atoms covering the tile's
            // rows, contiguous in the [kblock][row / 128][512] layout
            const int nb128 = (p.V_local + 127) / 128;
            const int nsf = ELT == 3 ? min(((v0 & 127) + width - 1) / 128 + 1, nb128 - v0 / 128) : 0;
            mbar_arrive_expect_tx(&full[stage], (load_x ? p.a_box_bytes : 0) +
                                                    (load_w ? nbox * wbox * TC_KBYTES / kWDiv : 0) +
                                                    (ELT == 3 && load_w ? nsf * TC_SF_ATOM : 0));
            if constexpr (ELT == 3) {
              AMUN_DCHECK(v0 % TC_F4_ALIGN == 0 && nsf >= 1 && nsf <= TC_SF_RAW);
              if (load_w)
                bulk_load(ssf_raw + stage * TC_SF_RAW * TC_SF_ATOM,
                          p.w_sf + ((long long)kb * nb128 + v0 / 128) * TC_SF_ATOM,
                          nsf * TC_SF_ATOM, &full[stage]);
            }
            if (load_x)
              tma_load_2d(&tmX, &full[stage], sA + stage * TC_A_BYTES, kb * kBlockElems, mt * TC_BM,
                          pol_x);
            if (p.mc > 1) {
              // this CTA's box of the W tile, multicast to the whole cluster
              for (int j = (int)mc_rank; load_w && j < nbox; j += p.mc)
                tma_load_2d_mc(&tmW, &full[stage], sB + stage * kBBytes + j * wbox * TC_KBYTES,
                               kb * kBlockElems, v0 + j * wbox, (uint16_t)((1u << p.mc) - 1u));
            }
            for (int j = 0; load_w && p.mc <= 1 && j < nbox; ++j) {
              // (the L2 hint measured the same as evict_first / evict_normal / none)
              tma_load_2d(tw, &full[stage], sB + stage * kBBytes + j * wbox * TC_KBYTES,
                          kb * kBlockElems, v0 + j * wbox, 0ull);
            }
          }
          __syncwarp();
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ++tile;
      }
    } else if (role == 1) {
      // ------------------------------------------------ MMA issuer
      // The whole warp waits; lane 0 issues tcgen05.mma and the commits (a
      // commit tracks the MMAs issued by the same thread).
      TileIter it{start, stop, dyn.sch};
      it.taper = p.taper;
      if constexpr (ELT == 3) it.wmax = TC_BN_F4;
      int mt, v0, width;
      bool last;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int mtile = 0;
      while (it.next(mt, v0, width, last)) {
        mbar_wait_spin(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0 && mtile < TL_N - TL_MMA0) tl_mark(p.tl, TL_MMA0 + mtile);
        ++mtile;
        const uint32_t d = tmem_base + acc * TC_BN;
        const uint32_t idesc = ELT == 1 ? idesc_e4m3_f32(TC_BM, width)
                             : ELT == 2 ? idesc_tf32_f32(TC_BM, width)
                                        : idesc_bf16_f32(TC_BM, width);
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait_spin(&full[stage], phase);
          if constexpr (ELT == 3) mbar_wait_spin(&sfready[stage], phase);   // re-based scales
          tc_fence_after();
          if (lane == 0) {
            if (kb == 0 && mtile == 1) tl_mark(p.tl, TL_FULL0);
            const uint64_t ad = sdesc_k<TC_KBYTES>(smem_u32(sA + stage * TC_A_BYTES));
            const uint64_t bd = sdesc_k<TC_KBYTES>(smem_u32(sB + stage * kBBytes));
            uint32_t sfb = 0;
            if constexpr (ELT == 3) {   // this stage's W scales -> TMEM (ordered before the MMAs)
              sfb = tmem_base + tc_sfb_col(stage);
              const uint32_t s0 = smem_u32(ssf + stage * 2 * TC_SF_ATOM);
              tmem_cp_sf(sfb, sdesc_rows16(s0));
              if (width > 128) tmem_cp_sf(sfb + 4, sdesc_rows16(s0 + TC_SF_ATOM));
            }
#pragma unroll
            for (int k = 0; k < TC_KBYTES / 32; ++k) {   // +32 bytes of K per MMA (>>4 = 2)
              if constexpr (ELT == 0)
                mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
              else if constexpr (ELT == 1)
                mma_e4m3(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
              else if constexpr (ELT == 3)   // K step k uses byte k of each scale word
                mma_mxf4(d, ad + 2 * k, bd + 2 * k, idesc_mxf4_f32(TC_BM, width, k, k),
                         (tmem_base + TC_SFA_COL) | ((uint32_t)k << 30), sfb | ((uint32_t)k << 30),
                         (kb | k) != 0);
              else
                mma_tf32(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            }
            if (p.mc > 1)   // the slot is free in every cluster CTA once all their MMAs finish
              mma_commit_mc(&empty[stage], (uint16_t)((1u << p.mc) - 1u));
            else
              mma_commit(&empty[stage]);            // smem slot free once these MMAs finish
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
      if (lane == 0) tl_mark(p.tl, TL_MMA_END);
    } else if (ELT == 3 && role == 2) {
      // ------------------------------------------------ mxfp4 scale re-basing
      // Per stage: the raw atoms hold rows 128 a + (0..383) of the K block's
      // scales (a = v0 / 128); the tile's row n = 32 b + n' (b = (v0 % 128) /
      // 32) goes to re-based atom n / 128, row n % 32, word (n / 32) % 4.
      // Lane m0 moves the 8 words of rows m0 + 32 j, j < 8.
      TileIter it{start, stop, dyn.sch};
      it.wmax = TC_BN_F4;
      int mt, v0, width;
      bool last;
      int stage = 0;
      uint32_t phase = 0;
      while (it.next(mt, v0, width, last)) {
        const int b = (v0 & 127) >> 5;
        for (int kb = 0; kb < p.n_kblk; ++kb) {
          mbar_wait_spin(&full[stage], phase);
          const uint32_t* raw =
              reinterpret_cast<const uint32_t*>(ssf_raw + stage * TC_SF_RAW * TC_SF_ATOM);
          uint32_t* dst = reinterpret_cast<uint32_t*>(ssf + stage * 2 * TC_SF_ATOM);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int g = b + j;   // 32-row group of the raw atoms
            dst[(j >> 2) * (TC_SF_ATOM / 4) + 4 * lane + (j & 3)] =
                raw[(g >> 2) * (TC_SF_ATOM / 4) + 4 * lane + (g & 3)];
          }
          fence_proxy_async_smem();   // generic writes -> tcgen05.cp (async proxy)
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfready[stage]);
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    reg_alloc<Cfg::kEpiRegs>();
    if constexpr (MODE == 0 || MODE == 4) {
      gen = read_generation(p.gen_ctr);
      // the next launch's tail counter (tail.cuh "Counters")
      if (blockIdx.x == 0 && threadIdx.x == 0) p.arrive[(gen + 1u) & 1u] = 0u;
    }
    tc_epilogue<KB, MODE, NG, false, ELT>(p, tmem_base, start, stop, tfull, tempty, bfull, sbias, xch,
                                     thr_x, gen, warp, lane, 0u, cta, dyn, sscale);
    if (threadIdx.x == 0) tl_mark(p.tl, TL_EPI_END);
    if constexpr (MODE == 0 || MODE == 4) {
      // The merge in this launch (tail.cuh), run by the epilogue warps INSIDE
      // their branch: code after the roles rejoin is register-allocated for
      // the control warps' setmaxnreg budget (56), where the merge spilled.
      // The barrier orders every epilogue warp's partial records (and its
      // use of the exchange area) before the CTA's arrival.
      if (p.tail) {
        tc_fence_before();
        named_bar_sync(11, Cfg::kEpiThreads);
        if (threadIdx.x == 0) tl_mark(p.tl, TL_BARRIER);
        grid_tail<KB>(p, dyn, reinterpret_cast<uint8_t*>(xch), gen);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (p.mc > 1) cluster_sync();   // no CTA leaves while peers may still signal into it
  if (threadIdx.x == 0 && !p.tail) tl_mark(p.tl, TL_BARRIER);
  if (role == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
  if constexpr (MODE == 0 || MODE == 4) {
    if (!p.tail && threadIdx.x == 0) finish_generation(p.gen_ctr);
  }
}

}  // namespace amun
