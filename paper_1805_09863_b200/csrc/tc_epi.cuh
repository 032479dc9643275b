// tc_epi.cuh — the epilogue of the fused tcgen05 kernels (steps 2-4 on the
// TMEM accumulator), shared by the single-CTA and the CTA-pair kernels.
//
// NG epilogue warpgroups; warp (grp, q) owns TMEM lane quadrant q (rows
// 32q..32q+31 of the CTA's M-tile) and the 32-column chunks c = grp,
// grp + NG, ... of every tile. Thread = hypothesis row. Per chunk:
// tcgen05.ld of 32 fp32 columns, + bias (from the shared-memory ring the TMA
// producer fills), online max / sum-of-exp (Alg. 4 with the exp(Delta)
// rescale), and the gated register k-best (RowState::chunk32r).
// After each tile: publish / refresh the cross-CTA k-th-best hint. At the end
// of a CTA's range in an M-tile the NG groups' states are combined in NG-1
// rounds through one exchange area and group 0 writes the partial record.
#pragma once
#include "merge.cuh"
#include "peer.cuh"

namespace amun {

struct TcParams {
  int N, V_local, v_offset, n_kblk;
  Schedule sch;
  const float* __restrict__ bias;
  float* __restrict__ part;   // [slots][128][stride]
  int stride, k_max;
  float* __restrict__ logits; // MODE 1: [N][V_local]
  unsigned long long* __restrict__ hint;   // [N] cross-CTA k-th-best hints
  int use_hint;                            // 0: CTA ranges too short to profit from them
  unsigned int* __restrict__ gen_ctr;      // {generation, CTAs done}: device-side, so every
                                           // launch (graph replays too) gets a fresh tag
  const int* __restrict__ N_dev;           // amun_output_layer_dev: N on the device (else NULL)
  const float* __restrict__ x_scale;       // e4m3 plans: [N] per-row scales of X (else NULL)
  const float* __restrict__ w_scale;       // e4m3 plans: [V_local] per-row scales of W
  const uint8_t* __restrict__ w_sf;        // mxfp4 plans: W's E8M0 block scales, atom layout
                                           // [V_local/128][n_kblk][512] (amun.h)
  int a_box_bytes;                         // bytes of one X box (rows x 128; single-CTA kernel)
  int num_sms;                             // the device schedule's CTA count
  // Fused tail (tail.cuh): after every CTA of the grid has emitted its
  // partial records, the epilogue warps of all CTAs run the merge, so the
  // whole path is ONE launch. TAIL_NONE leaves the records in the workspace
  // (amun_ol_scores; a separate merge kernel follows).
  int tail;                                // TAIL_NONE / TAIL_SENT / TAIL_ROWS / TAIL_ARGMAX
  MergeParams mp;                          // the merge's parameters (outputs, offsets, ...)
  unsigned int* __restrict__ arrive;       // [2] tail arrival counters, by tag parity (tail.cuh)
  unsigned long long* __restrict__ tl;     // timeline probe [grid][TL_N] (amun_debug_timeline), else NULL
  OneShotTail os;                          // TAIL_ONESHOT: the peer buffers (peer.cuh)
  int taper;                               // single-CTA kernel: narrow final tiles (TileIter)
  int prepass;                             // k-best bound pre-pass over a segment's first n tiles
  int wbox;                                // W rows per TMA box (single-CTA kernel: 256 or 64)
  int pdl;                                 // launched with programmatic stream serialization
  int mma_only;                            // (experiment, MODE 2) MMAs re-read the first stages
  int mc;                                  // > 1: clusters of mc M-tile CTAs share W (multicast)
  int wnarrow;                             // single-CTA kernel: narrow tiles load 64-row W boxes
};

// Timeline probe points (globaltimer ns; per CTA; see amun_debug_timeline).
enum { TL_ENTRY = 0, TL_SETUP = 1, TL_TMA0 = 2, TL_FULL0 = 3, TL_MMA_END = 4, TL_EPI_LAST = 5,
       TL_EPI_END = 6, TL_BARRIER = 7, TL_RELEASED = 8, TL_TAIL_END = 9, TL_TILE0 = 10,
       TL_MMA0 = 24, TL_N = 40 };
__device__ __forceinline__ void tl_mark(const unsigned long long* tl_base, int point) {
  if (tl_base) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const_cast<unsigned long long*>(tl_base)[(long long)blockIdx.x * TL_N + point] = t;
  }
}
enum { TAIL_NONE = 0, TAIL_SENT = 1, TAIL_ROWS = 2, TAIL_ARGMAX = 3, TAIL_ONESHOT = 4,
       TAIL_X_NOWORK = 16, TAIL_X_NOCOOP = 32,      // experiment flags (env AMUN_TAIL)
       TAIL_X_FENCE = 64, TAIL_X_SLEEP = 128 };

// Per-launch values that amun_output_layer_dev only knows on the device:
// the row count, the schedule derived from it and the hint switch.
struct TcDyn {
  int N, use_hint;
  Schedule sch;
};
template <bool PAIR>
__device__ __forceinline__ TcDyn tc_dyn(const TcParams& p) {
  TcDyn d{p.N, p.use_hint, p.sch};
  if (p.N_dev) {
    d.N = max(0, min(*p.N_dev, p.N));      // p.N = max_rows
    const int unit = PAIR ? 2 * 128 : 128;  // rows per schedule unit (a CTA pair: 256)
    d.sch = schedule_for((max(d.N, 1) + unit - 1) / unit, p.sch.Vp, PAIR ? p.num_sms / 2 : p.num_sms);
    if (d.N == 0) d.sch.total = 0;          // nothing to do: every CTA range is empty
    d.use_hint = d.sch.C >= 4 * 256 ? 1 : 0;
  }
  return d;
}

constexpr int TC_BM = 128;
#ifndef TC_BN_OVERRIDE
constexpr int TC_BN = 256;
#else
constexpr int TC_BN = TC_BN_OVERRIDE;
#endif
constexpr int TC_BK = 64;                            // bf16 elements per K block (pair kernel)
#ifndef TC1_KBYTES   // 64 (SW64, 8 stages) measured 1.3x slower per tile at cfg beam
#define TC1_KBYTES 128
#endif
constexpr int TC_KBYTES = TC1_KBYTES;                 // bytes of K per block, single-CTA kernel
constexpr int TC_NBIAS = 10;                         // bias ring slots (see producer bound)
constexpr int TC_BIAS_BYTES = TC_NBIAS * TC_BN * 4;
constexpr int TC_XCH_FLOATS = 2 + 2 * 16;            // one row's state in the exchange area
constexpr int TC_XCH_BYTES = 128 * TC_XCH_FLOATS * 4;
#if defined(AMUN_WITH_NG3) || defined(AMUN_WITH_NG4)
constexpr int TC_THRX_BYTES = 4 * 128 * 8;           // per-(group, row) k-th-best words (NG <= 4)
#else
constexpr int TC_THRX_BYTES = 2 * 128 * 8;           // per-(group, row) k-th-best words (NG = 2)
#endif
// e4m3 column-scale ring. 4 slots suffice when a tile has more K blocks than
// pipeline stages: the producer can only start tile t after the MMA started
// tile t-1, which needed the epilogue of tile t-3 to have released its
// accumulator, so tile t-4's slot is no longer read. Otherwise (small H) the
// epilogue reads the scales from global memory.
constexpr int TC_NSCALE = 4;
constexpr int TC_SCALE_BYTES = TC_NSCALE * TC_BN * 4;
// MXFP4 plans (ELT 3). The block-scaled MMA costs about the same per
// instruction at N = 128 as at N = 256 (bare GEMM at cfg beam 93 vs 51 us),
// so tiles stay wide: TC_BN_F4 = 224 columns, the two accumulators in TMEM
// columns [0, 224) and [256, 480), the scales in the 64 columns left: A's
// (constant 1.0, written once) at TC_SFA_COL, B's of pipeline stage s (two
// 512-byte atoms = 256 rows, 8 columns) at tc_sfb_col(s). Tiles start on
// 32-row boundaries (schedule_for align 32): the stage's atoms are re-based
// to the tile's first row in shared memory by a helper warp (the MMA's
// scale address can only move in 64-row steps).
constexpr int TC_BN_F4 = 224;
constexpr int TC_F4_ALIGN = 32;
constexpr int TC_SF_ATOM = 512;
constexpr int TC_SF_RAW = 3;   // 128-row atoms a stage's tile rows can touch
constexpr uint32_t TC_SFA_COL = 224;
__host__ __device__ constexpr uint32_t tc_sfb_col(int stage) {
  return stage < 3 ? 228u + 8u * (uint32_t)stage : 480u + 8u * (uint32_t)(stage - 3);
}

// Launch configuration of NG epilogue warpgroups (warps 0 .. 4NG-1) + the
// control warpgroup (TMA producer warp, MMA warp, 2 idle warps), and the setmaxnreg budget,
// which only redistributes the CTA's launch register pool (a warpgroup can
// grow only into what the others released, else setmaxnreg.inc blocks).
template <int NG>
struct TcCfg {
  static_assert(NG * 128 * 8 <= TC_THRX_BYTES, "thr_x area too small for NG epilogue groups");
  static constexpr int kEpiThreads = NG * 128;
  static constexpr int kThreads = 128 + kEpiThreads;
  static constexpr int kLaunchRegs = 65536 / kThreads / 8 * 8 > 248 ? 248 : 65536 / kThreads / 8 * 8;
  static constexpr int kCtrlRegs = NG >= 4 ? 32 : 56;
  static constexpr int kEpiRegs0 = (kLaunchRegs * kThreads - 128 * kCtrlRegs) / kEpiThreads / 8 * 8;
  static constexpr int kEpiRegs = kEpiRegs0 > 248 ? 248 : kEpiRegs0;
  static_assert(128 * kCtrlRegs + kEpiThreads * kEpiRegs <= kLaunchRegs * kThreads,
                "setmaxnreg budget exceeds the launch register pool");
};

// Read the launch generation (all CTAs, before any of them finishes).
__device__ __forceinline__ uint32_t read_generation(const unsigned int* gen_ctr) {
  return 1u + *reinterpret_cast<const volatile unsigned int*>(gen_ctr);
}
// Called once per CTA after all its work: the last CTA advances the generation.
// No fences: every CTA read the generation at its start, long before the last
// one finishes, and the next launch sees the new value (and the reset count)
// across the kernel boundary; a fence here only delayed each CTA's exit
// behind its partial-record stores (ncu: ~6% of greedy's stall samples).
// atomicInc wraps the count to 0 at the last CTA itself, so a count left at
// any value (e.g. by a caller reusing memory) heals after one launch.
__device__ __forceinline__ void finish_generation(unsigned int* gen_ctr) {
  const unsigned int prev = atomicInc(gen_ctr + 1, gridDim.x - 1);
  if (prev == gridDim.x - 1) atomicAdd(gen_ctr, 1u);   // every CTA has read the generation
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Producer side of the bias ring: slot (tile % TC_NBIAS) receives the tile's
// bias (its 16-byte-aligned part; a <= 3-float tail is read from global).
// The producer runs at most 2 + ceil(STAGES / n_kblk) - 1 <= 2 + STAGES tiles
// ahead of the slowest epilogue warp (the MMA cannot start tile t+2 before
// every epilogue warp released tile t), so TC_NBIAS >= 2 + STAGES suffices.
__device__ __forceinline__ void bias_ring_load(const TcParams& p, float* sbias, uint64_t* bfull,
                                               int tile, int v0, int width,
                                               float* sscale = nullptr) {
  const int slot = tile % TC_NBIAS;
  const int limit = min(width, p.V_local - v0);
  const uint32_t bytes = (uint32_t)(limit & ~3) * 4u;
  mbar_arrive_expect_tx(&bfull[slot], sscale ? 2 * bytes : bytes);
  if (bytes) {
    bulk_load(sbias + slot * TC_BN, p.bias + v0, bytes, &bfull[slot]);
    // e4m3: the column scales ride along, into the 4-slot scale ring
    // (safe when n_kblk > STAGES, see scale_ring_ok), completing on bfull too
    if (sscale) bulk_load(sscale + (tile % TC_NSCALE) * TC_BN, p.w_scale + v0, bytes, &bfull[slot]);
  }
}

// The epilogue. PAIR: the CTA is rank `rank` of a CTA pair (its M-tile is
// 2 mp + rank of the pair schedule; TMEM-empty arrivals go to the leader).
__device__ __forceinline__ bool scale_ring_ok(const TcParams& p, int stages) {
  return p.n_kblk > stages;
}

template <int KB, int MODE, int NG, bool PAIR, int ELT = 0>
__device__ __forceinline__ void tc_epilogue(const TcParams& p, uint32_t tmem_base, long long start,
                                            long long stop, uint64_t* tfull, uint64_t* tempty,
                                            uint64_t* bfull, const float* sbias, float* xch,
                                            unsigned long long* thr_x, uint32_t gen, int warp,
                                            int lane, uint32_t rank, long long slot_base,
                                            const TcDyn dyn, const float* sscale = nullptr) {
  const int grp = warp >> 2;                       // epilogue warps are 0 .. 4NG-1
  const int q = warp & 3;                          // TMEM lane quadrant of this warp
  const int row_local = q * 32 + lane;
  const uint32_t t_lane = (uint32_t)(q * 32) << 16;
  uint32_t tempty_addr[2];
  if constexpr (PAIR) {
    tempty_addr[0] = mapa_shared(smem_u32(&tempty[0]), 0);
    tempty_addr[1] = mapa_shared(smem_u32(&tempty[1]), 0);
  }
  RowState<KB> st;
  st.reset();
  TileIter it{start, stop, dyn.sch};
  it.taper = PAIR ? 0 : p.taper;
  if constexpr (ELT == 3) it.wmax = TC_BN_F4;
  int unit, v0, width;
  bool last;
  int acc = 0, tile = 0;
  uint32_t acc_phase = 0;
  float hintv = kNegInf, published = kNegInf;
  // The groups of a CTA hold disjoint chunks of the same rows: each publishes
  // its k-th best in shared memory (tagged with the M-tile, so a word from an
  // earlier segment is never used) and gates with the best of all groups.
  unsigned long long* my_thr = thr_x + grp * 128 + row_local;
  float shared_kth = kNegInf;
  // Pre-pass bound (first tile of a segment, when the row lists are empty and
  // every chunk would pass the k-best gate): the KB-th largest group maximum
  // over this group's chunks of the tile. KB distinct elements reach it, so
  // nothing below it can be in the row's top-KB (the same argument as the
  // list-filling bound of kbest32 and reading G15); ties at it are kept.
  float pre = kNegInf;
  int seg_tile = 0;   // tiles of the current segment processed so far
  while (it.next(unit, v0, width, last)) {
    const int mt = PAIR ? 2 * unit + (int)rank : unit;
    const uint32_t tag = (uint32_t)mt + 1u;
    const int row = mt * TC_BM + row_local;
    // warp-uniform: this warp's 32 rows hold at least one real row (N <= 96
    // leaves whole lane quadrants, and a pair's padding M-tile all four, idle)
    const bool live = mt * TC_BM + q * 32 < dyn.N;
    const int limit = min(width, p.V_local - v0);
    const int nch = (width + 31) >> 5;
    const float* bsl = sbias + (tile % TC_NBIAS) * TC_BN;
    const float xs = ((ELT == 1 || ELT == 3) && row < dyn.N) ? __ldg(p.x_scale + row)
                                                              : 1.f;   // e4m3 row scale
    // request the newest cross-CTA hint now (L2, not L1: other SMs update it);
    // it is folded in after this tile's chunks, for the next tile of the segment
    // (per-chunk exchange halves the insertions but its loads and atomics cost
    // as much as it saves: DESIGN.md §6.1)
    unsigned long long hraw = 0ull;
    if ((MODE == 0 || MODE == 4) && dyn.use_hint && row < dyn.N && !last) hraw = __ldcg(p.hint + row);
    mbar_wait(&bfull[tile % TC_NBIAS], (uint32_t)(tile / TC_NBIAS) & 1u);
    mbar_wait(&tfull[acc], acc_phase);
    tc_fence_after();
    if (warp == 0 && lane == 0 && p.tl) {
      if (tile < TL_N - TL_TILE0) tl_mark(p.tl, TL_TILE0 + tile);
      tl_mark(p.tl, TL_EPI_LAST);
    }
    const uint32_t tbase = tmem_base + t_lane + acc * TC_BN;
    // biased (and, e4m3, scaled) logits of 32-column chunk c from its TMEM words
    auto build_x = [&](const uint32_t (&r)[32], int c, float (&x)[32]) {
      const int c0 = c * 32;
      const int nv = limit - c0;
      if (nv >= 32) {   // full chunk: bias from the ring (same address in all lanes)
        const uint32_t b4 = smem_u32(bsl + c0);
        if constexpr (ELT == 3) {   // mxfp4 W (block scales inside the MMA): acc * x_scale + b
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bq = lds128(b4 + 16 * j);
            ffma2(x[4 * j + 0], x[4 * j + 1], __uint_as_float(r[4 * j + 0]),
                  __uint_as_float(r[4 * j + 1]), xs, xs, bq.x, bq.y);
            ffma2(x[4 * j + 2], x[4 * j + 3], __uint_as_float(r[4 * j + 2]),
                  __uint_as_float(r[4 * j + 3]), xs, xs, bq.z, bq.w);
          }
        } else if constexpr (ELT != 1) {   // bf16 / tf32x3: + bias
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bq = lds128(b4 + 16 * j);
            fadd2(x[4 * j + 0], x[4 * j + 1], __uint_as_float(r[4 * j + 0]),
                  __uint_as_float(r[4 * j + 1]), bq.x, bq.y);
            fadd2(x[4 * j + 2], x[4 * j + 3], __uint_as_float(r[4 * j + 2]),
                  __uint_as_float(r[4 * j + 3]), bq.z, bq.w);
          }
        } else {
          // e4m3: logit = acc * (x_scale[row] * w_scale[v]) + b[v]; the 32
          // column scales (the same for every lane) from the scale ring,
          // else an L1-broadcast global load (small H, see scale_ring_ok)
          const float4* ws4 = reinterpret_cast<const float4*>(p.w_scale + v0 + c0);
          const uint32_t s4 = sscale ? smem_u32(sscale + (tile % TC_NSCALE) * TC_BN + c0) : 0u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bq = lds128(b4 + 16 * j);
            const float4 wq = sscale ? lds128(s4 + 16 * j) : __ldg(ws4 + j);
            float s0, s1, s2, s3;
            fmul2(s0, s1, wq.x, wq.y, xs, xs);
            fmul2(s2, s3, wq.z, wq.w, xs, xs);
            ffma2(x[4 * j + 0], x[4 * j + 1], __uint_as_float(r[4 * j + 0]),
                  __uint_as_float(r[4 * j + 1]), s0, s1, bq.x, bq.y);
            ffma2(x[4 * j + 2], x[4 * j + 3], __uint_as_float(r[4 * j + 2]),
                  __uint_as_float(r[4 * j + 3]), s2, s3, bq.z, bq.w);
          }
        }
      } else {          // vocabulary tail: mask, and the unstaged <= 3-float bias tail
        const int nv4 = (limit & ~3) - c0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float bj = (j < nv4) ? bsl[c0 + j] : ((j < nv) ? __ldg(p.bias + v0 + c0 + j) : 0.f);
          if constexpr (ELT == 3) {
            x[j] = (j < nv) ? fmaf(__uint_as_float(r[j]), xs, bj) : kNegInf;
          } else if constexpr (ELT != 1) {
            x[j] = (j < nv) ? __uint_as_float(r[j]) + bj : kNegInf;
          } else {
            const float sj = (j < nv) ? xs * __ldg(p.w_scale + v0 + c0 + j) : 0.f;
            x[j] = (j < nv) ? fmaf(__uint_as_float(r[j]), sj, bj) : kNegInf;
          }
        }
      }
    };
    if constexpr (MODE == 0 && KB > 1) {
      if (live && seg_tile < p.prepass) {
        float top[KB];
#pragma unroll
        for (int i = 0; i < KB; ++i) top[i] = kNegInf;
        for (int c = grp; c < nch; c += NG) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          float x[32];
          tmem_ld_wait(r);
          build_x(r, c, x);
          float g[8];
          RowState<KB>::groups32(x, g);
#pragma unroll
          for (int j = 0; j < 8; ++j) {   // insert g[j] into the descending top[]
            float t = g[j];
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              const float hi = fmaxf(top[i], t);
              t = fminf(top[i], t);
              top[i] = hi;
            }
          }
        }
        if (top[KB - 1] > pre) {   // bounds only rise within a segment
          pre = top[KB - 1];
          sts_u64(smem_u32(my_thr), ((unsigned long long)tag << 32) | f2o(fmaxf(pre, st.l[KB - 1])));
        }
      }
    }
    if (live) {
      for (int c = grp; c < nch; c += NG) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        const int c0 = c * 32;
        const int nv = limit - c0;
        float x[32];
        tmem_ld_wait(r);
        build_x(r, c, x);
        if constexpr (MODE == 1) {
          if (row < dyn.N) {
            float* out = p.logits + (long long)row * p.V_local + v0 + c0;
            for (int j = 0; j < 32 && j < nv; ++j) out[j] = x[j];
          }
        } else if constexpr (MODE == 2) {
          uint32_t a = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) a ^= r[j];
          st.s += __uint_as_float(a & 0x007fffffu);   // keep the loads alive
        } else if constexpr (MODE == 3) {
          st.template chunk32r<false>(x, p.v_offset + v0 + c0, hintv);
        } else {
#pragma unroll
          for (int g2 = 0; g2 < NG; ++g2) {
            if (g2 != grp && AMUN_EXP != 3) {
              const unsigned long long w = lds_u64(smem_u32(thr_x + g2 * 128 + row_local));
              if ((uint32_t)(w >> 32) == tag) shared_kth = fmaxf(shared_kth, o2f((uint32_t)w));
            }
          }
          const float before = st.l[KB - 1];
          st.template chunk32r<true, MODE != 4>(x, p.v_offset + v0 + c0,
                                                fmaxf(fmaxf(hintv, shared_kth), pre));
          if (AMUN_EXP != 3 && st.l[KB - 1] > before && st.l[KB - 1] > pre)
            sts_u64(smem_u32(my_thr), ((unsigned long long)tag << 32) | f2o(st.l[KB - 1]));
        }
      }
    }
    tc_fence_before();
    if constexpr (PAIR) {
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr[acc]);
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if ((MODE == 0 || MODE == 4) && dyn.use_hint && row < dyn.N && !last) {
      // publish our k-th best only if it beats what is already known (with
      // many CTAs per row, e.g. one M-tile over 148 CTAs, unconditional
      // atomics would serialise on the row's word); never after the segment's
      // last tile (the other CTAs of the row are finishing too)
      if (AMUN_EXP != 3 && st.l[KB - 1] > published && st.l[KB - 1] > hintv) {
        published = st.l[KB - 1];
        atomicMax(p.hint + row, hint_encode(published, gen));
      }
      hintv = fmaxf(hintv, hint_decode(hraw, gen));   // 0 (no hint) when `last`
    }
    ++seg_tile;
    if (last) {
      hintv = kNegInf;   // the next segment is another M-tile (other rows)
      published = kNegInf;
      shared_kth = kNegInf;
      pre = kNegInf;
      seg_tile = 0;
      if constexpr (MODE != 1) {
        float* xr = xch + row_local * TC_XCH_FLOATS;
        for (int g = 1; g < NG; ++g) {
          if (grp == g) {
            xr[0] = st.m;
            xr[1] = st.s;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              xr[2 + i] = st.l[i];
              xr[2 + 16 + i] = __int_as_float(st.v[i]);
            }
          }
          named_bar_sync(1 + q, NG * 32);
          if (grp == 0) {
            float l2[KB];
            int v2[KB];
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              l2[i] = xr[2 + i];
              v2[i] = __float_as_int(xr[2 + 16 + i]);
            }
            st.combine(xr[0], xr[1], l2, v2);
          }
          named_bar_sync(5 + q, NG * 32);
        }
        if (grp == 0 && row < dyn.N) {
          const long long slot = PAIR ? (slot_base + unit) * 2 + rank : slot_base + unit;
          AMUN_DCHECK(p.mp.part_floats == 0 ||
                      (slot * TC_BM + row_local + 1) * p.stride <= p.mp.part_floats);
          st.emit(p.part + (slot * TC_BM + row_local) * p.stride, p.k_max);
        }
      }
      st.reset();
    }
    acc ^= 1;
    if (acc == 0) acc_phase ^= 1;
    ++tile;
  }
}

}  // namespace amun
