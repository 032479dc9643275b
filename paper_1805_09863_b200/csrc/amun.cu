// amun.cu — host side of the C-ABI declared in include/amun.h.
// Validation, persistent-grid schedule, TMA tensor-map cache and launches.
// No device memory is allocated here and no stream is synchronised (except
// amun_compact with counts_host).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "../../include/amun.h"
#include "compact.cuh"
#include "merge.cuh"
#include "ol_simt.cuh"
#include "launch_tc.cuh"
#include "tail.cuh"
#include "oneshot.cuh"
#include "quant.cuh"

using namespace amun;

namespace {

thread_local std::string g_err;

amun_status fail(amun_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

}  // namespace

amun_status amun::launch_fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return AMUN_ECUDA;
}

namespace {

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(AMUN_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));          \
  } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapEntry {
  const void* ptr = nullptr;
  long long rows = -1;
  int box_rows = 0;
  int kbytes = 0;
  CUtensorMap map;
};

// k-best capacity buckets compiled into the kernels (a row keeps exactly
// kbucket(k_max) >= k_max entries; smaller = fewer insertions).
inline int kbucket(int k) {
  return k <= 6 ? (k < 1 ? 1 : k) : k <= 8 ? 8 : k <= 12 ? 12 : 16;
}
#define AMUN_KB_SWITCH(kb, CALL) \
  switch (kb) {                  \
    case 1: return CALL(1);      \
    case 2: return CALL(2);      \
    case 3: return CALL(3);      \
    case 4: return CALL(4);      \
    case 5: return CALL(5);      \
    case 6: return CALL(6);      \
    case 8: return CALL(8);      \
    case 12: return CALL(12);    \
    default: return CALL(16);    \
  }
inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace

struct amun_ol {
  int H, V_local, v_offset, V_total, k_max, kb, max_rows, max_sentences, device, num_sms;
  amun_dtype dtype;
  int stride;
  size_t ws_bytes;
  size_t slots_bytes;          // partial-record slots at the start of the workspace
  size_t hint_bytes;               // per-row hint words after the slots, then 2 x u32
                                   // {generation, CTAs done} (device-side counters)
  size_t flags_bytes;              // (reserved after the counters; 0)
  const void* hint_ws = nullptr;   // workspace whose hint / counter / flag region is initialised
  int tail_mode = 0;    // env AMUN_TAIL: 0 fused tail (one launch per call), 1 "off" (separate merge kernel)
  unsigned long long* tl = nullptr;   // amun_debug_timeline buffer (device), else NULL
  int ng_override = 0;  // env AMUN_NG: 2 or 4 epilogue warpgroups (experiments)
  int taper = 0;        // env AMUN_TAPER=1: narrow final tiles (experiments; measured slower:
                        // less W in flight per SM in the narrow tiles)
  int prepass = 1;      // env AMUN_PREPASS=n: the k-best bound pre-pass on a segment's first n
                        // tiles (0 = off; experiments)
  int wbox = 256;       // env AMUN_WBOX: W rows per TMA box, 256 or 64 (64 for tapered tiles)
  int mma_only = 0;     // (amun_bench_variant 5: the MMA issue rate alone)
  int mc = 0;           // env AMUN_MC: W multicast cluster size (experiment; ol_tc.cuh)
  int wnarrow = 1;      // env AMUN_WNARROW=0: remainder tiles load full 256-row W boxes
  int pdl = 1;          // env AMUN_PDL=0: no programmatic dependent launch of the fused kernel
                        // (single-CTA kernel; greedy path 20.7 -> 19.7 us)
  int pairs_mode = 0;   // env AMUN_PAIRS: 0 auto, 1 never ("off"), 2 always ("force"; tests)
  MapEntry xmaps[4];
  MapEntry wmaps[16];   // (two maps per W: 256- and 64-row boxes)
  int xnext = 0, wnext = 0;
};

namespace {

// Tensor map of a row-major [rows, H] bf16 matrix, box [box_rows, 64],
// 128-byte swizzle (matches sdesc_k_sw128), OOB rows/columns read as zero.
amun_status encode_map(amun_ol* pl, const void* ptr, long long rows, int box_rows, int kbytes,
                       bool is_w, CUtensorMap* out) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(AMUN_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  // box rows of `kbytes` bytes (128: 64 bf16, 128 e4m3 codes or 32 fp32 of the
  // 3H-wide tf32x3 rows; 64: half of that), swizzled to match sdesc_k<kbytes>.
  // MXFP4 W: packed E2M1 pairs in HBM (H/2 bytes per row); the 16U4_ALIGN16B
  // type spreads each 8 bytes (16 codes) over 16 bytes of shared memory, the
  // layout kind::mxf8f6f4 reads, so a box of 128 codes fills 128 bytes.
  const bool f4 = pl->dtype == AMUN_MXFP4 && is_w;
  const bool f8 = pl->dtype == AMUN_E4M3 || (pl->dtype == AMUN_MXFP4 && !is_w);
  const bool t3 = pl->dtype == AMUN_TF32X3;
  const cuuint64_t K = t3 ? 3ull * pl->H : (cuuint64_t)pl->H;
  const cuuint32_t esz = f8 || f4 ? 1 : t3 ? 4 : 2;   // smem bytes per element
  cuuint64_t dims[2] = {K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {f4 ? K / 2 : K * esz};
  cuuint32_t box[2] = {(cuuint32_t)kbytes / esz, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out,
                   f4 ? CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B
                   : f8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                      : t3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   kbytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(AMUN_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return AMUN_OK;
}

amun_status get_map(amun_ol* pl, MapEntry* cache, int n, int& next, const void* ptr,
                    long long rows, int box_rows, int kbytes, const CUtensorMap** out) {
  const bool is_w = cache == pl->wmaps;
  for (int i = 0; i < n; ++i)
    if (cache[i].ptr == ptr && cache[i].rows == rows && cache[i].box_rows == box_rows &&
        cache[i].kbytes == kbytes) {
      *out = &cache[i].map;
      return AMUN_OK;
    }
  MapEntry& e = cache[next];
  next = (next + 1) % n;
  amun_status s = encode_map(pl, ptr, rows, box_rows, kbytes, is_w, &e.map);
  if (s != AMUN_OK) {
    e.ptr = nullptr;
    return s;
  }
  e.ptr = ptr;
  e.rows = rows;
  e.box_rows = box_rows;
  e.kbytes = kbytes;
  *out = &e.map;
  return AMUN_OK;
}

// CTA pairs (tcgen05 cta_group::2) for bf16 when the 128-row M-tiles pair up
// with little padding: an even count, or >= 9 (<= 1/10 padded). A pair
// computes 256 rows, so with an odd count one CTA of the last pair computes
// padding; measured at 5 M-tiles (cfg "beam") the single-CTA kernel wins,
// at 96 (cfg "shard") pairs are 1.35x faster under the power cap
// (tools/power_probe.py).
bool use_pairs(const amun_ol* pl, int N) {
  if (pl->dtype != AMUN_BF16 || pl->pairs_mode == 1) return false;
  const long long n_mt = cdiv(N > 0 ? N : 1, 128);
  if (pl->pairs_mode == 2) return n_mt >= 2;
  return n_mt >= 2 && (n_mt % 2 == 0 || n_mt >= 9);
}

// Schedule over "units" of M rows: 128-row M-tiles for single CTAs, 256-row
// pair tiles for CTA pairs (then *grid counts CTAs = 2 x pairs).
Schedule make_schedule(const amun_ol* pl, int N, int* grid) {
  const bool pairs = use_pairs(pl, N);
  const long long G = pairs ? pl->num_sms / 2 : pl->num_sms;
  const long long n_mt = cdiv(N > 0 ? N : 1, pairs ? 256 : 128);
  const long long align = pl->dtype == AMUN_MXFP4 ? TC_F4_ALIGN : 16;   // mxfp4: 32-row groups
  Schedule s = schedule_for(n_mt, cdiv(pl->V_local, align) * align, G, align);
  const int units = (int)cdiv((n_mt - 1) * s.band + s.Vp, s.C);
  *grid = pairs ? 2 * units : units;
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int KB>
amun_status launch_simt(const SimtParams& sp, int grid, cudaStream_t st, int mode) {
  if (mode == 0)
    ol_simt_kernel<KB, 0><<<grid, 128, 0, st>>>(sp);
  else
    ol_simt_kernel<1, 1><<<grid, 128, 0, st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}

// Stage 1: fused GEMM + epilogue into the workspace slots (mode 0) or the
// debug logits (mode 1).
// amun_output_layer_dev: CTA pairs or single CTAs must be chosen at launch,
// without N; pairs when max_rows spans >= 9 M-tiles (the host rule for
// large N), unless AMUN_PAIRS=off / force.
bool dev_pairs(const amun_ol* pl) {
  if (pl->dtype != AMUN_BF16 || pl->pairs_mode == 1) return false;
  return pl->pairs_mode == 2 || cdiv(pl->max_rows, 128) >= 9;
}

// tail != TAIL_NONE (modes 0 / 4, tcgen05 plans): the merge runs in the same
// launch (tail.cuh) with the parameters in *tmp; its part / layout / schedule
// / N are filled in here.
amun_status run_scores(amun_ol* pl, const void* X, const void* W, const float* b, int N,
                       void* workspace, float* logits, cudaStream_t st, int mode,
                       const int* N_dev = nullptr, const float* x_scale = nullptr,
                       const float* w_scale = nullptr, int tail = TAIL_NONE,
                       const MergeParams* tmp = nullptr, const OneShotTail* os = nullptr) {
  if (N == 0) return AMUN_OK;
  CUDA_TRY(cudaSetDevice(pl->device));
  int grid;
  Schedule sch = make_schedule(pl, N, &grid);
  if (N_dev) {   // N = max_rows here; every SM gets a CTA, the device picks the schedule
    const bool dp = dev_pairs(pl);
    sch = schedule_for(cdiv(N, dp ? 256 : 128), cdiv(pl->V_local, 16) * 16,
                       dp ? pl->num_sms / 2 : pl->num_sms);
    grid = dp ? pl->num_sms / 2 * 2 : pl->num_sms;
  }
  if (pl->dtype != AMUN_F32) {   // tcgen05: bf16 (kind::f16) or e4m3 (kind::f8f6f4)
    const bool pairs = N_dev ? dev_pairs(pl) : use_pairs(pl, N);
    const CUtensorMap *mx, *mw;
    // N < 128: the X box covers only the rows that exist (rounded up to 8).
    // A 128-row box that is mostly out of bounds made TMA measurably slower
    // (cfg beam at S = 1: 59 vs 53 us per call); the MMA still reads the full
    // 128-row A tile, whose extra rows only feed accumulator rows >= N.
    const int a_rows = (!pairs && !N_dev && N < TC_BM) ? (int)cdiv(N, 8) * 8 : TC_BM;
    // bytes of K per pipeline block: the pair kernel 128 (SW128), the
    // single-CTA kernel TC_KBYTES (ol_tc.cuh)
    const int kbytes = pairs ? 128 : TC_KBYTES;
    // W multicast clusters (env AMUN_MC = cluster size, experiment): when the
    // aligned schedule has exactly mc M-tiles, the mc CTAs of one vocab split
    // form a cluster and share each W K-block (one multicast per 64-row box)
    int mc = 0;
    if (pl->mc > 1 && !pairs && !N_dev && mode != 1 && sch.band != sch.Vp &&
        cdiv(N, TC_BM) == pl->mc && grid % pl->mc == 0)
      mc = pl->mc;
    const int wbox = pl->dtype == AMUN_MXFP4 ? TC_BN_F4 : mc > 1 ? 64 : pl->wbox;
    amun_status s = get_map(pl, pl->xmaps, 4, pl->xnext, X, N, a_rows, kbytes, &mx);
    if (s != AMUN_OK) return s;
    s = get_map(pl, pl->wmaps, 16, pl->wnext, W, pl->V_local, pairs ? TC_BN / 2 : wbox, kbytes,
                &mw);
    if (s != AMUN_OK) return s;
    // single CTAs with 256-row W boxes: a second map of 64-row boxes for the
    // narrow remainder tile of each CTA range (ol_tc.cuh)
    const CUtensorMap* mwn = mw;
    const bool wnarrow = pl->wnarrow && !pairs && pl->dtype != AMUN_MXFP4 && wbox == 256 &&
                         mc <= 1;
    if (wnarrow) {
      s = get_map(pl, pl->wmaps, 16, pl->wnext, W, pl->V_local, 64, kbytes, &mwn);
      if (s != AMUN_OK) return s;
    }
    TcParams tp;
    memset(&tp, 0, sizeof(tp));
    tp.mp.part_floats = (long long)(pl->slots_bytes / 4);   // (checked builds' bound)
    tp.N = N;
    tp.V_local = pl->V_local;
    tp.v_offset = pl->v_offset;
    // smem bytes of K per row (mxfp4 W: one byte per code once unpacked)
    const long long kbytes_total = pl->dtype == AMUN_E4M3 || pl->dtype == AMUN_MXFP4 ? pl->H
                                 : pl->dtype == AMUN_TF32X3 ? 12LL * pl->H : 2LL * pl->H;
    tp.n_kblk = (int)cdiv(kbytes_total, kbytes);
    tp.x_scale = x_scale;
    if (pl->dtype == AMUN_MXFP4)   // (the mxfp4 entry points pass W's block scales here)
      tp.w_sf = reinterpret_cast<const uint8_t*>(w_scale);
    else
      tp.w_scale = w_scale;
    tp.a_box_bytes = a_rows * kbytes;   // kbytes of K per row (every dtype)
    tp.sch = sch;
    tp.bias = b;
    tp.part = static_cast<float*>(workspace);
    tp.stride = pl->stride;
    tp.k_max = pl->k_max;
    tp.logits = logits;
    tp.hint = reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) + pl->slots_bytes);
    tp.gen_ctr = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + pl->slots_bytes +
                                                 pl->hint_bytes);
    // cross-CTA hints pay off only when a CTA's range holds several tiles: with
    // ~2 (cfg greedy) they arrive too late and their atomics contend (148
    // publishers per row word)
    tp.use_hint = sch.C >= 4 * TC_BN ? 1 : 0;
    tp.N_dev = N_dev;
    tp.num_sms = pl->num_sms;
    tp.arrive = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + pl->slots_bytes +
                                                pl->hint_bytes + 8);   // after {generation, count}
    if ((mode == 0 || mode == 4) && tail != TAIL_NONE) {
      tp.tail = tail | (pl->tail_mode == 2 ? TAIL_X_NOWORK : 0) | (pl->tail_mode == 3 ? TAIL_X_NOCOOP : 0) |
                (pl->tail_mode == 4 ? TAIL_X_FENCE : 0) | (pl->tail_mode == 5 ? TAIL_X_SLEEP : 0) |
                (pl->tail_mode == 6 ? TAIL_X_NOWORK | TAIL_X_NOCOOP : 0) |
                (pl->tail_mode == 7 ? TAIL_X_NOWORK | TAIL_X_FENCE : 0);
      tp.mp = *tmp;
      tp.mp.part = static_cast<const float*>(workspace);
      tp.mp.layout = pairs ? 2 : 0;
      tp.mp.sch = sch;
      tp.mp.N = N;
      tp.mp.N_dev = nullptr;   // the kernel passes its own resolved N / schedule (TcDyn)
      tp.mp.num_sms = pl->num_sms;
    }
    if (os) tp.os = *os;
    tp.tl = pl->tl;
    tp.taper = pairs ? 0 : pl->taper;
    tp.prepass = pl->prepass;
    tp.wbox = wbox;
    tp.mc = mc;
    tp.pdl = pairs ? 0 : pl->pdl;
    tp.mma_only = pl->mma_only;
    tp.wnarrow = wnarrow ? 1 : 0;
    if ((mode == 0 || mode == 4) && pl->hint_ws != workspace) {
      // hint words carry the launch generation (advanced on the device by the
      // kernel itself); zero words + counters + tail flags once per workspace
      // (amun_ol_workspace_init does the same on request)
      CUDA_TRY(cudaMemsetAsync(tp.hint, 0, pl->hint_bytes + 256 + pl->flags_bytes, st));
      pl->hint_ws = workspace;
    }
#define TC_CALL(K) launch_tc<K>((int)pl->dtype, pl->ng_override, mx, mw, mwn, tp, grid, st, mode, \
                                pairs)
    AMUN_KB_SWITCH(mode == 1 || mode == 4 ? 1 : pl->kb, TC_CALL)
#undef TC_CALL
  } else {
    SimtParams sp;
    sp.N = N;
    sp.V_local = pl->V_local;
    sp.v_offset = pl->v_offset;
    sp.H = pl->H;
    sp.sch = sch;
    sp.X = static_cast<const float*>(X);
    sp.W = static_cast<const float*>(W);
    sp.bias = b;
    sp.part = static_cast<float*>(workspace);
    sp.stride = pl->stride;
    sp.k_max = pl->k_max;
    sp.logits = logits;
    if (mode == 4) return launch_simt<1>(sp, grid, st, 0);   // argmax: the k = 1 records
#define SIMT_CALL(K) launch_simt<K>(sp, grid, st, mode)
    AMUN_KB_SWITCH(mode == 1 ? 1 : pl->kb, SIMT_CALL)
#undef SIMT_CALL
  }
}

template <int KB>
amun_status launch_merge(const MergeParams& mp, bool rows, int grid, cudaStream_t st) {
  if (grid == 0) return AMUN_OK;
  // Plain stream-ordered launch. Programmatic dependent launch (scheduling
  // this grid early, waiting in griddepcontrol.wait) measured slower inside
  // CUDA graphs: cfg beam 108.5 vs 107.0 us, greedy 20.5 vs 19.8 us
  // (DESIGN.md §6.2).
  if (rows)
    merge_rows_kernel<KB><<<grid, MS_WARPS * 32, 0, st>>>(mp);
  else   // grid = S; k_max = 1 takes a warp per sentence
    merge_sentences_kernel<KB><<<KB == 1 ? (grid + MS_WARPS - 1) / MS_WARPS : grid, MS_WARPS * 32,
                                 0, st>>>(mp);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}

amun_status run_merge(amun_ol* pl, const MergeParams& mp, bool rows, int grid, cudaStream_t st) {
#define MERGE_CALL(K) launch_merge<K>(mp, rows, grid, st)
  AMUN_KB_SWITCH(pl->kb, MERGE_CALL)
#undef MERGE_CALL
}

amun_status check_select_args(const amun_ol* pl, const float* prev_cost,
                              const int32_t* beam_offsets, int N, int S, int k,
                              const int64_t* out_idx, const float* out_cost) {
  if (N < 0 || N > pl->max_rows) return fail(AMUN_EINVAL, "N=%d out of [0, max_rows=%d]", N, pl->max_rows);
  if (S < 0 || S > pl->max_sentences)
    return fail(AMUN_EINVAL, "S=%d out of [0, max_sentences=%d]", S, pl->max_sentences);
  if (k < 1 || k > pl->k_max) return fail(AMUN_EINVAL, "k=%d out of [1, k_max=%d]", k, pl->k_max);
  if (S > 0 && (!beam_offsets || !out_idx || !out_cost))
    return fail(AMUN_EINVAL, "NULL beam_offsets/out_idx/out_cost");
  if (N > 0 && !prev_cost) return fail(AMUN_EINVAL, "NULL prev_cost");
  return AMUN_OK;
}

amun_status check_score_args(const amun_ol* pl, const void* X, const void* W, const float* b,
                             int N, const void* workspace) {
  if (!pl) return fail(AMUN_EINVAL, "NULL plan");
  if (N < 0 || N > pl->max_rows) return fail(AMUN_EINVAL, "N=%d out of [0, max_rows=%d]", N, pl->max_rows);
  if (N == 0) return AMUN_OK;
  if (!X || !W || !b || !workspace) return fail(AMUN_EINVAL, "NULL X/W/b/workspace");
  if (!aligned16(X) || !aligned16(W)) return fail(AMUN_EINVAL, "X and W must be 16-byte aligned");
  if (!aligned16(b)) return fail(AMUN_EINVAL, "b must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(AMUN_EINVAL, "workspace must be 256-byte aligned");
  return AMUN_OK;
}

MergeParams base_merge(const amun_ol* pl) {
  MergeParams mp;
  memset(&mp, 0, sizeof(mp));
  mp.stride = pl->stride;
  mp.part_floats = (long long)(pl->slots_bytes / 4);   // the workspace's record slots
  mp.k_max = pl->k_max;
  mp.V_total = pl->V_total;
  return mp;
}

// The sentence-phase parameters of one call (merge kernel or fused tail).
MergeParams sent_merge(const amun_ol* pl, const float* prev_cost, const int32_t* beam_offsets,
                       int N, int S, const int32_t* k_s, int k, int64_t* out_idx, float* out_cost) {
  MergeParams mp = base_merge(pl);
  mp.N = N;
  mp.S = S;
  mp.prev_cost = prev_cost;
  mp.offsets = beam_offsets;
  mp.k_s = k_s;
  mp.k = k;
  mp.out_idx = reinterpret_cast<long long*>(out_idx);
  mp.out_cost = out_cost;
  return mp;
}

// The merge runs in the fused kernel's tail (one launch per call) for the
// tcgen05 plans, unless AMUN_TAIL=off; N = 0 still needs the merge kernel
// (no fused launch happens, the outputs are padded by the merge).
bool use_tail(const amun_ol* pl, int N) {
  return pl->tail_mode != 1 && pl->dtype != AMUN_F32 && N > 0;
}

// Plans whose entry points carry scales (*_e4m3, *_mxfp4).
bool scaled_plan(const amun_ol* pl) { return pl->dtype == AMUN_E4M3 || pl->dtype == AMUN_MXFP4; }

}  // namespace

namespace {
// Vocab-shard piece 1 for any tcgen05 / SIMT plan: the fused kernel, then
// the row-mode merge into one record per row (scales: e4m3 plans only).
amun_status partial_impl(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                         float* partial, void* workspace, void* stream, const float* x_scale,
                         const float* w_scale) {
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  if (N == 0) return AMUN_OK;
  if (!partial) return fail(AMUN_EINVAL, "NULL partial");
  if (use_tail(plan, N)) {
    MergeParams mp = base_merge(plan);
    mp.N = N;
    mp.out_part = partial;
    return run_scores(plan, X, W, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0,
                      nullptr, x_scale, w_scale, TAIL_ROWS, &mp);
  }
  s = run_scores(plan, X, W, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0,
                 nullptr, x_scale, w_scale);
  if (s != AMUN_OK) return s;
  MergeParams mp = base_merge(plan);
  int grid_unused;
  mp.part = static_cast<const float*>(workspace);
  mp.layout = use_pairs(plan, N) ? 2 : 0;
  mp.sch = make_schedule(plan, N, &grid_unused);
  mp.N = N;
  mp.out_part = partial;
  return run_merge(plan, mp, true, (int)cdiv(N, MS_WARPS), static_cast<cudaStream_t>(stream));
}
}  // namespace

extern "C" {

int amun_abi_version(void) { return AMUN_ABI_VERSION; }

const char* amun_last_error(void) { return g_err.c_str(); }

const char* amun_status_string(amun_status s) {
  switch (s) {
    case AMUN_OK: return "AMUN_OK";
    case AMUN_EINVAL: return "AMUN_EINVAL";
    case AMUN_EUNSUPPORTED: return "AMUN_EUNSUPPORTED";
    case AMUN_ECUDA: return "AMUN_ECUDA";
  }
  return "AMUN_UNKNOWN";
}

amun_status amun_ol_create(amun_ol** plan, int H, int V_local, int v_offset, int V_total,
                           amun_dtype dtype, int k_max, int max_rows, int max_sentences,
                           int device) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan pointer");
  *plan = nullptr;
  if (dtype != AMUN_F32 && dtype != AMUN_BF16 && dtype != AMUN_E4M3 && dtype != AMUN_TF32X3 &&
      dtype != AMUN_MXFP4)
    return fail(AMUN_EINVAL, "unknown dtype %d", (int)dtype);
  if (H < 1) return fail(AMUN_EINVAL, "H=%d must be >= 1", H);
  if (dtype == AMUN_BF16 && H % 8 != 0) return fail(AMUN_EINVAL, "bf16 needs H %% 8 == 0 (H=%d)", H);
  if ((dtype == AMUN_F32 || dtype == AMUN_TF32X3) && H % 4 != 0)
    return fail(AMUN_EINVAL, "f32 / tf32x3 need H %% 4 == 0 (H=%d)", H);
  if (dtype == AMUN_E4M3 && H % 16 != 0) return fail(AMUN_EINVAL, "e4m3 needs H %% 16 == 0 (H=%d)", H);
  if (dtype == AMUN_MXFP4 && H % 128 != 0)
    return fail(AMUN_EINVAL, "mxfp4 needs H %% 128 == 0 (H=%d)", H);
  if (V_local < 1) return fail(AMUN_EINVAL, "V_local=%d must be >= 1", V_local);
  if (v_offset < 0 || V_total < 1 || (long long)v_offset + V_local > V_total)
    return fail(AMUN_EINVAL, "need 0 <= v_offset and v_offset + V_local <= V_total");
  if (k_max < 1 || k_max > AMUN_MAX_K) return fail(AMUN_EINVAL, "k_max=%d out of [1, %d]", k_max, AMUN_MAX_K);
  if (max_rows < 0 || max_sentences < 0) return fail(AMUN_EINVAL, "negative capacity");
  if ((long long)max_rows * V_total >= (1LL << 62)) return fail(AMUN_EINVAL, "max_rows * V_total overflows");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(AMUN_EINVAL, "device %d out of range (%d devices)", device, ndev);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(AMUN_EUNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a (B200)",
                device, prop.major, prop.minor);
  amun_ol* pl = new (std::nothrow) amun_ol();
  if (!pl) return fail(AMUN_EINVAL, "out of host memory");
  pl->H = H;
  pl->V_local = V_local;
  pl->v_offset = v_offset;
  pl->V_total = V_total;
  pl->dtype = dtype;
  pl->k_max = k_max;
  pl->kb = kbucket(k_max);
  pl->max_rows = max_rows;
  pl->max_sentences = max_sentences;
  pl->device = device;
  pl->num_sms = prop.multiProcessorCount;
  {   // (experiment AMUN_SMS: the plan schedules over fewer SMs, e.g. to share
      // the GPU with a concurrent kernel on another stream)
    const char* e = getenv("AMUN_SMS");
    if (e && atoi(e) > 0 && atoi(e) < pl->num_sms) pl->num_sms = atoi(e);
  }
  pl->stride = 2 + 2 * k_max;
  {
    const char* g = getenv("AMUN_NG");
    pl->ng_override = g ? atoi(g) : 0;
    if (pl->ng_override < 2 || pl->ng_override > 4) pl->ng_override = 0;
  }
  {
    const char* e = getenv("AMUN_PAIRS");
    pl->pairs_mode = !e ? 0 : (strcmp(e, "off") == 0 ? 1 : (strcmp(e, "force") == 0 ? 2 : 0));
    // experiments: off | wait (no merge work) | nocoop | fence | sleep
    const char* t = getenv("AMUN_TAIL");
    pl->tail_mode = !t ? 0 : strcmp(t, "off") == 0 ? 1 : strcmp(t, "wait") == 0 ? 2
                  : strcmp(t, "nocoop") == 0 ? 3 : strcmp(t, "fence") == 0 ? 4
                  : strcmp(t, "sleep") == 0 ? 5 : strcmp(t, "waitnocoop") == 0 ? 6
                  : strcmp(t, "arriveonly") == 0 ? 7 : 0;
    const char* mcv = getenv("AMUN_MC");
    if (mcv) pl->mc = atoi(mcv);
    const char* pd = getenv("AMUN_PDL");
    if (pd) pl->pdl = atoi(pd) != 0;
    const char* wn = getenv("AMUN_WNARROW");
    if (wn) pl->wnarrow = atoi(wn) != 0;
    const char* wb = getenv("AMUN_WBOX");
    if (wb) pl->wbox = atoi(wb) == 64 ? 64 : 256;
    const char* pp = getenv("AMUN_PREPASS");
    if (pp) pl->prepass = atoi(pp);
    const char* tp = getenv("AMUN_TAPER");
    if (tp) pl->taper = atoi(tp) != 0;
    if (pl->taper) pl->wbox = 64;   // narrow tiles load only their own rows
  }
  const long long slots = pl->num_sms + cdiv(max_rows > 0 ? max_rows : 1, 128) + 1;
  pl->slots_bytes = (size_t)cdiv(slots * 128LL * pl->stride * 4, 256) * 256;
  pl->hint_bytes = (size_t)cdiv((long long)(max_rows > 0 ? max_rows : 1) * 8, 256) * 256;
  pl->flags_bytes = 0;   // the 256-byte counter block holds {generation, count, arrive[2]}
  pl->ws_bytes = pl->slots_bytes + pl->hint_bytes + 256 + pl->flags_bytes;
  *plan = pl;
  return AMUN_OK;
}

amun_status amun_ol_destroy(amun_ol* plan) {
  delete plan;
  return AMUN_OK;
}

size_t amun_ol_workspace_bytes(const amun_ol* plan) { return plan ? plan->ws_bytes : 0; }

amun_status amun_ol_workspace_init(amun_ol* plan, void* workspace, void* stream) {
  if (!plan || !workspace) return fail(AMUN_EINVAL, "NULL plan or workspace");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(AMUN_EINVAL, "workspace must be 256-byte aligned");
  CUDA_TRY(cudaSetDevice(plan->device));
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(workspace) + plan->slots_bytes, 0,
                           plan->hint_bytes + 256 + plan->flags_bytes,
                           static_cast<cudaStream_t>(stream)));
  plan->hint_ws = workspace;
  return AMUN_OK;
}

int amun_ol_partial_stride(const amun_ol* plan) { return plan ? plan->stride : 0; }

int amun_ol_launches_per_call(const amun_ol* plan, int call) {
  if (!plan || call < 0 || call > 2) return -1;
  if (call == 2) return 1;
  return use_tail(plan, 1) ? 1 : 2;
}

amun_status amun_ol_scores(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                           void* workspace, void* stream) {
  if (plan && scaled_plan(plan))
    return fail(AMUN_EINVAL, "e4m3 / mxfp4 plans take their own entry points (they carry the scales)");
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  return run_scores(plan, X, W, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0);
}

amun_status amun_ol_select(amun_ol* plan, const void* workspace, const float* prev_cost,
                           const int32_t* beam_offsets, int N, int S,
                           const int32_t* k_per_sentence, int k, int64_t* out_idx,
                           float* out_cost, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  amun_status s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  if (N > 0 && !workspace) return fail(AMUN_EINVAL, "NULL workspace");
  if (S == 0) return AMUN_OK;
  CUDA_TRY(cudaSetDevice(plan->device));
  MergeParams mp = base_merge(plan);
  int grid_unused;
  mp.part = static_cast<const float*>(workspace);
  mp.layout = use_pairs(plan, N > 0 ? N : 1) ? 2 : 0;
  mp.sch = make_schedule(plan, N > 0 ? N : 1, &grid_unused);
  mp.N = N;
  mp.S = S;
  mp.prev_cost = prev_cost;
  mp.offsets = beam_offsets;
  mp.k_s = k_per_sentence;
  mp.k = k;
  mp.out_idx = reinterpret_cast<long long*>(out_idx);
  mp.out_cost = out_cost;
  return run_merge(plan, mp, false, S, static_cast<cudaStream_t>(stream));
}

amun_status amun_output_layer(amun_ol* plan, const void* X, const void* W, const float* b,
                              const float* prev_cost, const int32_t* beam_offsets, int N, int S,
                              const int32_t* k_per_sentence, int k, int64_t* out_idx,
                              float* out_cost, void* workspace, void* stream) {
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  if (!scaled_plan(plan) && use_tail(plan, N)) {
    const MergeParams mp = sent_merge(plan, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                                      out_idx, out_cost);
    return run_scores(plan, X, W, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0,
                      nullptr, nullptr, nullptr, TAIL_SENT, &mp);
  }
  s = amun_ol_scores(plan, X, W, b, N, workspace, stream);
  if (s != AMUN_OK) return s;
  return amun_ol_select(plan, workspace, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                        out_idx, out_cost, stream);
}

amun_status amun_output_layer_dev(amun_ol* plan, const void* X, const void* W, const float* b,
                                  const float* prev_cost, const int32_t* beam_offsets,
                                  const int32_t* N_dev, int S, const int32_t* k_per_sentence,
                                  int k, int64_t* out_idx, float* out_cost, void* workspace,
                                  void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  if (!N_dev) return fail(AMUN_EINVAL, "NULL N_dev");
  if (plan->dtype != AMUN_BF16 && plan->dtype != AMUN_TF32X3)
    return fail(AMUN_EUNSUPPORTED, "device-side N: bf16 / tf32x3 plans only");
  const int Nmax = plan->max_rows;
  amun_status s = check_score_args(plan, X, W, b, Nmax, workspace);
  if (s != AMUN_OK) return s;
  s = check_select_args(plan, prev_cost, beam_offsets, Nmax, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_tail(plan, Nmax)) {
    const MergeParams mp = sent_merge(plan, prev_cost, beam_offsets, Nmax, S, k_per_sentence, k,
                                      out_idx, out_cost);
    return run_scores(plan, X, W, b, Nmax, workspace, nullptr, st, 0, N_dev, nullptr, nullptr,
                      TAIL_SENT, &mp);
  }
  s = run_scores(plan, X, W, b, Nmax, workspace, nullptr, st, 0, N_dev);
  if (s != AMUN_OK) return s;
  if (S == 0) return AMUN_OK;
  MergeParams mp = base_merge(plan);
  mp.part = static_cast<const float*>(workspace);
  const bool dp = dev_pairs(plan);
  mp.layout = dp ? 2 : 0;
  mp.sch = schedule_for(cdiv(Nmax, dp ? 256 : 128), cdiv(plan->V_local, 16) * 16,
                        dp ? plan->num_sms / 2 : plan->num_sms);
  mp.N = Nmax;
  mp.N_dev = N_dev;
  mp.num_sms = plan->num_sms;
  mp.S = S;
  mp.prev_cost = prev_cost;
  mp.offsets = beam_offsets;
  mp.k_s = k_per_sentence;
  mp.k = k;
  mp.out_idx = reinterpret_cast<long long*>(out_idx);
  mp.out_cost = out_cost;
  return run_merge(plan, mp, false, S, st);
}

amun_status amun_output_layer_partial(amun_ol* plan, const void* X, const void* W,
                                      const float* b, int N, float* partial, void* workspace,
                                      void* stream) {
  if (plan && scaled_plan(plan))
    return fail(AMUN_EINVAL, "e4m3 / mxfp4 plans take their own entry points (they carry the scales)");
  return partial_impl(plan, X, W, b, N, partial, workspace, stream, nullptr, nullptr);
}

amun_status amun_output_layer_partial_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                           const uint8_t* W8, const float* w_scale, const float* b,
                                           int N, float* partial, void* workspace, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  if (plan->dtype != AMUN_E4M3) return fail(AMUN_EINVAL, "plan dtype is not AMUN_E4M3");
  if (N > 0 && (!x_scale || !w_scale)) return fail(AMUN_EINVAL, "NULL x_scale / w_scale");
  if (N > 0 && !aligned16(w_scale)) return fail(AMUN_EINVAL, "w_scale must be 16-byte aligned");
  return partial_impl(plan, X8, W8, b, N, partial, workspace, stream, x_scale, w_scale);
}

amun_status amun_merge_partials(amun_ol* plan, const float* partials, int G,
                                const float* prev_cost, const int32_t* beam_offsets, int N, int S,
                                const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                float* out_cost, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  if (G < 1) return fail(AMUN_EINVAL, "G=%d must be >= 1", G);
  amun_status s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  if (N > 0 && !partials) return fail(AMUN_EINVAL, "NULL partials");
  if ((reinterpret_cast<uintptr_t>(partials) & 7) != 0)
    return fail(AMUN_EINVAL, "partials must be 8-byte aligned");
  if (S == 0) return AMUN_OK;
  CUDA_TRY(cudaSetDevice(plan->device));
  MergeParams mp = base_merge(plan);
  mp.part = partials;
  mp.layout = 1;
  mp.G = G;
  mp.N = N;
  mp.part_floats = (long long)G * N * plan->stride;
  mp.S = S;
  mp.prev_cost = prev_cost;
  mp.offsets = beam_offsets;
  mp.k_s = k_per_sentence;
  mp.k = k;
  mp.out_idx = reinterpret_cast<long long*>(out_idx);
  mp.out_cost = out_cost;
  return run_merge(plan, mp, false, S, static_cast<cudaStream_t>(stream));
}

amun_status amun_debug_logits(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                              float* logits, void* workspace, void* stream) {
  if (plan && scaled_plan(plan))
    return fail(AMUN_EINVAL, "e4m3 / mxfp4 plans take their own entry points (they carry the scales)");
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  if (N > 0 && !logits) return fail(AMUN_EINVAL, "NULL logits");
  return run_scores(plan, X, W, b, N, workspace, logits, static_cast<cudaStream_t>(stream), 1);
}

namespace {
amun_status argmax_impl(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                        int64_t* out_token, float* out_logit, void* workspace, void* stream,
                        const float* x_scale, const float* w_scale) {
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  if (N > 0 && (!out_token || !out_logit)) return fail(AMUN_EINVAL, "NULL out_token / out_logit");
  if (N == 0) return AMUN_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_tail(plan, N)) {
    MergeParams mp = base_merge(plan);
    mp.N = N;
    mp.out_idx = reinterpret_cast<long long*>(out_token);
    mp.out_cost = out_logit;
    return run_scores(plan, X, W, b, N, workspace, nullptr, st, 4, nullptr, x_scale, w_scale,
                      TAIL_ARGMAX, &mp);
  }
  s = run_scores(plan, X, W, b, N, workspace, nullptr, st, 4, nullptr, x_scale, w_scale);
  if (s != AMUN_OK) return s;
  MergeParams mp = base_merge(plan);
  int grid_unused;
  mp.part = static_cast<const float*>(workspace);
  mp.layout = use_pairs(plan, N) ? 2 : 0;
  mp.sch = make_schedule(plan, N, &grid_unused);
  mp.N = N;
  // one warp per row (more CTAs spread the latency-bound reduction)
  argmax_rows_kernel<<<(unsigned)N, 32, 0, st>>>(mp, reinterpret_cast<long long*>(out_token),
                                                 out_logit);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}
}  // namespace

amun_status amun_argmax(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                        int64_t* out_token, float* out_logit, void* workspace, void* stream) {
  if (plan && scaled_plan(plan))
    return fail(AMUN_EINVAL, "e4m3 / mxfp4 plans take their own entry points (they carry the scales)");
  return argmax_impl(plan, X, W, b, N, out_token, out_logit, workspace, stream, nullptr, nullptr);
}

amun_status amun_argmax_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                             const uint8_t* W8, const float* w_scale, const float* b, int N,
                             int64_t* out_token, float* out_logit, void* workspace, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  if (plan->dtype != AMUN_E4M3) return fail(AMUN_EINVAL, "plan dtype is not AMUN_E4M3");
  if (N > 0 && (!x_scale || !w_scale)) return fail(AMUN_EINVAL, "NULL x_scale / w_scale");
  if (N > 0 && !aligned16(w_scale)) return fail(AMUN_EINVAL, "w_scale must be 16-byte aligned");
  return argmax_impl(plan, X8, W8, b, N, out_token, out_logit, workspace, stream, x_scale, w_scale);
}

amun_status amun_ol_scores_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                const uint8_t* W8, const float* w_scale, const float* b, int N,
                                int variant, void* workspace, void* stream) {
  amun_status s = check_score_args(plan, X8, W8, b, N, workspace);
  if (s != AMUN_OK) return s;
  if (plan->dtype != AMUN_E4M3) return fail(AMUN_EINVAL, "plan dtype is not AMUN_E4M3");
  if (variant != 0 && variant != 2 && variant != 3)
    return fail(AMUN_EINVAL, "variant %d not in {0, 2, 3}", variant);
  if (N > 0 && (!x_scale || !w_scale)) return fail(AMUN_EINVAL, "NULL x_scale / w_scale");
  if (N > 0 && !aligned16(w_scale)) return fail(AMUN_EINVAL, "w_scale must be 16-byte aligned");
  return run_scores(plan, X8, W8, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream),
                    variant, nullptr, x_scale, w_scale);
}

amun_status amun_output_layer_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                   const uint8_t* W8, const float* w_scale, const float* b,
                                   const float* prev_cost, const int32_t* beam_offsets, int N,
                                   int S, const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                   float* out_cost, void* workspace, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  amun_status s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  if (use_tail(plan, N)) {
    s = check_score_args(plan, X8, W8, b, N, workspace);
    if (s != AMUN_OK) return s;
    if (plan->dtype != AMUN_E4M3) return fail(AMUN_EINVAL, "plan dtype is not AMUN_E4M3");
    if (!x_scale || !w_scale) return fail(AMUN_EINVAL, "NULL x_scale / w_scale");
    if (!aligned16(w_scale)) return fail(AMUN_EINVAL, "w_scale must be 16-byte aligned");
    const MergeParams mp = sent_merge(plan, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                                      out_idx, out_cost);
    return run_scores(plan, X8, W8, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0,
                      nullptr, x_scale, w_scale, TAIL_SENT, &mp);
  }
  s = amun_ol_scores_e4m3(plan, X8, x_scale, W8, w_scale, b, N, 0, workspace, stream);
  if (s != AMUN_OK) return s;
  return amun_ol_select(plan, workspace, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                        out_idx, out_cost, stream);
}

// ------------------------------------------------------------ MXFP4 W (f4)
namespace {
amun_status check_mxfp4(const amun_ol* plan, const float* x_scale, const void* W4,
                        const uint8_t* w_sf, int N) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  if (plan->dtype != AMUN_MXFP4) return fail(AMUN_EINVAL, "plan dtype is not AMUN_MXFP4");
  if (N > 0 && (!x_scale || !w_sf)) return fail(AMUN_EINVAL, "NULL x_scale / w_sf");
  if (N > 0 && (reinterpret_cast<uintptr_t>(W4) & 31) != 0)
    return fail(AMUN_EINVAL, "W4 must be 32-byte aligned (TMA 16U4_ALIGN16B)");
  if (N > 0 && !aligned16(w_sf)) return fail(AMUN_EINVAL, "w_sf must be 16-byte aligned");
  return AMUN_OK;
}
// the SF pointer travels in run_scores' w_scale slot (run_scores: tp.w_sf)
inline const float* sf_arg(const uint8_t* w_sf) { return reinterpret_cast<const float*>(w_sf); }
}  // namespace

size_t amun_mxfp4_sf_bytes(int R, int H) {
  if (R < 0 || H < 128 || H % 128 != 0) return 0;
  return (size_t)cdiv(R, 128) * (size_t)(H / 128) * 512;
}

amun_status amun_quantize_mxfp4(const void* src, amun_dtype src_dtype, int R, int H,
                                uint8_t* codes, uint8_t* sf, void* stream) {
  if (src_dtype != AMUN_F32 && src_dtype != AMUN_BF16)
    return fail(AMUN_EINVAL, "src_dtype must be AMUN_F32 or AMUN_BF16");
  if (R < 0 || H < 128 || H % 128 != 0) return fail(AMUN_EINVAL, "need R >= 0, H %% 128 == 0");
  if (R == 0) return AMUN_OK;
  if (!src || !codes || !sf) return fail(AMUN_EINVAL, "NULL src / codes / sf");
  if ((reinterpret_cast<uintptr_t>(codes) & 1) != 0) return fail(AMUN_EINVAL, "codes must be 2-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long tasks = cdiv(R, 128) * 128 * (H / 128);
  const unsigned grid = (unsigned)std::min<long long>(cdiv(tasks, QZ_THREADS / 32), 4096);
  if (src_dtype == AMUN_BF16)
    quantize_mxfp4_kernel<true><<<grid, QZ_THREADS, 0, st>>>(src, R, H, codes, sf);
  else
    quantize_mxfp4_kernel<false><<<grid, QZ_THREADS, 0, st>>>(src, R, H, codes, sf);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}

amun_status amun_ol_scores_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                 const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                                 int variant, void* workspace, void* stream) {
  amun_status s = check_score_args(plan, X8, W4, b, N, workspace);
  if (s != AMUN_OK) return s;
  s = check_mxfp4(plan, x_scale, W4, w_sf, N);
  if (s != AMUN_OK) return s;
  if (variant != 0 && (variant < 2 || variant > 7))
    return fail(AMUN_EINVAL, "variant %d not in {0, 2, ..., 7}", variant);
  // 5 / 6 / 7: the bare GEMM re-reading the first stages (as amun_bench_variant)
  plan->mma_only = variant >= 5 ? variant - 4 : 0;
  const amun_status s2 = run_scores(plan, X8, W4, b, N, workspace, nullptr,
                                    static_cast<cudaStream_t>(stream),
                                    variant >= 5 ? 2 : variant, nullptr, x_scale, sf_arg(w_sf));
  plan->mma_only = 0;
  return s2;
}

amun_status amun_output_layer_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                    const uint8_t* W4, const uint8_t* w_sf, const float* b,
                                    const float* prev_cost, const int32_t* beam_offsets, int N,
                                    int S, const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                    float* out_cost, void* workspace, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  amun_status s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  if (use_tail(plan, N)) {
    s = check_score_args(plan, X8, W4, b, N, workspace);
    if (s != AMUN_OK) return s;
    s = check_mxfp4(plan, x_scale, W4, w_sf, N);
    if (s != AMUN_OK) return s;
    const MergeParams mp = sent_merge(plan, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                                      out_idx, out_cost);
    return run_scores(plan, X8, W4, b, N, workspace, nullptr, static_cast<cudaStream_t>(stream), 0,
                      nullptr, x_scale, sf_arg(w_sf), TAIL_SENT, &mp);
  }
  s = amun_ol_scores_mxfp4(plan, X8, x_scale, W4, w_sf, b, N, 0, workspace, stream);
  if (s != AMUN_OK) return s;
  return amun_ol_select(plan, workspace, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                        out_idx, out_cost, stream);
}

amun_status amun_argmax_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                              const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                              int64_t* out_token, float* out_logit, void* workspace,
                              void* stream) {
  amun_status s = check_mxfp4(plan, x_scale, W4, w_sf, N);
  if (s != AMUN_OK) return s;
  return argmax_impl(plan, X8, W4, b, N, out_token, out_logit, workspace, stream, x_scale,
                     sf_arg(w_sf));
}

amun_status amun_debug_logits_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                    const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                                    float* logits, void* workspace, void* stream) {
  amun_status s = check_score_args(plan, X8, W4, b, N, workspace);
  if (s != AMUN_OK) return s;
  s = check_mxfp4(plan, x_scale, W4, w_sf, N);
  if (s != AMUN_OK) return s;
  if (N > 0 && !logits) return fail(AMUN_EINVAL, "NULL logits");
  return run_scores(plan, X8, W4, b, N, workspace, logits, static_cast<cudaStream_t>(stream), 1,
                    nullptr, x_scale, sf_arg(w_sf));
}

amun_status amun_quantize_e4m3(const void* src, amun_dtype src_dtype, int R, int H, uint8_t* dst,
                               float* scale, void* stream) {
  if (R < 0 || H < 0 || (H & 1)) return fail(AMUN_EINVAL, "R=%d, H=%d: need R, H >= 0 and H even", R, H);
  if (src_dtype != AMUN_F32 && src_dtype != AMUN_BF16)
    return fail(AMUN_EINVAL, "src_dtype must be AMUN_F32 or AMUN_BF16");
  if (R == 0 || H == 0) return AMUN_OK;
  if (!src || !dst || !scale) return fail(AMUN_EINVAL, "NULL src/dst/scale");
  if ((reinterpret_cast<uintptr_t>(dst) & 1) != 0) return fail(AMUN_EINVAL, "dst must be 2-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<long long>(R, 148LL * 16);
  if (src_dtype == AMUN_BF16)
    quantize_e4m3_kernel<true><<<grid, QZ_THREADS, 0, st>>>(src, R, H, dst, scale);
  else
    quantize_e4m3_kernel<false><<<grid, QZ_THREADS, 0, st>>>(src, R, H, dst, scale);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}

amun_status amun_debug_timeline(amun_ol* plan, unsigned long long* timeline) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  plan->tl = timeline;
  return AMUN_OK;
}

amun_status amun_bench_variant(amun_ol* plan, const void* X, const void* W, const float* b,
                               int N, int variant, void* workspace, void* stream) {
  amun_status s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  if (variant < 2 || variant > 7) return fail(AMUN_EINVAL, "variant %d not in [2, 7]", variant);
  if (plan->dtype != AMUN_BF16) return fail(AMUN_EUNSUPPORTED, "variants exist for bf16 only");
  // 5 = bare GEMM whose MMAs re-read the first stages; 6 / 7 = only X / only W
  // copied again after the first stages
  plan->mma_only = variant >= 5 ? variant - 4 : 0;
  const amun_status s2 = run_scores(plan, X, W, b, N, workspace, nullptr,
                                    static_cast<cudaStream_t>(stream), variant >= 5 ? 2 : variant);
  plan->mma_only = 0;
  return s2;
}

}  // extern "C"

namespace {
// Validate and copy the state columns: src holds n_src rows, dst receives up
// to n_dst rows; src and dst ranges must not overlap.
amun_status fill_columns(CompactParams& cp, const amun_column* cols, int n_cols, long long n_src,
                         long long n_dst) {
  if (n_cols < 0 || n_cols > AMUN_MAX_COLUMNS)
    return fail(AMUN_EINVAL, "n_cols=%d out of [0, %d]", n_cols, AMUN_MAX_COLUMNS);
  if (n_cols > 0 && !cols) return fail(AMUN_EINVAL, "NULL cols");
  for (int c = 0; c < n_cols; ++c) {
    const amun_column& col = cols[c];
    if (col.row_bytes <= 0 || (col.row_bytes & 3))
      return fail(AMUN_EINVAL, "column %d: row_bytes=%lld must be a positive multiple of 4", c,
                  (long long)col.row_bytes);
    if ((n_src > 0 || n_dst > 0) && (!col.src || !col.dst))
      return fail(AMUN_EINVAL, "column %d: NULL src/dst", c);
    if (((reinterpret_cast<uintptr_t>(col.src) | reinterpret_cast<uintptr_t>(col.dst)) & 3) != 0)
      return fail(AMUN_EINVAL, "column %d: src/dst must be 4-byte aligned", c);
    const uintptr_t s0 = reinterpret_cast<uintptr_t>(col.src), d0 = reinterpret_cast<uintptr_t>(col.dst);
    const uintptr_t ls = (uintptr_t)col.row_bytes * (uintptr_t)n_src;
    const uintptr_t ld = (uintptr_t)col.row_bytes * (uintptr_t)n_dst;
    if (ls > 0 && ld > 0 && s0 < d0 + ld && d0 < s0 + ls)
      return fail(AMUN_EINVAL, "column %d: src and dst overlap", c);
    cp.col[c].src = static_cast<const uint8_t*>(col.src);
    cp.col[c].dst = static_cast<uint8_t*>(col.dst);
    cp.col[c].row_bytes = col.row_bytes;
  }
  cp.n_cols = n_cols;
  return AMUN_OK;
}

amun_status launch_compact(CompactParams& cp, int N, int S, int32_t* counts, int32_t* counts_host,
                           cudaStream_t st) {
  cp.N = N;
  cp.S = S;
  cp.counts = counts;
  cp.blk_log2 = 6;   // 64 flags per prefix block, doubled until <= CP_MAXBLK blocks
  while ((1LL << cp.blk_log2) * CP_MAXBLK < N) ++cp.blk_log2;
  const long long nblk = cdiv(N > 0 ? N : 1, 1LL << cp.blk_log2);
  static const bool small_smem = getenv("AMUN_CP_SMALLSMEM") != nullptr;   // (experiment)
  cp.flags_in_smem = (N <= CP_SFLAGS && !small_smem) ? 1 : 0;
  const size_t dyn0 = (size_t)((nblk + 1) * 4 + 15) / 16 * 16 +
                      (cp.flags_in_smem ? (size_t)cdiv(N, 64) * 64 : 0);
  cp.dyn_off_at = (int)dyn0;
  cp.cnt_pre = (S + 1 <= CP_CNTPRE && !small_smem) ? 1 : 0;
  const size_t dyn = dyn0 + (S + 1 <= CP_CNTPRE && !small_smem ? (size_t)(S + 1) * 4 : 0);
  static const int exp_env = getenv("AMUN_CP_EXP") ? atoi(getenv("AMUN_CP_EXP")) : 0;
  cp.exp = exp_env;
  // CTAs: 8 output rows each while that fits one wave (CP_CTAS_PER_SM per
  // SM), then up to CP_MAXR rows each; at least one thread per sentence
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  static int nsm_cache[64] = {0};
  int nsm = dev < 64 ? nsm_cache[dev] : 0;
  if (nsm == 0) {
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (dev < 64) nsm_cache[dev] = nsm;
  }
  const long long wave = (long long)CP_CTAS_PER_SM * nsm;
  // (+1: CTA 0 counts the sentences and gathers nothing)
  const int grid = 1 + (int)std::max<long long>(
      {1LL, cdiv(N, CP_MAXR), std::min<long long>(cdiv(N, CP_ROWS), wave - 1),
       cdiv((long long)S + 1, CP_THREADS)});
  // counts[1] accumulates the CTAs' alive-sentence counts (compact_kernel step 4)
  compact_kernel<<<grid, CP_THREADS, dyn, st>>>(cp);
  CUDA_TRY(cudaGetLastError());
  if (counts_host) {
    CUDA_TRY(cudaMemcpyAsync(counts_host, counts, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return AMUN_OK;
}

long long a256(long long n) { return (n + 255) / 256 * 256; }
}  // namespace

extern "C" {

amun_status amun_sentence_alive(const int32_t* new_beam_offsets, int S, uint8_t* alive_s,
                                int32_t* unit_offsets, void* stream) {
  if (S < 0) return fail(AMUN_EINVAL, "negative S");
  if (!new_beam_offsets || !unit_offsets || (S > 0 && !alive_s))
    return fail(AMUN_EINVAL, "NULL new_beam_offsets / alive_s / unit_offsets");
  const int grid = (int)std::min<long long>(cdiv(S + 1, 256), 1024);
  sentence_alive_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      new_beam_offsets, S, alive_s, unit_offsets);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}

amun_status amun_compact(const amun_column* cols, int n_cols, const uint8_t* alive, int N,
                         const int32_t* beam_offsets, int S, int32_t* new_beam_offsets,
                         int32_t* src_row, int32_t* counts, int32_t* counts_host, void* stream) {
  if (N < 0 || S < 0) return fail(AMUN_EINVAL, "negative N or S");
  if (!beam_offsets || !new_beam_offsets || !counts) return fail(AMUN_EINVAL, "NULL offsets/counts");
  if (N > 0 && (!alive || !src_row)) return fail(AMUN_EINVAL, "NULL alive/src_row");
  CompactParams cp;
  memset(&cp, 0, sizeof(cp));
  amun_status s = fill_columns(cp, cols, n_cols, N, N);
  if (s != AMUN_OK) return s;
  cp.alive = alive;
  cp.offsets = beam_offsets;
  cp.new_offsets = new_beam_offsets;
  cp.src_row = src_row;
  return launch_compact(cp, N, S, counts, counts_host, static_cast<cudaStream_t>(stream));
}

size_t amun_beam_advance_workspace_bytes(int S, int k) {
  if (S < 0 || k < 1) return 0;
  const long long n = (long long)S * k;
  return (size_t)(a256(n) + 2 * a256(4 * n));
}

amun_status amun_beam_advance(const int64_t* out_idx, const float* out_cost, int S, int k,
                              int64_t V_total, int eos_token, int N, const amun_column* cols,
                              int n_cols, int32_t* new_beam_offsets, int32_t* src_row,
                              int32_t* new_token, float* new_cost, int32_t* counts,
                              int32_t* counts_host, void* workspace, void* stream) {
  if (S < 0 || k < 1 || N < 0) return fail(AMUN_EINVAL, "S=%d, k=%d, N=%d: need S >= 0, k >= 1, N >= 0", S, k, N);
  if (V_total < 1) return fail(AMUN_EINVAL, "V_total=%lld must be >= 1", (long long)V_total);
  if (!new_beam_offsets || !counts) return fail(AMUN_EINVAL, "NULL new_beam_offsets/counts");
  const long long n = (long long)S * k;
  if (n > (1LL << 30)) return fail(AMUN_EINVAL, "S*k=%lld too large", n);
  if (n > 0 && (!out_idx || !out_cost || !src_row || !new_token || !new_cost || !workspace))
    return fail(AMUN_EINVAL, "NULL out_idx/out_cost/src_row/new_token/new_cost/workspace");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(AMUN_EINVAL, "workspace must be 256-byte aligned");
  CompactParams cp;
  memset(&cp, 0, sizeof(cp));
  amun_status s = fill_columns(cp, cols, n_cols, N, n);
  if (s != AMUN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* live = static_cast<uint8_t*>(workspace);
  int* parent = reinterpret_cast<int*>(live + a256(n));
  int* tok = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(parent) + a256(4 * n));
  if (n > 0) {
    beam_classify_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(
        reinterpret_cast<const long long*>(out_idx), (int)n, (long long)V_total, eos_token, live,
        parent, tok);
    CUDA_TRY(cudaGetLastError());
  }
  cp.alive = live;
  cp.off_stride = k;
  cp.new_offsets = new_beam_offsets;
  cp.src_row = src_row;
  cp.parent = parent;
  cp.vtok = tok;
  cp.vcost = out_cost;
  cp.tok_out = new_token;
  cp.cost_out = new_cost;
  return launch_compact(cp, (int)n, S, counts, counts_host, st);
}

#if AMUN_EXP == 4
amun_status amun_debug_counters(unsigned long long* host8, int reset) {
  cudaMemcpyFromSymbol(host8, amun::amun_dbg, 8 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(amun::amun_dbg, z, sizeof(z));
  }
  return AMUN_OK;
}
#endif

amun_status amun_split_tf32x3(const float* src, int R, int H, int role, float* dst, void* stream) {
  if (R < 0 || H < 0 || (H & 3)) return fail(AMUN_EINVAL, "R=%d, H=%d: need R, H >= 0, H %% 4 == 0", R, H);
  if (role != 0 && role != 1) return fail(AMUN_EINVAL, "role %d not in {0 (X), 1 (W)}", role);
  if (R == 0 || H == 0) return AMUN_OK;
  if (!src || !dst) return fail(AMUN_EINVAL, "NULL src/dst");
  const long long n = (long long)R * H;
  const int grid = (int)std::min<long long>(cdiv(n, 256), 148LL * 32);
  split_tf32x3_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, n, H, role, dst);
  CUDA_TRY(cudaGetLastError());
  return AMUN_OK;
}


// ------------------------------------------------------------ NVLink one-shot (NEXT f3)
}  // extern "C"

namespace {

size_t oneshot_recv_elems(const amun_ol* pl, int G) {
  return (size_t)G * (size_t)std::max(pl->max_rows, 1) * (size_t)pl->stride;
}

// CTAs per rank: all co-resident (cooperative launch); the count may differ
// between calls and ranks (the signal counters count calls, not CTAs).
template <int KB>
amun_status oneshot_launch(const amun_ol* pl, OneShotParams& q, int ranks, cudaStream_t st) {
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oneshot_kernel<KB>, MS_WARPS * 32, 0));
  // as many CTAs as there are rows (one warp each) or sentences (one CTA
  // each), up to what is co-resident (<= 4 per SM)
  if (occ < 1) return fail(AMUN_ECUDA, "one-shot kernel does not fit on an SM");
  const int cap = std::max(1, pl->num_sms * std::min(occ, 4) / ranks);
  const int want = std::max((int)cdiv(q.dst.N, MS_WARPS), q.dst.S);
  q.nb = std::max(1, std::min(cap, want));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)q.nb, (unsigned)ranks, 1);
  cfg.blockDim = dim3(MS_WARPS * 32, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, oneshot_kernel<KB>, q));
  return AMUN_OK;
}

amun_status oneshot_run(const amun_ol* pl, OneShotParams& q, int ranks, cudaStream_t st) {
#define OS_CALL(K) oneshot_launch<K>(pl, q, ranks, st)
  AMUN_KB_SWITCH(pl->kb, OS_CALL)
#undef OS_CALL
}

MergeParams oneshot_src(amun_ol* pl, void* workspace, int N) {
  MergeParams mp = base_merge(pl);
  int grid_unused;
  mp.part = static_cast<const float*>(workspace);
  mp.layout = use_pairs(pl, N > 0 ? N : 1) ? 2 : 0;
  mp.sch = make_schedule(pl, N > 0 ? N : 1, &grid_unused);
  mp.N = N;
  return mp;
}

MergeParams oneshot_dst(const amun_ol* pl, int G, const float* prev_cost,
                        const int32_t* beam_offsets, int N, int S, const int32_t* k_s, int k) {
  MergeParams mp = base_merge(pl);
  mp.layout = 1;
  mp.G = G;
  mp.N = N;
  mp.S = S;
  mp.prev_cost = prev_cost;
  mp.offsets = beam_offsets;
  mp.k_s = k_s;
  mp.k = k;
  return mp;
}

amun_status check_bufs(void* const* bufs, int G) {
  if (G < 1 || G > OS_MAX_G) return fail(AMUN_EINVAL, "G=%d out of [1, %d]", G, OS_MAX_G);
  if (!bufs) return fail(AMUN_EINVAL, "NULL bufs");
  for (int p = 0; p < G; ++p)
    if (!bufs[p] || (reinterpret_cast<uintptr_t>(bufs[p]) & 255) != 0)
      return fail(AMUN_EINVAL, "bufs[%d] NULL or not 256-byte aligned", p);
  return AMUN_OK;
}

}  // namespace

extern "C" {

size_t amun_oneshot_buffer_bytes(const amun_ol* plan, int G) {
  if (!plan || G < 1 || G > OS_MAX_G) return 0;
  return OS_CTRL_BYTES + 2 * oneshot_recv_elems(plan, G) * sizeof(float);
}

amun_status amun_oneshot_alloc(const amun_ol* plan, int G, void** buf, void* ipc_handle) {
  if (!plan || !buf) return fail(AMUN_EINVAL, "NULL plan or buf");
  const size_t bytes = amun_oneshot_buffer_bytes(plan, G);
  if (!bytes) return fail(AMUN_EINVAL, "G=%d out of [1, %d]", G, OS_MAX_G);
  CUDA_TRY(cudaSetDevice(plan->device));
  *buf = nullptr;
  CUDA_TRY(cudaMalloc(buf, bytes));
  cudaError_t e = cudaMemset(*buf, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ipc_handle)
    e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(ipc_handle), *buf);
  if (e != cudaSuccess) {
    cudaFree(*buf);
    *buf = nullptr;
    return fail(AMUN_ECUDA, "one-shot buffer: %s", cudaGetErrorString(e));
  }
  return AMUN_OK;
}

amun_status amun_oneshot_free(void* buf) {
  if (buf) CUDA_TRY(cudaFree(buf));
  return AMUN_OK;
}

amun_status amun_oneshot_open(const void* ipc_handle, int device, void** peer) {
  if (!ipc_handle || !peer) return fail(AMUN_EINVAL, "NULL handle or peer");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(peer, h, cudaIpcMemLazyEnablePeerAccess));
  return AMUN_OK;
}

amun_status amun_oneshot_error(const void* buf, int* err) {
  if (!buf || !err) return fail(AMUN_EINVAL, "NULL buf or err");
  unsigned int w = 0;
  CUDA_TRY(cudaMemcpy(&w, static_cast<const unsigned int*>(buf) + OS_ERR, sizeof(w),
                      cudaMemcpyDeviceToHost));
  *err = (int)w;
  return AMUN_OK;
}

amun_status amun_oneshot_close(void* peer) {
  if (peer) CUDA_TRY(cudaIpcCloseMemHandle(peer));
  return AMUN_OK;
}

amun_status amun_output_layer_oneshot(amun_ol* plan, const void* X, const void* W, const float* b,
                                      const float* prev_cost, const int32_t* beam_offsets, int N,
                                      int S, const int32_t* k_per_sentence, int k,
                                      void* const* bufs, int G, int rank, int64_t* out_idx,
                                      float* out_cost, void* workspace, void* stream) {
  if (!plan) return fail(AMUN_EINVAL, "NULL plan");
  amun_status s = check_bufs(bufs, G);
  if (s != AMUN_OK) return s;
  if (rank < 0 || rank >= G) return fail(AMUN_EINVAL, "rank=%d out of [0, G=%d)", rank, G);
  s = check_score_args(plan, X, W, b, N, workspace);
  if (s != AMUN_OK) return s;
  s = check_select_args(plan, prev_cost, beam_offsets, N, S, k, out_idx, out_cost);
  if (s != AMUN_OK) return s;
  CUDA_TRY(cudaSetDevice(plan->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_tail(plan, N)) {
    // ONE launch: the fused kernel whose tail runs the row phase, the peer
    // stores, the signal, the wait and the sentence phase (tail.cuh)
    OneShotTail os;
    memset(&os, 0, sizeof(os));
    for (int p = 0; p < G; ++p) os.buf[p] = static_cast<char*>(bufs[p]);
    os.G = G;
    os.rank = rank;
    os.recv_elems = (long long)oneshot_recv_elems(plan, G);
    const MergeParams mp = sent_merge(plan, prev_cost, beam_offsets, N, S, k_per_sentence, k,
                                      out_idx, out_cost);
    return run_scores(plan, X, W, b, N, workspace, nullptr, st, 0, nullptr, nullptr, nullptr,
                      TAIL_ONESHOT, &mp, &os);
  }
  if (N > 0) {
    s = run_scores(plan, X, W, b, N, workspace, nullptr, st, 0);
    if (s != AMUN_OK) return s;
  }
  OneShotParams q;
  memset(&q, 0, sizeof(q));
  q.src[0] = oneshot_src(plan, workspace, N);
  q.dst = oneshot_dst(plan, G, prev_cost, beam_offsets, N, S, k_per_sentence, k);
  for (int p = 0; p < G; ++p) q.buf[p] = static_cast<char*>(bufs[p]);
  q.out_idx[0] = reinterpret_cast<long long*>(out_idx);
  q.out_cost[0] = out_cost;
  q.G = G;
  q.rank = rank;
  q.emulate = 0;
  q.recv_elems = (long long)oneshot_recv_elems(plan, G);
  return oneshot_run(plan, q, 1, st);
}

amun_status amun_output_layer_oneshot_emulated(amun_ol* const* plans, int G, const void* X,
                                               const void* const* W, const float* const* b,
                                               const float* prev_cost, const int32_t* beam_offsets,
                                               int N, int S, const int32_t* k_per_sentence, int k,
                                               void* const* bufs, int64_t* const* out_idx,
                                               float* const* out_cost, void* const* workspaces,
                                               void* stream) {
  amun_status s = check_bufs(bufs, G);
  if (s != AMUN_OK) return s;
  if (!plans || !W || !b || !out_idx || !out_cost || !workspaces)
    return fail(AMUN_EINVAL, "NULL array argument");
  for (int p = 0; p < G; ++p) {
    if (!plans[p]) return fail(AMUN_EINVAL, "NULL plans[%d]", p);
    if (plans[p]->k_max != plans[0]->k_max || plans[p]->max_rows != plans[0]->max_rows ||
        plans[p]->V_total != plans[0]->V_total || plans[p]->device != plans[0]->device ||
        plans[p]->max_sentences != plans[0]->max_sentences)
      return fail(AMUN_EINVAL, "plans differ in k_max / max_rows / V_total / device");
    s = check_score_args(plans[p], X, W[p], b[p], N, workspaces[p]);
    if (s != AMUN_OK) return s;
    s = check_select_args(plans[p], prev_cost, beam_offsets, N, S, k, out_idx[p], out_cost[p]);
    if (s != AMUN_OK) return s;
  }
  CUDA_TRY(cudaSetDevice(plans[0]->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  OneShotParams q;
  memset(&q, 0, sizeof(q));
  for (int p = 0; p < G; ++p) {
    // the ranks' fused kernels do not wait on anything: sequential launches
    if (N > 0) {
      s = run_scores(plans[p], X, W[p], b[p], N, workspaces[p], nullptr, st, 0);
      if (s != AMUN_OK) return s;
    }
    q.src[p] = oneshot_src(plans[p], workspaces[p], N);
    q.buf[p] = static_cast<char*>(bufs[p]);
    q.out_idx[p] = reinterpret_cast<long long*>(out_idx[p]);
    q.out_cost[p] = out_cost[p];
  }
  q.dst = oneshot_dst(plans[0], G, prev_cost, beam_offsets, N, S, k_per_sentence, k);
  q.G = G;
  q.rank = 0;
  q.emulate = 1;
  q.recv_elems = (long long)oneshot_recv_elems(plans[0], G);
  return oneshot_run(plans[0], q, G, st);
}

}  // extern "C"
