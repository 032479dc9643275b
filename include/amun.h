/*
 * amun.h — C-ABI of the B200-native NMT output-layer hot path
 * (arXiv 1805.09863, "Fast Neural Machine Translation Implementation",
 *  Amun @ WNMT 2018). Library: paper_1805_09863_b200/libamun.so (sm_100a).
 *
 * The path (§2.2 list of the four output-layer steps):
 *   1. p = W x   logits GEMM, tcgen05/TMEM
 *   2. p = p + b   fused into the GEMM epilogue
 *   3. softmax   online max / sum-of-exp
 *                                             (Alg. 4, rescale
 *                                             P:193-200 read with exp(Delta))
 *   4. k-best                        ("k-best search is a simple
 *                                             extension"), generalised to beam
 *                                             search: per sentence, top-k_s over
 *                                             beam x vocab of
 *                                             cost = prev_cost[r] + log p[r][v]
 *   + mini-batching (Alg. 2): remove finished hypotheses
 *     ("Remove h from b") by stable compaction, or fused with the
 *     beam reorder (amun_beam_advance); greedy argmax without the softmax
 *     (Alg. 5, amun_argmax); 8-bit storage (amun_*_e4m3) and
 *     block-scaled 4-bit W (amun_*_mxfp4).
 *
 * Conventions (all entry points):
 *   - Every pointer argument that names device memory is a CUDA device
 *     pointer (cudaMalloc / torch CUDA storage) on the plan's device.
 *     The CALLER owns all memory: inputs, outputs and workspace. The library
 *     never allocates device memory and never synchronises the stream, except
 *     amun_compact() / amun_beam_advance() when counts_host != NULL.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream). Calls are stream-ordered and CUDA-graph capturable (except
 *     those two with counts_host).
 *   - Layouts are row-major, C order. dtype AMUN_BF16 means IEEE bfloat16
 *     storage (fp32 accumulation); AMUN_F32 means fp32 storage and true fp32
 *     products (SIMT kernel); AMUN_E4M3 means OCP FP8 E4M3 codes with fp32
 *     per-row scales (fp32 accumulation; the *_e4m3 entry points);
 *     AMUN_MXFP4 means E4M3 X with per-row scales and OCP MXFP4 W (E2M1
 *     codes + one E8M0 scale per 32 elements; the *_mxfp4 entry points).
 *   - Errors: every call returns amun_status; no exception crosses the ABI.
 *     The message of the last failure on the calling thread is returned by
 *     amun_last_error(). Host-side validation happens before anything is
 *     launched: on AMUN_EINVAL / AMUN_EUNSUPPORTED nothing was enqueued.
 *     Inputs are assumed finite; non-finite inputs give
 *     unspecified (but memory-safe) results.
 *   - Ties (reading G3 of DESIGN.md, P:174/P:210/P:247 strict '>' scans):
 *     equal biased logits in a row rank by lower token id; equal costs in a
 *     sentence rank by lower row, then higher logit, then lower token id.
 */
#ifndef AMUN_H_
#define AMUN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMUN_ABI_VERSION 1
#define AMUN_MAX_K 16          /* largest k-best width per row / sentence */
#define AMUN_MAX_COLUMNS 16    /* largest number of columns one amun_compact call moves */

typedef enum amun_status {
  AMUN_OK = 0,
  AMUN_EINVAL = 1,        /* bad argument (shape, alignment, range, NULL) */
  AMUN_EUNSUPPORTED = 2,  /* valid but not supported (device not sm_100, dtype) */
  AMUN_ECUDA = 3          /* a CUDA runtime/driver call failed */
} amun_status;

typedef enum amun_dtype {
  AMUN_F32 = 0,     /* fp32 X, W: SIMT kernel, true fp32 products */
  AMUN_BF16 = 1,    /* bf16 X, W: tcgen05 kind::f16 */
  AMUN_E4M3 = 2,    /* E4M3 codes + per-row fp32 scales: tcgen05 kind::f8f6f4 (*_e4m3 calls) */
  AMUN_TF32X3 = 3,  /* fp32 as 3xTF32 on tcgen05 kind::tf32: X, W passed pre-split by
                       amun_split_tf32x3 as [N, 3H] / [V_local, 3H] fp32 rows */
  AMUN_MXFP4 = 4    /* E4M3 X (per-row scales) x MXFP4 W (E2M1 + E8M0 per 32 K):
                       tcgen05 kind::mxf8f6f4.block_scale (*_mxfp4 calls), H % 128 == 0 */
} amun_dtype;

/* Opaque plan: shapes, kernel choice, persistent-grid schedule and cached TMA
 * tensor maps. Not thread-safe: use one plan per host thread. */
typedef struct amun_ol amun_ol;

int         amun_abi_version(void);
const char* amun_last_error(void);
const char* amun_status_string(amun_status s);

/* Create a plan for one vocabulary shard.
 *   H         hidden size (K of the GEMM). bf16: H % 8 == 0; f32, tf32x3:
 *             H % 4 == 0; e4m3: H % 16 == 0 (TMA / vector alignment: a row
 *             is a multiple of 16 bytes).
 *   V_local   rows of W (and entries of b) this plan owns, 1 <= V_local.
 *   v_offset  global token id of local row 0 (vocab sharding; 0 on one GPU).
 *   V_total   global vocabulary size; out_idx encodes r * V_total + token.
 *             Requires v_offset + V_local <= V_total.
 *   dtype     storage type of X and W.
 *   k_max     largest k any later call uses, 1..AMUN_MAX_K. Partial records
 *             hold k_max entries.
 *   max_rows, max_sentences  capacity the workspace is sized for.
 *   device    CUDA ordinal; must be compute capability 10.0 (B200, sm_100a).
 * On success *plan is set; destroy with amun_ol_destroy. */
amun_status amun_ol_create(amun_ol** plan, int H, int V_local, int v_offset, int V_total,
                           amun_dtype dtype, int k_max, int max_rows, int max_sentences,
                           int device);
amun_status amun_ol_destroy(amun_ol* plan);

/* Bytes of device workspace the caller must pass to the calls below
 * (per-CTA partial states of the fused kernel, then the cross-CTA hint
 * words, the launch-generation counters and the fused tail's per-CTA
 * arrival words). 256-byte aligned.
 *
 * The workspace is STATE of the plan, not scratch: it must be dedicated to
 * one plan and keep its contents between that plan's calls (the generation
 * counter and the arrival words tag every launch, CUDA-graph replays
 * included, so nothing is reset per call). A buffer the plan has not used
 * before must be initialised once: the library does so itself (a
 * stream-ordered memset) the first time it sees a workspace ADDRESS; a
 * caller that hands the plan memory at an address it already used, after
 * the memory served something else, calls amun_ol_workspace_init first.
 * A fused tail that finds the arrival words inconsistent (never a silent
 * wrong result) traps after 10 s. */
size_t amun_ol_workspace_bytes(const amun_ol* plan);

/* Zero the hint / counter / arrival region of `workspace` on `stream` and
 * register it as initialised for `plan` (see amun_ol_workspace_bytes).
 * Errors: AMUN_EINVAL (NULL, misaligned), AMUN_ECUDA. */
amun_status amun_ol_workspace_init(amun_ol* plan, void* workspace, void* stream);

/* Kernels of this library one call enqueues (for launch accounting in
 * benchmarks): `call` = 0 amun_output_layer / _dev / _e4m3 / amun_argmax,
 * 1 amun_output_layer_partial, 2 amun_merge_partials. With the fused tail
 * (the default for tcgen05 plans, see amun_output_layer) calls 0 and 1 are
 * ONE launch; otherwise two. N = 0 calls may enqueue fewer. Returns -1 for
 * a NULL plan or an unknown `call`. */
int amun_ol_launches_per_call(const amun_ol* plan, int call);

/* Floats per row of a partial record: 2 + 2*k_max, laid out as
 *   { m, s, l[0..k_max-1], v[0..k_max-1] }
 * m = max biased logit of the covered vocabulary, s = sum exp(l - m) over it,
 * l = the k_max largest biased logits (desc, ties -> lower v), v = their
 * GLOBAL token ids stored as int32 bit patterns. Unused entries: (-inf, -1);
 * a record covering no vocabulary has m = -inf, s = 0. */
int amun_ol_partial_stride(const amun_ol* plan);

/* Full single-GPU path: steps 1-4 (GEMM + bias + softmax + beam k-best).
 *   X            [N, H] dtype; row r is the decoder state of hypothesis r.
 *   W            [V_local, H] dtype (row v = output embedding of token
 *                v_offset + v).
 *   b            [V_local] fp32 bias (full precision).
 *   prev_cost    [N] fp32 cumulative log-prob of each hypothesis.
 *   beam_offsets [S+1] int32, o_0 = 0 <= o_1 <= ... <= o_S = N; sentence s
 *                owns rows [o_s, o_{s+1}) (a sentence may be empty).
 *   k_per_sentence  [S] int32 or NULL (then every sentence uses k);
 *                0 <= k_s <= k (Amun-style shrinking beam, reading G6).
 *   k            output width per sentence, 1 <= k <= k_max.
 *   out_idx      [S, k] int64: r * V_total + token of the i-th best candidate
 *                of sentence s (r = global row index), -1 padding.
 *   out_cost     [S, k] fp32: prev_cost[r] + log p[r][token], -inf padding.
 *                Each sentence's entries are sorted by cost, descending.
 *   workspace    amun_ol_workspace_bytes(plan) bytes, 256-byte aligned.
 * 0 <= N <= max_rows, 0 <= S <= max_sentences. X and W must be 16-byte
 * aligned (TMA). Enqueues ONE kernel for tcgen05 plans: the fused
 * GEMM/epilogue whose tail (after a grid-wide arrival, cooperative launch)
 * runs the merge/select (AMUN_TAIL=off in the environment at plan creation:
 * 2 kernels, the fused kernel then the separate select kernel); fp32 SIMT
 * plans and N = 0 enqueue the 2-kernel form. */
amun_status amun_output_layer(amun_ol* plan, const void* X, const void* W, const float* b,
                              const float* prev_cost, const int32_t* beam_offsets, int N, int S,
                              const int32_t* k_per_sentence, int k, int64_t* out_idx,
                              float* out_cost, void* workspace, void* stream);

/* amun_output_layer with the row count in DEVICE memory:
 * N = *N_dev, read by the kernels themselves (e.g. counts[0] written by
 * amun_beam_advance or amun_compact), so a decode loop needs no host sync
 * per step and can be captured in one CUDA graph.
 *   X         [max_rows, H] bf16 (rows >= N are ignored), prev_cost [max_rows];
 *   N_dev     device int32, clamped to [0, max_rows];
 *   beam_offsets [S+1] device (o_S = N), other arguments as amun_output_layer.
 * The fused kernel is launched with one CTA per SM and derives its schedule
 * from N on the device (CTAs without work only take part in setup). The
 * kernel is chosen from max_rows: CTA pairs (cta_group::2) when max_rows
 * spans >= 9 M-tiles of 128 rows, else single CTAs (always for tf32x3).
 * bf16 and tf32x3 plans (X then [max_rows, 3H] fp32); EUNSUPPORTED otherwise.
 * Enqueues 2 kernels. */
amun_status amun_output_layer_dev(amun_ol* plan, const void* X, const void* W, const float* b,
                                  const float* prev_cost, const int32_t* beam_offsets,
                                  const int32_t* N_dev, int S, const int32_t* k_per_sentence,
                                  int k, int64_t* out_idx, float* out_cost, void* workspace,
                                  void* stream);

/* The two stages of amun_output_layer, exposed so a caller can time or
 * overlap them: stage 1 writes per-(row, vocab split) partial records into
 * `workspace`; stage 2 reads them (same N) and selects per sentence. */
amun_status amun_ol_scores(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                           void* workspace, void* stream);
amun_status amun_ol_select(amun_ol* plan, const void* workspace, const float* prev_cost,
                           const int32_t* beam_offsets, int N, int S,
                           const int32_t* k_per_sentence, int k, int64_t* out_idx,
                           float* out_cost, void* stream);

/* Vocab-sharded path, piece 1 (Alg. 6 shard step): the per-row
 * partial record of THIS shard (all of its V_local tokens combined):
 *   partial [N, amun_ol_partial_stride(plan)] fp32 (see layout above). */
amun_status amun_output_layer_partial(amun_ol* plan, const void* X, const void* W,
                                      const float* b, int N, float* partial, void* workspace,
                                      void* stream);

/* Vocab-sharded path, piece 2 (Alg. 6 reduce step): exact merge of
 * G shards' partial records, combined in shard order g = 0..G-1, then the
 * per-sentence selection of amun_output_layer.
 *   partials [G, N, amun_ol_partial_stride(plan)] fp32, 8-byte aligned (e.g.
 *            the result of an all-gather of every rank's
 *            amun_output_layer_partial output).
 * Other arguments as amun_output_layer. Token ids are already global. */
amun_status amun_merge_partials(amun_ol* plan, const float* partials, int G,
                                const float* prev_cost, const int32_t* beam_offsets, int N, int S,
                                const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                float* out_cost, void* stream);

/* Greedy decoding, Alg. 5 "argmax_1best": for every
 * row, the token with the largest biased logit, WITHOUT the softmax (it is
 * monotone, so the argmax needs no exp; observation 1). Ties go to
 * the lowest token id (reading G3).
 *   X, W, b      as amun_output_layer (single GPU: v_offset = 0 plans only
 *                give global ids when V_local = V_total).
 *   out_token    [N] int64: the winning token id (v_offset + v).
 *   out_logit    [N] fp32: its biased logit (W x + b)[token] (NOT a log-prob).
 * Same fused kernel with the softmax statistics compiled out and k = 1,
 * then a per-row argmax over the vocab-split records. Enqueues 2 kernels.
 * Errors: EINVAL for N < 0, N > max_rows or NULL outputs with N > 0. */
amun_status amun_argmax(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                        int64_t* out_token, float* out_logit, void* workspace, void* stream);

/* FP8 path (the modern analogue of the paper's 16-bit
 * storage, section 2.3): X and W as OCP E4M3 codes with one fp32
 * scale per row, the logits computed as
 *   L[r][v] = (sum_h x8[r][h] w8[v][h]) * x_scale[r] * w_scale[v] + b[v]
 * on tcgen05.mma kind::f8f6f4 (fp32 accumulation), then the same softmax /
 * k-best / merge as amun_output_layer. Plan: amun_ol_create(..., AMUN_E4M3,
 * ...), H % 16 == 0; single-CTA kernel; vocab shards through
 * amun_output_layer_partial_e4m3 + amun_merge_partials.
 *   X8 [N, H] uint8, x_scale [N] fp32, W8 [V_local, H] uint8, w_scale
 *   [V_local] fp32 (16-byte aligned), other arguments as amun_output_layer.
 * Enqueues 2 kernels. Parity: the oracle computes on the exactly dequantised
 * values (oracle.dequant_rows_e4m3). */
amun_status amun_output_layer_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                   const uint8_t* W8, const float* w_scale, const float* b,
                                   const float* prev_cost, const int32_t* beam_offsets, int N,
                                   int S, const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                   float* out_cost, void* workspace, void* stream);
/* Stage 1 alone of amun_output_layer_e4m3 (then amun_ol_select), or with
 * variant 2 / 3 the bare-GEMM / no-k-best benchmark builds (as
 * amun_bench_variant). variant 0 = the real stage 1. */
amun_status amun_ol_scores_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                const uint8_t* W8, const float* w_scale, const float* b, int N,
                                int variant, void* workspace, void* stream);
/* Vocab-shard piece 1 for e4m3 plans (as amun_output_layer_partial; the
 * records merge with amun_merge_partials like bf16 ones). Arguments as
 * amun_ol_scores_e4m3, partial [N, amun_ol_partial_stride(plan)] fp32. */
amun_status amun_output_layer_partial_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                           const uint8_t* W8, const float* w_scale, const float* b,
                                           int N, float* partial, void* workspace, void* stream);
/* Greedy argmax (Alg. 5) for e4m3 plans: as amun_argmax, out_logit =
 * (sum_h x8 w8) * x_scale[r] * w_scale[token] + b[token]. */
amun_status amun_argmax_e4m3(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                             const uint8_t* W8, const float* w_scale, const float* b, int N,
                             int64_t* out_token, float* out_logit, void* workspace, void* stream);
/* 3xTF32 split for AMUN_TF32X3 plans: every fp32 value x is
 * split as hi = tf32(x) (round to nearest), lo = tf32(x - hi), and a row of H
 * values becomes 3H values: role 0 (X) [hi | hi | lo], role 1 (W)
 * [hi | lo | hi], so the plain tf32 GEMM over K = 3H computes
 * X_hi W_hi + X_hi W_lo + X_lo W_hi (the 3xTF32 product; the dropped
 * X_lo W_lo term is ~2^-22 relative).
 *   src [R, H] fp32, dst [R, 3H] fp32, device; H % 4 == 0. One launch. */
amun_status amun_split_tf32x3(const float* src, int R, int H, int role, float* dst, void* stream);

/* Per-row E4M3 quantisation: scale[r] = max_h |src[r][h]| / 448 (1 for an
 * all-zero row), dst[r][h] = RNE-to-E4M3(src[r][h] / scale[r]), saturating;
 * IEEE fp32 arithmetic, so the codes equal oracle.quantize_rows_e4m3 bit for
 * bit. src [R, H] fp32 (src_dtype AMUN_F32) or bf16 (AMUN_BF16), H even,
 * device; dst [R, H] uint8, scale [R] fp32, device. One launch. */
amun_status amun_quantize_e4m3(const void* src, amun_dtype src_dtype, int R, int H, uint8_t* dst,
                               float* scale, void* stream);

/* Block-scaled 4-bit W (the 4-bit analogue of the paper's
 * reduced-precision storage, section 2.3; reading G20 in
 * DESIGN.md): W in the OCP Microscaling format MXFP4 (v1.0): each row's H
 * values in blocks of 32 sharing one E8M0 scale 2^(c - 127), each element an
 * E2M1 code (values 0, 0.5, 1, 1.5, 2, 3, 4, 6 and their negatives). X stays
 * E4M3 with per-row fp32 scales (amun_quantize_e4m3). The logits are
 *   L[r][v] = (sum_h x8[r][h] * e2m1(w4[v][h]) * 2^(sf[v][h/32] - 127)) * x_scale[r] + b[v]
 * computed by tcgen05.mma kind::mxf8f6f4.block_scale (the block scales are
 * applied inside the tensor core; fp32 accumulation), then the same
 * softmax / k-best / merge as amun_output_layer. Plan: amun_ol_create(...,
 * AMUN_MXFP4, ...), H % 128 == 0; single-CTA kernel, 224-column tiles
 * (tensor memory holds the scales beside the two accumulators).
 *
 * Layouts (device):
 *   W4   [V_local, H/2] uint8: two codes per byte, element 2j in the low
 *        nibble of byte j; 32-byte aligned (TMA 16U4_ALIGN16B).
 *   w_sf amun_mxfp4_sf_bytes(V_local, H) bytes, 16-byte aligned, in the
 *        scale-atom order the kernel copies to tensor memory unchanged: for
 *        W row v and element h, the E8M0 code of block h/32 is at byte
 *          ((h/128) * ceil(V_local/128) + v/128) * 512
 *            + 16 * (v%32) + 4 * ((v%128)/32) + (h%128)/32.
 *        Rows beyond V_local in the last 128-row atom: any code (their W
 *        rows read as zero and their columns are masked).
 * Parity: the oracle computes on the exactly dequantised values
 * (oracle.dequant_rows_mxfp4 / dequant_rows_e4m3). */
size_t amun_mxfp4_sf_bytes(int R, int H);   /* 0 if H % 128 != 0 or R < 0 */
/* Quantise R rows of H values (fp32 or bf16, device) to MXFP4 in the layouts
 * above: shared exponent e = floor(log2(max |x| of the block)) - 2 (E8M0
 * code e + 127 clamped to [0, 254]; 127 for an all-zero block), code =
 * round-to-nearest-even E2M1 of x * 2^-e, saturating at +-6, sign kept (-0
 * possible); equals oracle.quantize_rows_mxfp4 bit for bit. H % 128 == 0;
 * codes [R, H/2] (2-byte aligned), sf amun_mxfp4_sf_bytes(R, H) bytes. One
 * launch. */
amun_status amun_quantize_mxfp4(const void* src, amun_dtype src_dtype, int R, int H,
                                uint8_t* codes, uint8_t* sf, void* stream);
/* Steps 1-4 for AMUN_MXFP4 plans: arguments as amun_output_layer_e4m3 with
 * W4 / w_sf for W8 / w_scale. One launch (the merge in the fused kernel's
 * tail), two with AMUN_TAIL=off. */
amun_status amun_output_layer_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                    const uint8_t* W4, const uint8_t* w_sf, const float* b,
                                    const float* prev_cost, const int32_t* beam_offsets, int N,
                                    int S, const int32_t* k_per_sentence, int k, int64_t* out_idx,
                                    float* out_cost, void* workspace, void* stream);
/* Stage 1 alone (variant 0; then amun_ol_select), or the benchmark builds
 * of amun_bench_variant: bare GEMM (2), no k-best (3), bare GEMM re-reading
 * the first stages (5), with only X (6) / only W (7) copied again. */
amun_status amun_ol_scores_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                 const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                                 int variant, void* workspace, void* stream);
/* Greedy argmax (Alg. 5) for AMUN_MXFP4 plans: as amun_argmax, out_logit =
 * L[r][token] as defined above. One launch. */
amun_status amun_argmax_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                              const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                              int64_t* out_token, float* out_logit, void* workspace,
                              void* stream);
/* Test hook (as amun_debug_logits): L [N, V_local] fp32 of an AMUN_MXFP4 plan. */
amun_status amun_debug_logits_mxfp4(amun_ol* plan, const uint8_t* X8, const float* x_scale,
                                    const uint8_t* W4, const uint8_t* w_sf, const float* b, int N,
                                    float* logits, void* workspace, void* stream);

/* Test hook: steps 1-2 only. Writes the biased logits of the same tcgen05
 * (bf16) or SIMT (f32) GEMM to logits [N, V_local] fp32 (these never reach
 * HBM on the real path). For bit-exact GEMM checks in the integer regime. */
amun_status amun_debug_logits(amun_ol* plan, const void* X, const void* W, const float* b, int N,
                              float* logits, void* workspace, void* stream);

/* Benchmark hook (the analogue of the paper's Table 4 breakdown):
 * the same fused kernel with part of the epilogue compiled out.
 *   variant 2: bare GEMM, the epilogue only drains the TMEM accumulators;
 *   variant 3: GEMM + bias + online max/sum-of-exp, no k-best;
 *   variant 4: the first kernel of amun_argmax alone (k = 1, no exp);
 *   variant 5: variant 2 whose MMAs re-read the first pipeline stages after
 *              they are loaded once (the MMA issue rate without TMA traffic);
 *   variant 6 / 7: the same, but X / W is still copied for every block.
 * Results are meaningless scratch in `workspace`; bf16 plans only. */
amun_status amun_bench_variant(amun_ol* plan, const void* X, const void* W, const float* b,
                               int N, int variant, void* workspace, void* stream);

/* Measurement hook: when `timeline` (device memory, >= #SMs x 40 u64,
 * caller-owned) is non-NULL, every later fused launch of the single-CTA
 * tcgen05 kernel through `plan` writes per-CTA %globaltimer stamps (ns):
 * [cta][0] entry, [1] after setup (barriers, TMEM), [2] first TMA issue,
 * [3] first stage landed at the MMA warp, [4] last MMA issued, [5] last
 * accumulator ready at the epilogue, [6] epilogue done, [7] final barrier,
 * [8] tail released (all CTAs arrived), [9] tail merge done, [10..23]
 * the time the epilogue takes up tile 0..13 (its accumulator ready and the
 * previous tile's epilogue done), [24..37] the time the MMA issuer starts
 * tile 0..13 (its accumulator released by the epilogue). NULL switches it off. Not
 * synchronised; for tools/timeline.py. */
amun_status amun_debug_timeline(amun_ol* plan, unsigned long long* timeline);

/* Sentence-level state after a row compaction (optional
 * part: compact the per-sentence encoder-context columns too). Alg. 2
 * removes finished hypotheses; a sentence none of whose rows
 * survived is finished, and its sentence-level state (encoder context,
 * source length, ...) can go as well. Writes
 *   alive_s      [S] uint8 device: 1 iff new_beam_offsets[s+1] > new_beam_offsets[s];
 *   unit_offsets [S+1] int32 device: 0, 1, ..., S;
 * from new_beam_offsets [S+1] (device, the output of amun_compact /
 * amun_beam_advance). Then amun_compact(sentence columns, alive_s, N = S,
 * unit_offsets, S, ...) gathers them stably (its src_row = the old sentence
 * of each kept sentence). One kernel, no sync; EINVAL on argument errors. */
amun_status amun_sentence_alive(const int32_t* new_beam_offsets, int S, uint8_t* alive_s,
                                int32_t* unit_offsets, void* stream);

/* Mini-batching (Alg. 2 "Remove h from b"): stable compaction.
 * One column = one per-hypothesis state array of N rows of row_bytes bytes:
 *   src  [N, row_bytes] device, dst [>= N', row_bytes] device (must not
 *   overlap src). row_bytes % 4 == 0, src/dst 4-byte aligned (16-byte rows
 *   and pointers take the vector path).
 *   alive         [N] uint8, nonzero = hypothesis survives this step.
 *   beam_offsets  [S+1] int32 of the input batch.
 *   new_beam_offsets [S+1] int32 out: number of surviving rows before o_s.
 *   src_row       [N] int32 out: src_row[j] = input row of output row j,
 *                 for j < N' (entries >= N' are not written).
 *   counts        [2] int32 device out: {N', S_alive} (S_alive = sentences
 *                 that keep at least one row).
 *   counts_host   optional host int32[2]; if non-NULL the call copies counts
 *                 back and SYNCHRONISES the stream (not graph-capturable).
 * 0 <= N, 0 <= S, n_cols <= AMUN_MAX_COLUMNS (n_cols may be 0: only the
 * scan outputs are produced). One kernel launch. Bit-exact. */
typedef struct amun_column {
  const void* src;
  void* dst;
  int64_t row_bytes;
} amun_column;

amun_status amun_compact(const amun_column* cols, int n_cols, const uint8_t* alive, int N,
                         const int32_t* beam_offsets, int S, int32_t* new_beam_offsets,
                         int32_t* src_row, int32_t* counts, int32_t* counts_host, void* stream);

/* Beam advance (SPEC S:324-332 expand_beam + Alg. 2 "if h =
 * EOS: remove h from b"): one step of beam-search bookkeeping after
 * the selection, replacing "reorder by parent, then compact" with one
 * gather. Sentence s's winners, in rank order, are out_idx[s, i] =
 * r * V_total + v (-1 = padding) with cost out_cost[s, i] (the outputs of
 * amun_output_layer). A winner whose token v == eos_token finishes (it stays
 * readable in out_idx / out_cost; the caller keeps it as a finished
 * hypothesis) and frees its slot; every other winner becomes row j of the
 * next batch, in sentence order then rank order:
 *   src_row[j] = r (its parent row in the current batch of N rows),
 *   new_token[j] = v, new_cost[j] = out_cost[s, i],
 *   dst rows j of every column = src rows r (duplicated when two winners
 *   share a parent),
 *   new_beam_offsets[s] = number of next-batch rows of sentences < s,
 *   counts = {N', S_alive} on the device (counts_host: optional host copy,
 *   implies a stream synchronisation; otherwise nothing syncs).
 *   out_idx [S, k] int64, out_cost [S, k] fp32, device; 0 <= S, 1 <= k,
 *   S * k <= 2^30; V_total >= 1.
 *   cols    as amun_compact, src [N, row_bytes], dst [>= S*k, row_bytes],
 *           non-overlapping.
 *   src_row, new_token [>= S*k] int32; new_cost [>= S*k] fp32; device.
 *   workspace  amun_beam_advance_workspace_bytes(S, k) bytes, 256-byte
 *           aligned, device scratch (winner flags, parents, tokens).
 * Enqueues 2 kernels (classify, then the compaction gather). EINVAL on
 * argument errors (nothing enqueued). */
size_t amun_beam_advance_workspace_bytes(int S, int k);
amun_status amun_beam_advance(const int64_t* out_idx, const float* out_cost, int S, int k,
                              int64_t V_total, int eos_token, int N, const amun_column* cols,
                              int n_cols, int32_t* new_beam_offsets, int32_t* src_row,
                              int32_t* new_token, float* new_cost, int32_t* counts,
                              int32_t* counts_host, void* workspace, void* stream);

/* 1 in *err if a one-shot wait on `buf` (this rank's own buffer) ever timed
 * out: a peer did not signal a call within 4 s (it failed validation, used
 * another N / G, or never called). The call that timed out wrote no outputs
 * and the exchange is out of step from then on. Synchronous (a blocking
 * device read). Errors: AMUN_EINVAL (NULL), AMUN_ECUDA. */
amun_status amun_oneshot_error(const void* buf, int* err);

/* ------------------------------------------------------------------------
 * NVLink one-shot exchange: the vocab-sharded output
 * layer (Alg. 6; the reduce of P:244-251 applied to the
 * (max, sum, k-best) partial states of P:232-242) with the exchange done by
 * the library's own kernel over peer memory instead of a collective call.
 * In the fused kernel's tail (one cooperative launch; N > 0, tcgen05 plans,
 * AMUN_TAIL not "off"), after every CTA has emitted its partial records, the
 * CTAs combine them into one record per row, store it into slot [rank] of
 * EVERY rank's receive buffer (CUDA IPC mappings: NVLink stores), signal
 * each rank (system-scope release, once per peer from the rank's last CTA),
 * wait for all G ranks' signals (acquire), and run the per-sentence top-k_s
 * over the G records of each row. (N = 0 or AMUN_TAIL=off: the fused kernel,
 * then a separate cooperative one-shot kernel doing the same.) Every rank returns the same result as amun_output_layer_partial on
 * each shard + an all-gather + amun_merge_partials.
 *
 * Buffer: one per rank, from amun_oneshot_alloc (a whole cudaMalloc
 * allocation, zeroed, the one place the library allocates: IPC exports whole
 * allocations), amun_oneshot_buffer_bytes(plan, G) bytes: a 256-byte control
 * block (monotonic per-source signal counters, the rank's call epoch) and
 * fp32 receive records [2][G][max_rows][stride], double-buffered by epoch
 * parity. The counters are never reset: every rank must make the same
 * sequence of calls with the same G (the epochs stay in lockstep), CUDA-graph
 * replays included. The calling processes must be on one node with
 * peer access between their GPUs (NVLink / NVSwitch).
 *
 * amun_oneshot_alloc: *buf = device buffer of this plan's device; if
 *   ipc_handle != NULL, 64 bytes (cudaIpcMemHandle_t) are written there for
 *   the other ranks. Synchronises the device (zeroing). EINVAL / ECUDA.
 * amun_oneshot_open: maps another process's buffer (ipc_handle from its
 *   amun_oneshot_alloc) into this process on `device`; *peer is that
 *   mapping. amun_oneshot_close unmaps it; amun_oneshot_free frees an own
 *   buffer. A process never opens its own handle (use its own pointer).
 * amun_output_layer_oneshot:
 *   plan, X, W, b, prev_cost, beam_offsets, N, S, k_per_sentence, k,
 *   out_idx, out_cost, workspace: as amun_output_layer for this rank's vocab
 *   shard (plan's v_offset / V_local / V_total); N, S, prev_cost,
 *   beam_offsets, k_per_sentence and k are the same on every rank.
 *   bufs    host array [G] of device pointers: bufs[p] = rank p's buffer as
 *           mapped in this process (bufs[rank] = the own buffer), 256-byte
 *           aligned; 1 <= G <= 8, 0 <= rank < G.
 *   Enqueues 1 kernel on `stream` (2 in the fallback forms above). The
 *   call returns before the peers have signalled. A wait is bounded: if a
 *   peer does not signal within 4 s the kernel sets the buffer's error word
 *   (amun_oneshot_error), writes no outputs for that call and exits — the
 *   GPU is never left spinning.
 *   EINVAL on argument errors (nothing enqueued).
 * amun_output_layer_oneshot_emulated (test / measurement hook): G ranks on
 *   ONE GPU. Runs the G shards' fused kernels one after another, then ONE
 *   cooperative launch with a grid row per rank (ranks whose blocks wait on
 *   one another must share a kernel on one GPU). plans[p] / W[p] / b[p] /
 *   workspaces[p] / bufs[p] / out_idx[p] / out_cost[p] are rank p's; the
 *   plans must agree in k_max, max_rows, max_sentences, V_total and device. */
size_t amun_oneshot_buffer_bytes(const amun_ol* plan, int G);
amun_status amun_oneshot_alloc(const amun_ol* plan, int G, void** buf, void* ipc_handle);
amun_status amun_oneshot_free(void* buf);
amun_status amun_oneshot_open(const void* ipc_handle, int device, void** peer);
amun_status amun_oneshot_close(void* peer);
amun_status amun_output_layer_oneshot(amun_ol* plan, const void* X, const void* W, const float* b,
                                      const float* prev_cost, const int32_t* beam_offsets, int N,
                                      int S, const int32_t* k_per_sentence, int k,
                                      void* const* bufs, int G, int rank, int64_t* out_idx,
                                      float* out_cost, void* workspace, void* stream);
amun_status amun_output_layer_oneshot_emulated(amun_ol* const* plans, int G, const void* X,
                                               const void* const* W, const float* const* b,
                                               const float* prev_cost, const int32_t* beam_offsets,
                                               int N, int S, const int32_t* k_per_sentence, int k,
                                               void* const* bufs, int64_t* const* out_idx,
                                               float* const* out_cost, void* const* workspaces,
                                               void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AMUN_H_ */
