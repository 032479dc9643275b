"""B200-native NMT output-layer hot path (arXiv 1805.09863, Amun @ WNMT 2018).

Thin Python binding over the C-ABI in include/amun.h (libamun.so). It only
marshals arguments: tensors become device pointers, the stream is torch's
current stream. Every step of the path runs in the library's sm_100a kernels;
there is no CPU fallback (a missing library raises on import).

    ol = OutputLayer(H, V, k_max=5, max_rows=640, max_sentences=128)
    idx, cost = ol(X, W, b, prev_cost, beam_offsets, k=5)      # steps 1-4
    n_alive, s_alive = compact([(src, dst), ...], alive, offsets, new_offsets, src_row)
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import AMUN_MAX_COLUMNS, AMUN_MAX_K, AmunError, check

_L = _lib.load()

__all__ = ["OutputLayer", "compact", "compact_sentences", "beam_advance", "quantize_e4m3",
           "quantize_mxfp4", "mxfp4_sf_bytes", "split_tf32x3", "AmunError", "AMUN_MAX_K",
           "AMUN_MAX_COLUMNS", "lib_path"]

lib_path = _lib.LIB_PATH


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _need(t, name, dtype, device, shape=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


class OutputLayer:
    """Plan for one vocabulary shard [v_offset, v_offset + V_local) of V_total.

    dtype "bf16": X, W bfloat16 (tcgen05 tensor cores, fp32 accumulate).
    dtype "f32" : X, W float32 (SIMT, true fp32 products).
    """

    def __init__(self, H: int, V_local: int, *, v_offset: int = 0, V_total: int | None = None,
                 dtype: str = "bf16", k_max: int = 16, max_rows: int = 1 << 16,
                 max_sentences: int = 1 << 16, device: int | torch.device | None = 0):
        if device is None:
            device = torch.cuda.current_device()
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.device = dev
        self.H, self.V_local, self.v_offset = H, V_local, v_offset
        self.V_total = V_local if V_total is None else V_total
        self.dtype = dtype
        self.tdtype = {"bf16": torch.bfloat16, "f32": torch.float32, "e4m3": torch.uint8,
                       "tf32x3": torch.float32, "mxfp4": torch.uint8}[dtype]
        self.K = 3 * H if dtype == "tf32x3" else H   # columns of X / W rows as passed
        self.k_max, self.max_rows, self.max_sentences = k_max, max_rows, max_sentences
        h = ctypes.c_void_p()
        check(_L.amun_ol_create(ctypes.byref(h), H, V_local, v_offset, self.V_total,
                                {"bf16": _lib.AMUN_BF16, "f32": _lib.AMUN_F32,
                                 "e4m3": _lib.AMUN_E4M3, "tf32x3": _lib.AMUN_TF32X3,
                                 "mxfp4": _lib.AMUN_MXFP4}[dtype],
                                k_max, max_rows, max_sentences, dev.index or 0))
        self._h = h
        self.stride = _L.amun_ol_partial_stride(h)
        nbytes = _L.amun_ol_workspace_bytes(h)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        # the workspace is plan state (amun.h): initialised once, kept between calls
        if hasattr(_L, "amun_ol_workspace_init"):   # (absent only in older A/B builds)
            check(_L.amun_ol_workspace_init(h, _ptr(self.workspace), _stream(dev)))
        # kernels one call enqueues: __call__ / argmax, partial, merge
        self.launches = ({c: _L.amun_ol_launches_per_call(h, i)
                          for i, c in enumerate(("call", "partial", "merge"))}
                         if hasattr(_L, "amun_ol_launches_per_call")
                         else {"call": 2, "partial": 2, "merge": 1})

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _L is not None:   # (_L is None at interpreter exit)
            _L.amun_ol_destroy(h)
            self._h = None

    # ------------------------------------------------------------- checks
    def _check_scores(self, X, W, b):
        N = X.shape[0]
        _need(X, "X", self.tdtype, self.device, (N, self.K))
        _need(W, "W", self.tdtype, self.device, (self.V_local, self.K))
        _need(b, "b", torch.float32, self.device, (self.V_local,))
        return N

    def _outputs(self, S, k, out_idx, out_cost):
        if out_idx is None:
            out_idx = torch.empty((S, k), dtype=torch.int64, device=self.device)
        if out_cost is None:
            out_cost = torch.empty((S, k), dtype=torch.float32, device=self.device)
        _need(out_idx, "out_idx", torch.int64, self.device, (S, k))
        _need(out_cost, "out_cost", torch.float32, self.device, (S, k))
        return out_idx, out_cost

    def _check_select(self, prev_cost, beam_offsets, N, k_per_sentence):
        S = beam_offsets.shape[0] - 1
        _need(prev_cost, "prev_cost", torch.float32, self.device, (N,))
        _need(beam_offsets, "beam_offsets", torch.int32, self.device)
        if k_per_sentence is not None:
            _need(k_per_sentence, "k_per_sentence", torch.int32, self.device, (S,))
        return S

    # ------------------------------------------------------------- calls
    def __call__(self, X, W, b, prev_cost, beam_offsets, k: int, k_per_sentence=None,
                 out_idx=None, out_cost=None):
        """Steps 1-4: returns (idx [S,k] int64 = row*V_total + token, cost [S,k] fp32)."""
        N = self._check_scores(X, W, b)
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_output_layer(self._h, _ptr(X), _ptr(W), _ptr(b), _ptr(prev_cost),
                                   _ptr(beam_offsets), N, S, _ptr(k_per_sentence), k,
                                   _ptr(out_idx), _ptr(out_cost), _ptr(self.workspace),
                                   _stream(self.device)))
        return out_idx, out_cost

    def oneshot(self, X, W, b, prev_cost, beam_offsets, k: int, bufs, rank: int,
                k_per_sentence=None, out_idx=None, out_cost=None):
        """Steps 1-4 of this rank's vocab shard with the NVLink one-shot
        exchange + merge (amun_output_layer_oneshot, NEXT f3). bufs: every
        rank's one-shot buffer as mapped here (device pointers, rank order;
        sharded.OneShotExchange). Every rank makes the same call."""
        N = self._check_scores(X, W, b)
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        arr = (ctypes.c_void_p * len(bufs))(*[int(p) for p in bufs])
        check(_L.amun_output_layer_oneshot(self._h, _ptr(X), _ptr(W), _ptr(b), _ptr(prev_cost),
                                           _ptr(beam_offsets), N, S, _ptr(k_per_sentence), k,
                                           arr, len(bufs), rank, _ptr(out_idx), _ptr(out_cost),
                                           _ptr(self.workspace), _stream(self.device)))
        return out_idx, out_cost

    def call_dev(self, X, W, b, prev_cost, beam_offsets, N_dev, k: int, k_per_sentence=None,
                 out_idx=None, out_cost=None):
        """Steps 1-4 with the row count on the device (N = N_dev[0], no host
        sync): X [max_rows, H], prev_cost [max_rows]; rows >= N are ignored."""
        M = self.max_rows
        _need(X, "X", self.tdtype, self.device, (M, self.K))
        _need(W, "W", self.tdtype, self.device, (self.V_local, self.K))
        _need(b, "b", torch.float32, self.device, (self.V_local,))
        _need(N_dev, "N_dev", torch.int32, self.device)
        S = self._check_select(prev_cost, beam_offsets, M, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_output_layer_dev(self._h, _ptr(X), _ptr(W), _ptr(b), _ptr(prev_cost),
                                       _ptr(beam_offsets), _ptr(N_dev), S, _ptr(k_per_sentence), k,
                                       _ptr(out_idx), _ptr(out_cost), _ptr(self.workspace),
                                       _stream(self.device)))
        return out_idx, out_cost

    def _check_e4m3(self, X8, xs, W8, ws, b):
        N = self._check_scores(X8, W8, b)
        _need(xs, "x_scale", torch.float32, self.device, (N,))
        _need(ws, "w_scale", torch.float32, self.device, (self.V_local,))
        return N

    def call_e4m3(self, X8, x_scale, W8, w_scale, b, prev_cost, beam_offsets, k: int,
                  k_per_sentence=None, out_idx=None, out_cost=None):
        """FP8 steps 1-4 (plan dtype "e4m3"): X8 / W8 uint8 E4M3 codes with
        per-row fp32 scales (see quantize_e4m3). Returns (idx, cost)."""
        N = self._check_e4m3(X8, x_scale, W8, w_scale, b)
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_output_layer_e4m3(self._h, _ptr(X8), _ptr(x_scale), _ptr(W8), _ptr(w_scale),
                                        _ptr(b), _ptr(prev_cost), _ptr(beam_offsets), N, S,
                                        _ptr(k_per_sentence), k, _ptr(out_idx), _ptr(out_cost),
                                        _ptr(self.workspace), _stream(self.device)))
        return out_idx, out_cost

    def scores_e4m3(self, X8, x_scale, W8, w_scale, b, variant: int = 0):
        """FP8 stage 1 (variant 0), or the bare-GEMM (2) / no-k-best (3) builds."""
        N = self._check_e4m3(X8, x_scale, W8, w_scale, b)
        check(_L.amun_ol_scores_e4m3(self._h, _ptr(X8), _ptr(x_scale), _ptr(W8), _ptr(w_scale),
                                     _ptr(b), N, variant, _ptr(self.workspace), _stream(self.device)))

    def partial_e4m3(self, X8, x_scale, W8, w_scale, b, out=None):
        """FP8 vocab-shard piece 1: per-row partial record [N, stride] fp32."""
        N = self._check_e4m3(X8, x_scale, W8, w_scale, b)
        if out is None:
            out = torch.empty((N, self.stride), dtype=torch.float32, device=self.device)
        _need(out, "partial", torch.float32, self.device, (N, self.stride))
        check(_L.amun_output_layer_partial_e4m3(self._h, _ptr(X8), _ptr(x_scale), _ptr(W8),
                                                _ptr(w_scale), _ptr(b), N, _ptr(out),
                                                _ptr(self.workspace), _stream(self.device)))
        return out

    def argmax_e4m3(self, X8, x_scale, W8, w_scale, b, out_token=None, out_logit=None):
        """FP8 greedy argmax (Alg. 5): (token [N] int64, scaled biased logit [N] fp32)."""
        N = self._check_e4m3(X8, x_scale, W8, w_scale, b)
        if out_token is None:
            out_token = torch.empty(N, dtype=torch.int64, device=self.device)
        if out_logit is None:
            out_logit = torch.empty(N, dtype=torch.float32, device=self.device)
        check(_L.amun_argmax_e4m3(self._h, _ptr(X8), _ptr(x_scale), _ptr(W8), _ptr(w_scale),
                                  _ptr(b), N, _ptr(out_token), _ptr(out_logit),
                                  _ptr(self.workspace), _stream(self.device)))
        return out_token, out_logit

    # ------------------------------------------------ MXFP4 W (amun_*_mxfp4)
    def _check_mxfp4(self, X8, xs, W4, w_sf, b):
        N = X8.shape[0]
        _need(X8, "X8", torch.uint8, self.device, (N, self.H))
        _need(W4, "W4", torch.uint8, self.device, (self.V_local, self.H // 2))
        _need(w_sf, "w_sf", torch.uint8, self.device, (_L.amun_mxfp4_sf_bytes(self.V_local, self.H),))
        _need(xs, "x_scale", torch.float32, self.device, (N,))
        _need(b, "b", torch.float32, self.device, (self.V_local,))
        return N

    def call_mxfp4(self, X8, x_scale, W4, w_sf, b, prev_cost, beam_offsets, k: int,
                   k_per_sentence=None, out_idx=None, out_cost=None):
        """Steps 1-4 for plan dtype "mxfp4": X8 E4M3 codes + per-row scales
        (quantize_e4m3), W4 / w_sf from quantize_mxfp4. Returns (idx, cost)."""
        N = self._check_mxfp4(X8, x_scale, W4, w_sf, b)
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_output_layer_mxfp4(self._h, _ptr(X8), _ptr(x_scale), _ptr(W4), _ptr(w_sf),
                                         _ptr(b), _ptr(prev_cost), _ptr(beam_offsets), N, S,
                                         _ptr(k_per_sentence), k, _ptr(out_idx), _ptr(out_cost),
                                         _ptr(self.workspace), _stream(self.device)))
        return out_idx, out_cost

    def scores_mxfp4(self, X8, x_scale, W4, w_sf, b, variant: int = 0):
        """MXFP4 stage 1 (variant 0), or the bare-GEMM (2) / no-k-best (3) builds."""
        N = self._check_mxfp4(X8, x_scale, W4, w_sf, b)
        check(_L.amun_ol_scores_mxfp4(self._h, _ptr(X8), _ptr(x_scale), _ptr(W4), _ptr(w_sf),
                                      _ptr(b), N, variant, _ptr(self.workspace),
                                      _stream(self.device)))

    def argmax_mxfp4(self, X8, x_scale, W4, w_sf, b, out_token=None, out_logit=None):
        """MXFP4 greedy argmax (Alg. 5): (token [N] int64, logit [N] fp32)."""
        N = self._check_mxfp4(X8, x_scale, W4, w_sf, b)
        if out_token is None:
            out_token = torch.empty(N, dtype=torch.int64, device=self.device)
        if out_logit is None:
            out_logit = torch.empty(N, dtype=torch.float32, device=self.device)
        check(_L.amun_argmax_mxfp4(self._h, _ptr(X8), _ptr(x_scale), _ptr(W4), _ptr(w_sf),
                                   _ptr(b), N, _ptr(out_token), _ptr(out_logit),
                                   _ptr(self.workspace), _stream(self.device)))
        return out_token, out_logit

    def debug_logits_mxfp4(self, X8, x_scale, W4, w_sf, b):
        """Test hook: the biased logits [N, V_local] fp32 of the MXFP4 GEMM."""
        N = self._check_mxfp4(X8, x_scale, W4, w_sf, b)
        out = torch.empty((N, self.V_local), dtype=torch.float32, device=self.device)
        check(_L.amun_debug_logits_mxfp4(self._h, _ptr(X8), _ptr(x_scale), _ptr(W4), _ptr(w_sf),
                                         _ptr(b), N, _ptr(out), _ptr(self.workspace),
                                         _stream(self.device)))
        return out

    def scores(self, X, W, b):
        """Stage 1 only (fused GEMM + bias + online softmax stats + row k-best)."""
        N = self._check_scores(X, W, b)
        check(_L.amun_ol_scores(self._h, _ptr(X), _ptr(W), _ptr(b), N, _ptr(self.workspace),
                                _stream(self.device)))

    def select(self, N, prev_cost, beam_offsets, k: int, k_per_sentence=None, out_idx=None,
               out_cost=None):
        """Stage 2 only (merge + per-sentence selection) on the last scores()."""
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_ol_select(self._h, _ptr(self.workspace), _ptr(prev_cost),
                                _ptr(beam_offsets), N, S, _ptr(k_per_sentence), k,
                                _ptr(out_idx), _ptr(out_cost), _stream(self.device)))
        return out_idx, out_cost

    def partial(self, X, W, b, out=None):
        """Vocab-shard piece 1: per-row partial record [N, stride] fp32."""
        N = self._check_scores(X, W, b)
        if out is None:
            out = torch.empty((N, self.stride), dtype=torch.float32, device=self.device)
        _need(out, "partial", torch.float32, self.device, (N, self.stride))
        check(_L.amun_output_layer_partial(self._h, _ptr(X), _ptr(W), _ptr(b), N, _ptr(out),
                                           _ptr(self.workspace), _stream(self.device)))
        return out

    def merge(self, partials, prev_cost, beam_offsets, k: int, k_per_sentence=None,
              out_idx=None, out_cost=None):
        """Vocab-shard piece 2: partials [G, N, stride] -> (idx, cost)."""
        if partials.dim() != 3 or partials.shape[2] != self.stride:
            raise ValueError(f"partials must be [G, N, {self.stride}]")
        G, N = partials.shape[0], partials.shape[1]
        _need(partials, "partials", torch.float32, self.device)
        S = self._check_select(prev_cost, beam_offsets, N, k_per_sentence)
        out_idx, out_cost = self._outputs(S, k, out_idx, out_cost)
        check(_L.amun_merge_partials(self._h, _ptr(partials), G, _ptr(prev_cost),
                                     _ptr(beam_offsets), N, S, _ptr(k_per_sentence), k,
                                     _ptr(out_idx), _ptr(out_cost), _stream(self.device)))
        return out_idx, out_cost

    def bench_variant(self, X, W, b, variant: int):
        """Benchmark hook: 2 = bare GEMM, 3 = GEMM + bias + softmax stats (no k-best),
        4 = the argmax (Alg. 5) fused kernel alone."""
        N = self._check_scores(X, W, b)
        check(_L.amun_bench_variant(self._h, _ptr(X), _ptr(W), _ptr(b), N, variant,
                                    _ptr(self.workspace), _stream(self.device)))

    def argmax(self, X, W, b, out_token=None, out_logit=None):
        """Greedy decoding, Alg. 5: per row the token with the
        largest biased logit (lowest id on ties), no softmax. Returns
        (token [N] int64, logit [N] fp32 = (W x + b)[token])."""
        N = self._check_scores(X, W, b)
        if out_token is None:
            out_token = torch.empty(N, dtype=torch.int64, device=self.device)
        if out_logit is None:
            out_logit = torch.empty(N, dtype=torch.float32, device=self.device)
        check(_L.amun_argmax(self._h, _ptr(X), _ptr(W), _ptr(b), N, _ptr(out_token),
                             _ptr(out_logit), _ptr(self.workspace), _stream(self.device)))
        return out_token, out_logit

    def debug_logits(self, X, W, b):
        """Test hook: the biased logits [N, V_local] of the same GEMM."""
        N = self._check_scores(X, W, b)
        out = torch.empty((N, self.V_local), dtype=torch.float32, device=self.device)
        check(_L.amun_debug_logits(self._h, _ptr(X), _ptr(W), _ptr(b), N, _ptr(out),
                                   _ptr(self.workspace), _stream(self.device)))
        return out


def compact(columns, alive, beam_offsets, new_offsets=None, src_row=None, counts=None,
            sync: bool = True):
    """Alg. 2 "Remove h from b": stable compaction of every (src, dst) column
    pair (2-D tensors, row = hypothesis) by the uint8 `alive` mask.
    Returns (N', S_alive, new_offsets, src_row, counts); with sync=False the
    first two are None and the counts stay on the device (no host sync)."""
    N = alive.shape[0]
    dev = alive.device
    S = beam_offsets.shape[0] - 1
    _need(alive, "alive", torch.uint8, dev, (N,))
    _need(beam_offsets, "beam_offsets", torch.int32, dev)
    if new_offsets is None:
        new_offsets = torch.empty(S + 1, dtype=torch.int32, device=dev)
    if src_row is None:
        src_row = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    if counts is None:
        counts = torch.empty(2, dtype=torch.int32, device=dev)
    if len(columns) > AMUN_MAX_COLUMNS:
        raise ValueError(f"at most {AMUN_MAX_COLUMNS} columns per call")
    arr = (_lib.amun_column * max(1, len(columns)))()
    for i, (src, dst) in enumerate(columns):
        if src.shape[0] != N or not src.is_contiguous() or not dst.is_contiguous():
            raise ValueError(f"column {i}: src must have N rows; src/dst contiguous")
        rb = src.element_size()
        for d in src.shape[1:]:
            rb *= int(d)
        if dst.numel() * dst.element_size() < rb * N:
            raise ValueError(f"column {i}: dst too small")
        arr[i] = _lib.amun_column(src.data_ptr(), dst.data_ptr(), rb)
    host = (ctypes.c_int32 * 2)() if sync else None
    check(_L.amun_compact(arr, len(columns), _ptr(alive), N, _ptr(beam_offsets), S,
                          _ptr(new_offsets), _ptr(src_row), _ptr(counts),
                          ctypes.cast(host, ctypes.c_void_p) if sync else None,
                          _stream(dev)))
    if sync:
        return int(host[0]), int(host[1]), new_offsets, src_row, counts
    return None, None, new_offsets, src_row, counts


def compact_sentences(columns, new_offsets, sync: bool = True):
    """Sentence-level columns (one row per sentence: encoder context, source
    lengths) after a row compaction: keep the sentences that still have rows
    (new_offsets [S+1] from compact / beam_advance), stably
    (amun_sentence_alive + amun_compact). Returns (S_kept, src_sentence,
    counts); with sync=False S_kept is None (no host sync)."""
    dev = new_offsets.device
    S = new_offsets.shape[0] - 1
    _need(new_offsets, "new_offsets", torch.int32, dev, (S + 1,))
    alive_s = torch.empty(max(S, 1), dtype=torch.uint8, device=dev)
    unit = torch.empty(S + 1, dtype=torch.int32, device=dev)
    check(_L.amun_sentence_alive(_ptr(new_offsets), S, _ptr(alive_s), _ptr(unit), _stream(dev)))
    n, _, _, src, counts = compact(columns, alive_s[:S], unit, sync=sync)
    return n, src, counts


def beam_advance(out_idx, out_cost, V_total: int, eos: int, N: int, columns=(), sync: bool = True,
                 out=None):
    """Beam advance (SPEC S:324-332 expand_beam + Alg. 2): from the selected
    winners out_idx / out_cost [S, k] (amun_output_layer's outputs), the next
    batch = every non-EOS winner, in sentence then rank order, with its parent
    row's state gathered from each (src [N, ...], dst [>= S*k, ...]) column.
    Returns (N', S_alive, new_offsets [S+1], src_row, new_token, new_cost,
    counts); with sync=False the first two are None (no host sync)."""
    dev = out_idx.device
    S, k = out_idx.shape
    _need(out_idx, "out_idx", torch.int64, dev, (S, k))
    _need(out_cost, "out_cost", torch.float32, dev, (S, k))
    n = max(S * k, 1)
    if out is None:
        out = {}
    def buf(name, size, dtype):
        t = out.get(name)
        return torch.empty(size, dtype=dtype, device=dev) if t is None else t
    new_offsets = buf("new_offsets", S + 1, torch.int32)
    src_row = buf("src_row", n, torch.int32)
    new_token = buf("new_token", n, torch.int32)
    new_cost = buf("new_cost", n, torch.float32)
    counts = buf("counts", 2, torch.int32)
    ws = out.get("workspace")
    if ws is None:
        ws = torch.empty(max(_L.amun_beam_advance_workspace_bytes(S, k), 256), dtype=torch.uint8,
                         device=dev)
    if len(columns) > AMUN_MAX_COLUMNS:
        raise ValueError(f"at most {AMUN_MAX_COLUMNS} columns per call")
    arr = (_lib.amun_column * max(1, len(columns)))()
    for i, (src, dst) in enumerate(columns):
        if src.shape[0] != N or not src.is_contiguous() or not dst.is_contiguous():
            raise ValueError(f"column {i}: src must have N rows; src/dst contiguous")
        rb = src.element_size()
        for d in src.shape[1:]:
            rb *= int(d)
        if dst.numel() * dst.element_size() < rb * S * k:
            raise ValueError(f"column {i}: dst must hold S*k rows")
        arr[i] = _lib.amun_column(src.data_ptr(), dst.data_ptr(), rb)
    host = (ctypes.c_int32 * 2)() if sync else None
    check(_L.amun_beam_advance(_ptr(out_idx), _ptr(out_cost), S, k, V_total, eos, N, arr,
                               len(columns), _ptr(new_offsets), _ptr(src_row), _ptr(new_token),
                               _ptr(new_cost), _ptr(counts),
                               ctypes.cast(host, ctypes.c_void_p) if sync else None, _ptr(ws),
                               _stream(dev)))
    if sync:
        return int(host[0]), int(host[1]), new_offsets, src_row, new_token, new_cost, counts
    return None, None, new_offsets, src_row, new_token, new_cost, counts


def quantize_e4m3(src, out=None, scale=None):
    """Per-row E4M3 quantisation on the GPU (amun_quantize_e4m3): src [R, H]
    fp32 or bf16 -> (codes [R, H] uint8, scale [R] fp32) with
    src ~= codes * scale[:, None]."""
    if src.dim() != 2 or not src.is_contiguous() or src.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("src must be a contiguous 2-D fp32 or bf16 tensor")
    R, H = src.shape
    dev = src.device
    if out is None:
        out = torch.empty((R, H), dtype=torch.uint8, device=dev)
    if scale is None:
        scale = torch.empty(R, dtype=torch.float32, device=dev)
    _need(out, "out", torch.uint8, dev, (R, H))
    _need(scale, "scale", torch.float32, dev, (R,))
    check(_L.amun_quantize_e4m3(_ptr(src), _lib.AMUN_BF16 if src.dtype == torch.bfloat16 else _lib.AMUN_F32,
                                R, H, _ptr(out), _ptr(scale), _stream(dev)))
    return out, scale


def mxfp4_sf_bytes(R: int, H: int) -> int:
    """Bytes of the MXFP4 scale-atom array of R rows of H values (amun.h)."""
    return int(_L.amun_mxfp4_sf_bytes(R, H))


def quantize_mxfp4(src, codes=None, sf=None):
    """OCP MXFP4 quantisation on the GPU (amun_quantize_mxfp4): src [R, H]
    fp32 or bf16, H % 128 == 0 -> (codes [R, H/2] uint8, two E2M1 codes per
    byte, low nibble first; sf [mxfp4_sf_bytes(R, H)] uint8 E8M0 scales in the
    kernel's atom layout)."""
    if src.dim() != 2 or not src.is_contiguous() or src.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("src must be a contiguous 2-D fp32 or bf16 tensor")
    R, H = src.shape
    dev = src.device
    if codes is None:
        codes = torch.empty((R, H // 2), dtype=torch.uint8, device=dev)
    if sf is None:
        sf = torch.empty(mxfp4_sf_bytes(R, H), dtype=torch.uint8, device=dev)
    _need(codes, "codes", torch.uint8, dev, (R, H // 2))
    _need(sf, "sf", torch.uint8, dev, (mxfp4_sf_bytes(R, H),))
    check(_L.amun_quantize_mxfp4(_ptr(src), _lib.AMUN_BF16 if src.dtype == torch.bfloat16 else _lib.AMUN_F32,
                                 R, H, _ptr(codes), _ptr(sf), _stream(dev)))
    return codes, sf


def split_tf32x3(src, role: str, out=None):
    """3xTF32 split for dtype="tf32x3" plans (amun_split_tf32x3): src [R, H]
    fp32 -> [R, 3H] fp32 rows [hi | hi | lo] (role "X") or [hi | lo | hi]
    (role "W"), hi = tf32(x), lo = tf32(x - hi)."""
    if src.dim() != 2 or src.dtype != torch.float32 or not src.is_contiguous():
        raise ValueError("src must be a contiguous 2-D fp32 tensor")
    R, H = src.shape
    if out is None:
        out = torch.empty((R, 3 * H), dtype=torch.float32, device=src.device)
    _need(out, "out", torch.float32, src.device, (R, 3 * H))
    check(_L.amun_split_tf32x3(_ptr(src), R, H, {"X": 0, "W": 1}[role], _ptr(out),
                               _stream(src.device)))
    return out
