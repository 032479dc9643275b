"""Vocab-sharded output layer over one process per GPU (torch.distributed).

The paper is single-GPU; its Alg. 6 shards the score vector and
reduces the per-shard (max, best) in a serial step. Here the shards are
vocabulary ranges of W/b on different GPUs: every rank computes the per-row
partial record {m, s, top-k} of its range (amun_output_layer_partial), one
all_gather_into_tensor exchanges the records (N x (2+2k) floats per rank),
and every rank runs the exact merge (amun_merge_partials) in rank order, so
all ranks hold identical results. PyTorch/NCCL is plumbing here; the compute
is the library's kernels.

exchange="oneshot" replaces the partial + all-gather +
merge with amun_output_layer_oneshot: the library's own kernel stores every
row's record directly into every rank's receive buffer (CUDA IPC mappings over
NVLink), signals, waits and merges. torch.distributed only carries the IPC
handles once, at construction (OneShotExchange).
"""
from __future__ import annotations

import torch


def shard_range(V: int, world: int, rank: int, align: int = 16):
    """Contiguous near-equal vocab range of `rank` (multiples of `align`
    except the last); ranks past the end get an empty range."""
    per = -(-V // world)
    per = -(-per // align) * align
    v0 = min(V, rank * per)
    v1 = min(V, v0 + per)
    return v0, v1


def exchange(partial: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather the [N, stride] partial records of every rank into
    [world, N, stride] in rank order (the only collective of the path). With a
    process group initialised the collective runs even at world 1."""
    import torch.distributed as dist
    if world == 1 and not (dist.is_available() and dist.is_initialized()):
        return partial.unsqueeze(0)
    N = partial.shape[0]
    out = torch.empty((world * N,) + tuple(partial.shape[1:]), dtype=partial.dtype,
                      device=partial.device)
    dist.all_gather_into_tensor(out, partial.contiguous(), group=group)
    return out.view((world, N) + tuple(partial.shape[1:]))


class _CBuffers:
    """The library's one-shot buffer calls (amun_oneshot_alloc / _open /
    _close / _free); tests substitute a fake with the same four methods."""

    def __init__(self):
        from . import _L, check
        self._L, self._check = _L, check

    def alloc(self, plan_handle, world):
        import ctypes
        buf, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        self._check(self._L.amun_oneshot_alloc(plan_handle, world, ctypes.byref(buf), handle))
        return buf.value, handle.raw

    def open(self, handle: bytes, device: int):
        import ctypes
        peer, h = ctypes.c_void_p(), ctypes.create_string_buffer(handle, 64)
        self._check(self._L.amun_oneshot_open(h, device, ctypes.byref(peer)))
        return peer.value

    def close(self, ptr):
        import ctypes
        self._check(self._L.amun_oneshot_close(ctypes.c_void_p(ptr)))

    def free(self, ptr):
        import ctypes
        self._check(self._L.amun_oneshot_free(ctypes.c_void_p(ptr)))


class OneShotExchange:
    """Collective constructor (every rank of `group`): allocates this rank's
    one-shot buffer, all-gathers the 64-byte IPC handles, opens every peer's
    buffer. `ptrs[p]` = rank p's buffer as mapped in this process
    (ptrs[rank] is the own allocation)."""

    def __init__(self, plan_handle, world: int, rank: int, device: int, group=None, lib=None):
        import torch.distributed as dist
        self.lib = lib if lib is not None else _CBuffers()
        self.world, self.rank = world, rank
        self.own, handle = self.lib.alloc(plan_handle, world)
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, handle, group=group)
        else:
            handles = [handle]
        self.ptrs = [self.own if p == rank else self.lib.open(handles[p], device)
                     for p in range(world)]
        if world > 1:   # every buffer zeroed and mapped before anyone signals
            dist.barrier(group=group)

    def error(self) -> bool:
        """True if a wait of this rank ever timed out (amun_oneshot_error;
        synchronous)."""
        import ctypes
        from . import _L, check
        e = ctypes.c_int(0)
        check(_L.amun_oneshot_error(ctypes.c_void_p(self.own), ctypes.byref(e)))
        return bool(e.value)

    def close(self):
        if getattr(self, "ptrs", None) is None:
            return
        for p, ptr in enumerate(self.ptrs):
            if p != self.rank:
                self.lib.close(ptr)
        self.lib.free(self.own)
        self.ptrs = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown: the library may be gone
            pass


class ShardedOutputLayer:
    """amun_output_layer on world == 1; otherwise partial + all-gather + merge
    (exchange="nccl") or the NVLink one-shot kernel (exchange="oneshot")."""

    def __init__(self, H, V, world, rank, *, dtype="bf16", k_max=16, max_rows=1 << 16,
                 max_sentences=1 << 16, device=None, group=None, exchange="nccl",
                 force_sharded=False):
        """force_sharded: run partial + exchange + merge even at world 1 (the
        multi-rank code path on one rank; tests)."""
        from . import OutputLayer
        if exchange not in ("nccl", "oneshot"):
            raise ValueError(f"exchange must be 'nccl' or 'oneshot', not {exchange!r}")
        self.world, self.rank, self.group, self.exchange = world, rank, group, exchange
        self.sharded = world > 1 or force_sharded
        self.v0, self.v1 = shard_range(V, world, rank)
        if self.v1 <= self.v0:
            raise ValueError(f"rank {rank} owns no vocabulary (V={V}, world={world})")
        self.ol = OutputLayer(H, self.v1 - self.v0, v_offset=self.v0, V_total=V, dtype=dtype,
                              k_max=k_max, max_rows=max_rows, max_sentences=max_sentences,
                              device=device)
        # kernels of ours per step (the NCCL all-gather kernel is not counted)
        L = self.ol.launches
        self.launches_per_step = L["partial"] + L["merge"] if self.sharded else L["call"]
        self.oneshot = None
        if exchange == "oneshot":
            dev = self.ol.device.index or 0
            self.oneshot = OneShotExchange(self.ol._h, world, rank, dev, group)
            self.launches_per_step = L["call"]   # the exchange runs in the fused kernel's tail
        self._part = None

    def __call__(self, X, W, b, prev_cost, beam_offsets, k, k_per_sentence=None, events=None,
                 out_idx=None, out_cost=None, stage_events=None):
        """W, b: this rank's shard. events: optional (start, stop) CUDA events
        recorded around the fused GEMM kernel (stage 1) on the current stream.
        stage_events (sharded path): 4 events recorded before the partial
        kernel, after it, after the exchange and after the merge.
        out_idx / out_cost: optional preallocated [S, k] outputs."""
        if self.oneshot is not None:
            return self.ol.oneshot(X, W, b, prev_cost, beam_offsets, k, self.oneshot.ptrs,
                                   self.rank, k_per_sentence, out_idx=out_idx, out_cost=out_cost)
        if not self.sharded and not events:   # one C-ABI call (amun_output_layer)
            return self.ol(X, W, b, prev_cost, beam_offsets, k, k_per_sentence,
                           out_idx=out_idx, out_cost=out_cost)
        if not self.sharded:
            events[0].record()
            self.ol.scores(X, W, b)
            events[1].record()
            return self.ol.select(X.shape[0], prev_cost, beam_offsets, k, k_per_sentence,
                                  out_idx=out_idx, out_cost=out_cost)
        ev = stage_events or ((events[0], events[1]) + (None, None) if events else None)
        N = X.shape[0]
        if self._part is None or self._part.shape[0] != N:
            self._part = torch.empty((N, self.ol.stride), dtype=torch.float32,
                                     device=self.ol.device)
        if ev and ev[0] is not None:
            ev[0].record()
        part = self.ol.partial(X, W, b, out=self._part)
        if ev and ev[1] is not None:
            ev[1].record()
        allp = exchange(part, self.world, self.group)
        if ev and ev[2] is not None:
            ev[2].record()
        res = self.ol.merge(allp, prev_cost, beam_offsets, k, k_per_sentence,
                            out_idx=out_idx, out_cost=out_cost)
        if ev and ev[3] is not None:
            ev[3].record()
        return res


class EmulatedOneShot:
    """G ranks of the one-shot path on ONE GPU (test / measurement hook,
    amun_output_layer_oneshot_emulated): the G shards' fused kernels in
    sequence, then one cooperative kernel with a grid row per rank. Keeps
    the G buffers across calls (their epochs advance like real ranks')."""

    def __init__(self, layers):
        import ctypes
        from . import _L, check
        self.layers, self.G = list(layers), len(layers)
        self._L, self._check = _L, check
        self.bufs = []
        for ol in self.layers:
            buf = ctypes.c_void_p()
            check(_L.amun_oneshot_alloc(ol._h, self.G, ctypes.byref(buf), None))
            self.bufs.append(buf.value)

    def __call__(self, X, Ws, bs, prev_cost, beam_offsets, k, k_per_sentence=None, outs=None):
        import ctypes
        from . import _ptr, _stream
        G, ol0 = self.G, self.layers[0]
        N = X.shape[0]
        S = beam_offsets.shape[0] - 1
        for ol, W, b in zip(self.layers, Ws, bs):
            ol._check_scores(X, W, b)
        if outs is None:
            outs = [ol0._outputs(S, k, None, None) for _ in range(G)]
        vp = ctypes.c_void_p
        arr = lambda xs: (vp * G)(*[vp(x) for x in xs])
        self._check(self._L.amun_output_layer_oneshot_emulated(
            arr([ol._h.value for ol in self.layers]), G, _ptr(X), arr([W.data_ptr() for W in Ws]),
            arr([b.data_ptr() for b in bs]), _ptr(prev_cost), _ptr(beam_offsets), N, S,
            _ptr(k_per_sentence), k, arr(self.bufs), arr([o[0].data_ptr() for o in outs]),
            arr([o[1].data_ptr() for o in outs]),
            arr([ol.workspace.data_ptr() for ol in self.layers]), _stream(ol0.device)))
        return outs

    def close(self):
        import ctypes
        for p in getattr(self, "bufs", []):
            self._check(self._L.amun_oneshot_free(ctypes.c_void_p(p)))
        self.bufs = []

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter shutdown: the library may be gone
            pass
