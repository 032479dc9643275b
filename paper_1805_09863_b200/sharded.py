"""Vocab-sharded output layer over one process per GPU (torch.distributed).

The paper is single-GPU; its Alg. 6 shards the score vector and
reduces the per-shard (max, best) in a serial step. Here the shards are
vocabulary ranges of W/b on different GPUs: every rank computes the per-row
partial record {m, s, top-k} of its range (amun_output_layer_partial), one
all_gather_into_tensor exchanges the records (N x (2+2k) floats per rank),
and every rank runs the exact merge (amun_merge_partials) in rank order, so
all ranks hold identical results. PyTorch/NCCL is plumbing here; the compute
is the library's kernels.
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
    [world, N, stride] in rank order (the only collective of the path)."""
    if world == 1:
        return partial.unsqueeze(0)
    import torch.distributed as dist
    N = partial.shape[0]
    out = torch.empty((world * N,) + tuple(partial.shape[1:]), dtype=partial.dtype,
                      device=partial.device)
    dist.all_gather_into_tensor(out, partial.contiguous(), group=group)
    return out.view((world, N) + tuple(partial.shape[1:]))


class ShardedOutputLayer:
    """amun_output_layer on world == 1; partial + all-gather + merge otherwise."""

    def __init__(self, H, V, world, rank, *, dtype="bf16", k_max=16, max_rows=1 << 16,
                 max_sentences=1 << 16, device=None, group=None):
        from . import OutputLayer
        self.world, self.rank, self.group = world, rank, group
        self.v0, self.v1 = shard_range(V, world, rank)
        if self.v1 <= self.v0:
            raise ValueError(f"rank {rank} owns no vocabulary (V={V}, world={world})")
        self.ol = OutputLayer(H, self.v1 - self.v0, v_offset=self.v0, V_total=V, dtype=dtype,
                              k_max=k_max, max_rows=max_rows, max_sentences=max_sentences,
                              device=device)
        # kernels of ours per step (the NCCL all-gather kernel is not counted)
        self.launches_per_step = 2 if world == 1 else 3

    def __call__(self, X, W, b, prev_cost, beam_offsets, k, k_per_sentence=None, events=None,
                 out_idx=None, out_cost=None):
        """W, b: this rank's shard. events: optional (start, stop) CUDA events
        recorded around the fused GEMM kernel (stage 1) on the current stream.
        out_idx / out_cost: optional preallocated [S, k] outputs."""
        if self.world == 1 and not events:   # one C-ABI call (amun_output_layer)
            return self.ol(X, W, b, prev_cost, beam_offsets, k, k_per_sentence,
                           out_idx=out_idx, out_cost=out_cost)
        if self.world == 1:
            if events:
                events[0].record()
            self.ol.scores(X, W, b)
            if events:
                events[1].record()
            return self.ol.select(X.shape[0], prev_cost, beam_offsets, k, k_per_sentence,
                                  out_idx=out_idx, out_cost=out_cost)
        if events:
            events[0].record()
        part = self.ol.partial(X, W, b)
        if events:
            events[1].record()
        allp = exchange(part, self.world, self.group)
        return self.ol.merge(allp, prev_cost, beam_offsets, k, k_per_sentence,
                             out_idx=out_idx, out_cost=out_cost)
