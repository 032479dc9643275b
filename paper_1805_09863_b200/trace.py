"""Decode-step trace: the paper's mini-batching comparison (§2.1,
Alg. 1 "Naive mini-batching" P:33-48 vs Alg. 2 "Mini-batching" P:52-73;
Fig. 2 "Time taken for each decoding step for a batch of 1280 sentences",
P:329-338).

The encoder-decoder model is out of scope: decoder
states are synthetic and fixed per hypothesis; each step runs the real hot
path on the live rows:

  dynamic (Alg. 2): output layer on the N_t live rows, then "Remove h from b"
                     = amun_compact of every state column by `alive`
                    (k_s = the sentence's live beam, reading G6);
  naive   (Alg. 1): output layer on all S*B rows every step until every
                    hypothesis has finished (reading G7), no compaction.

Finish schedule (SURVEY.md §8(d) "Config 4 schedule"): hypothesis j of
sentence s is decoded at steps 0 .. f[s, j]-1. Between the two kernels a
synthetic beam bookkeeping step sets prev_cost of live row j of sentence s to
the sentence's j-th best cost of this step (a stand-in for beam reordering);
it is driver glue (torch ops), timed separately from the path's kernels.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import OutputLayer, compact


@dataclass
class TraceStats:
    mode: str
    steps: int = 0
    rows: list = field(default_factory=list)          # N_t per step
    step_ms: list = field(default_factory=list)       # device time of path kernels per step
    glue_ms: list = field(default_factory=list)       # device time of the bookkeeping glue
    compact_ms: list = field(default_factory=list)    # device time of amun_compact per step
    compact_bytes: list = field(default_factory=list) # algorithmic bytes moved by compaction
    total_ms: float = 0.0                             # device time of the whole trace

    @property
    def useful_rows(self) -> int:
        return int(sum(self.rows)) if self.mode == "dynamic" else None

    def summary(self, useful_rows: int) -> dict:
        kern = sum(self.step_ms)
        cms = sum(self.compact_ms)
        cbytes = sum(self.compact_bytes)
        return {
            "mode": self.mode, "steps": self.steps, "rows_decoded": int(sum(self.rows)),
            "useful_rows": useful_rows, "total_ms": self.total_ms, "path_kernels_ms": kern,
            "glue_ms": sum(self.glue_ms), "compact_ms": cms,
            "compact_GBps": (cbytes / (cms * 1e-3) / 1e9) if cms > 0 else None,
            "useful_rows_per_s": useful_rows / (self.total_ms * 1e-3),
            "step_ms": self.step_ms, "rows_per_step": self.rows,
        }


class DecodeTrace:
    """Runs the mini-batching trace on one GPU through the C-ABI."""

    def __init__(self, H: int, V: int, S: int, B: int, *, dtype: str = "bf16",
                 device: int | torch.device = 0, state_floats: int | None = None):
        self.H, self.V, self.S, self.B = H, V, S, B
        self.N0 = S * B
        self.dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.state_floats = 2 * H if state_floats is None else state_floats
        self.ol = OutputLayer(H, V, dtype=dtype, k_max=B, max_rows=self.N0, max_sentences=S,
                              device=self.dev)

    def _ev(self):
        return torch.cuda.Event(enable_timing=True)

    def run(self, X0, W, b, prev0, finish, mode: str = "dynamic", check=None) -> TraceStats:
        """X0 [N0, H], prev0 [N0] fp32, finish [S, B] int64 (steps per hypothesis).
        `check(t, inputs, outputs)` (tests only) sees every step's data."""
        dev, S, B, N0 = self.dev, self.S, self.B, self.N0
        st = TraceStats(mode)
        fin = finish.to(dev).reshape(-1).contiguous()               # by original row id
        T = int(fin.max().item())
        # state columns (ping-pong buffers): X, decoder state, prev_cost, id
        cols = [X0.to(dev).contiguous(),
                torch.zeros(N0, self.state_floats, dtype=torch.float32, device=dev),
                prev0.to(dev).clone(),
                torch.arange(N0, dtype=torch.int64, device=dev)]
        cols[1].copy_(torch.arange(N0, dtype=torch.float32, device=dev)[:, None])
        spare = [torch.empty_like(c) for c in cols]
        offsets = (torch.arange(S + 1, dtype=torch.int32, device=dev) * B).contiguous()
        new_off = torch.empty_like(offsets)
        src_row = torch.empty(N0, dtype=torch.int32, device=dev)
        counts = torch.empty(2, dtype=torch.int32, device=dev)
        row_bytes = sum(c[0:1].numel() * c.element_size() for c in cols)
        N = N0
        t_all0, t_all1 = self._ev(), self._ev()
        evs = []
        torch.cuda.synchronize()
        t_all0.record()
        t = 0
        while N > 0 and t < T:
            X, prev, ids = cols[0][:N], cols[2][:N], cols[3][:N]
            seg = offsets[1:] - offsets[:-1]                          # live beam per sentence
            k_s = seg.to(torch.int32)
            e = [self._ev() for _ in range(4)]
            e[0].record()
            idx, cost = self.ol(X, W, b, prev, offsets, B, k_s)       # steps 1-4 (the path)
            e[1].record()
            # ---- synthetic beam bookkeeping (driver glue, not the path)
            sent = torch.repeat_interleave(torch.arange(S, device=dev), seg.to(torch.int64),
                                           output_size=N)
            slot = torch.arange(N, device=dev) - offsets[:-1].to(torch.int64)[sent]
            newprev = cost[sent, slot]
            if check is not None:
                check(t, (X, W, b, prev, offsets, k_s), (idx, cost))
            prev.copy_(newprev)
            e[2].record()
            if mode == "dynamic":
                alive = (fin[ids] > t + 1).to(torch.uint8)
                compact([(c[:N], d) for c, d in zip(cols, spare)], alive, offsets, new_off, src_row, counts,
                        sync=False)                                       # Alg. 2 removal
                e[3].record()
                n2 = int(counts[0].item())                                # N' to the host
                if check is not None:
                    check(t, ("compact", [c[:N] for c in cols], alive, offsets),
                          ([c[:n2] for c in spare], new_off, src_row[:n2], counts))
                st.compact_bytes.append(N + 2 * n2 * row_bytes + 4 * (n2 + S + 1))
                cols, spare = spare, cols
                offsets, new_off = new_off, offsets
            else:
                e[3].record()
                n2 = N                                                    # Alg. 1: nothing removed
            evs.append(e)
            st.rows.append(N)
            N = n2
            t += 1
        t_all1.record()
        torch.cuda.synchronize()
        for e in evs:
            st.step_ms.append(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]))
            st.glue_ms.append(e[1].elapsed_time(e[2]))
            if mode == "dynamic":
                st.compact_ms.append(e[2].elapsed_time(e[3]))
        st.steps = t
        st.total_ms = t_all0.elapsed_time(t_all1)
        return st

    def run_graph(self, X0, W, b, prev0, finish, log_steps=()) -> TraceStats:
        """Alg. 2 (dynamic) with every step on the device: N stays in device
        memory (amun_output_layer_dev reads it; amun_compact writes it), the
        bookkeeping glue uses fixed shapes over the N0-row buffers, and all
        T_max steps are captured in ONE CUDA graph, timed as one replay.
        Rows per step are logged on the device (they must equal the eager
        dynamic mode's: the finish schedule alone decides them). For the
        steps in log_steps, the step's inputs (X, prev_cost, offsets, k_s, N)
        and outputs (idx, cost) are copied on the device into st.logs (for
        oracle checks of the graph-mode winners; copies are graph nodes)."""
        dev, S, B, N0 = self.dev, self.S, self.B, self.N0
        st = TraceStats("dynamic_graph")
        fin = finish.to(dev).reshape(-1).contiguous()
        T = int(fin.max().item())
        ar = torch.arange(N0, device=dev)
        ar32 = ar.to(torch.int32)

        def fresh():
            cols = [X0.to(dev).contiguous(),
                    torch.zeros(N0, self.state_floats, dtype=torch.float32, device=dev),
                    prev0.to(dev).clone(), torch.arange(N0, dtype=torch.int64, device=dev)]
            cols[1].copy_(torch.arange(N0, dtype=torch.float32, device=dev)[:, None])
            return {"cols": [cols, [torch.empty_like(c) for c in cols]],
                    "off": [(torch.arange(S + 1, dtype=torch.int32, device=dev) * B),
                            torch.empty(S + 1, dtype=torch.int32, device=dev)],
                    "cnt": [torch.tensor([N0, S], dtype=torch.int32, device=dev),
                            torch.empty(2, dtype=torch.int32, device=dev)]}

        idx = torch.empty((S, B), dtype=torch.int64, device=dev)
        cost = torch.empty((S, B), dtype=torch.float32, device=dev)
        k_s = torch.empty(S, dtype=torch.int32, device=dev)
        alive = torch.empty(N0, dtype=torch.uint8, device=dev)
        src_row = torch.empty(N0, dtype=torch.int32, device=dev)
        rows_log = torch.zeros(T, dtype=torch.int32, device=dev)
        logs = {t: {"X": torch.empty_like(X0, device=dev), "prev": torch.empty(N0, device=dev),
                    "off": torch.empty(S + 1, dtype=torch.int32, device=dev),
                    "k_s": torch.empty(S, dtype=torch.int32, device=dev),
                    "N": torch.empty(1, dtype=torch.int32, device=dev),
                    "idx": torch.empty((S, B), dtype=torch.int64, device=dev),
                    "cost": torch.empty((S, B), dtype=torch.float32, device=dev)}
                for t in log_steps if t < T}

        def steps(state):
            for t in range(T):
                a, c = t % 2, (t + 1) % 2
                X, prev, ids = state["cols"][a][0], state["cols"][a][2], state["cols"][a][3]
                off, cnt = state["off"][a], state["cnt"][a]
                torch.sub(off[1:], off[:-1], out=k_s)                       # live beam per sentence
                if t in logs:   # the step's inputs, before the bookkeeping overwrites prev
                    for key, src in (("X", X), ("prev", prev), ("off", off), ("k_s", k_s),
                                     ("N", cnt[:1])):
                        logs[t][key].copy_(src)
                self.ol.call_dev(X, W, b, prev, off, cnt[:1], B, k_s, out_idx=idx, out_cost=cost)
                if t in logs:
                    logs[t]["idx"].copy_(idx)
                    logs[t]["cost"].copy_(cost)
                # synthetic beam bookkeeping (driver glue), fixed shapes over N0 rows
                sent = torch.searchsorted(off[1:], ar32, right=True).clamp_(max=S - 1)
                slot = (ar - off.to(torch.int64)[sent]).clamp_(0, B - 1)
                prev.copy_(cost[sent, slot])
                rows_log[t:t + 1].copy_(cnt[:1])
                torch.logical_and(fin[ids] > t + 1, ar < cnt[0], out=alive.view(torch.bool))
                compact([(x, y) for x, y in zip(state["cols"][a], state["cols"][c])], alive, off,
                        state["off"][c], src_row, state["cnt"][c], sync=False)

        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            steps(fresh())                     # warm-up: kernels, plans, tensor maps
            torch.cuda.synchronize()
            state = fresh()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                steps(state)
        e0, e1 = self._ev(), self._ev()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        st.total_ms = e0.elapsed_time(e1)
        st.rows = [int(n) for n in rows_log.cpu().tolist()]
        st.steps = T
        st.logs = {t: {k: v.cpu() for k, v in d.items()} for t, d in logs.items()}
        self._graph_state = state              # (tests read the final state)
        return st
