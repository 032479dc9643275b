"""Standalone compaction benchmark: N = 6400 rows of the
cfg4 per-hypothesis state (x bf16 2048 B + decoder state 8192 B + prev_cost
4 B + id 8 B = 10,252 B/row), alive masks: i.i.d. survival p in {0.99, 0.9,
0.5, 0.1}, the cfg4 schedule at t in {5, 20, 40}, all-alive, none-alive.
Achieved GB/s = (N + 2 N' 10252 + 4 (N' + S + 1)) / t against the measured HBM
peak. Device time per call from a CUDA graph of 50 calls (no host sync)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

N, B = 6400, 5
S = N // B
dev = torch.device("cuda", 0)
cols = [torch.randn(N, 1024, device=dev).to(torch.bfloat16), torch.randn(N, 2048, device=dev),
        torch.randn(N, device=dev), torch.arange(N, dtype=torch.int64, device=dev)]
dst = [torch.empty_like(c) for c in cols]
row_bytes = sum(c[0:1].numel() * c.element_size() for c in cols)
off = (torch.arange(S + 1, dtype=torch.int32, device=dev) * B)
new_off = torch.empty_like(off)
src_row = torch.empty(N, dtype=torch.int32, device=dev)
counts = torch.empty(2, dtype=torch.int32, device=dev)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    "MEASURED_PEAKS.json") else 6454.3
f = synth.eos_schedule(synth.BASE_SEED + 4, S, B).reshape(-1)
masks = {f"iid p={p}": synth.gen_alive(int(p * 100), N, p).to(dev) for p in (0.99, 0.9, 0.5, 0.1)}
for t in (5, 20, 40):
    masks[f"trace t={t}"] = (f > t).to(torch.uint8).to(dev)
masks["all-alive"] = torch.ones(N, dtype=torch.uint8, device=dev)
masks["none-alive"] = torch.zeros(N, dtype=torch.uint8, device=dev)
res = []
for name, alive in masks.items():
    def call():
        amun.compact(list(zip(cols, dst)), alive, off, new_off, src_row, counts, sync=False)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(50):
                call()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    n2 = int(alive.sum().item())
    byts = N + 2 * n2 * row_bytes + 4 * (n2 + S + 1)
    res.append({"mask": name, "N_alive": n2, "us": round(us, 2), "GBps": round(byts / (us * 1e-6) / 1e9, 1),
                "frac": round(byts / (us * 1e-6) / 1e9 / peak, 3)})
    print(json.dumps(res[-1]))

# ---- beam advance (amun_beam_advance, NEXT f1): the cfg4 batch's winners
# S x k = 1280 x 5 (parents inside each sentence's 5 rows, repeats allowed),
# EOS fraction p; the same 4 state columns gathered by parent row.
# Algorithmic bytes = S k (8 + 4) (winners) + 2 N' row_bytes + N' (4 + 4 + 4) + 4 (S + 1).
gen = torch.Generator().manual_seed(7)
dst_adv = [torch.empty_like(c) for c in cols]
ws = torch.empty(max(amun._L.amun_beam_advance_workspace_bytes(S, B), 256), dtype=torch.uint8, device=dev)
outs = {"new_offsets": torch.empty(S + 1, dtype=torch.int32, device=dev),
        "src_row": torch.empty(N, dtype=torch.int32, device=dev),
        "new_token": torch.empty(N, dtype=torch.int32, device=dev),
        "new_cost": torch.empty(N, dtype=torch.float32, device=dev),
        "counts": torch.empty(2, dtype=torch.int32, device=dev), "workspace": ws}
V, EOS = 90000, 2
for p in (0.0, 0.1, 0.5, 0.9):
    parent = (torch.arange(S)[:, None] * B + torch.randint(0, B, (S, B), generator=gen))
    tok = torch.randint(0, V, (S, B), generator=gen)
    tok[torch.rand((S, B), generator=gen) < p] = EOS
    idx = (parent * V + tok).to(dev)
    cost = (-torch.rand((S, B), generator=gen) * 20).to(dev)

    def call():
        amun.beam_advance(idx, cost, V, EOS, N, list(zip(cols, dst_adv)), sync=False, out=outs)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(50):
                call()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    n2 = int((tok != EOS).sum())
    byts = S * B * 12 + 2 * n2 * row_bytes + n2 * 12 + 4 * (S + 1)
    print(json.dumps({"beam_advance_eos_p": p, "N_next": n2, "us": round(us, 2),
                      "GBps": round(byts / (us * 1e-6) / 1e9, 1),
                      "frac": round(byts / (us * 1e-6) / 1e9 / peak, 3)}))
