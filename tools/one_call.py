"""Run the fused output layer a few times eagerly (for ncu captures).
  python tools/one_call.py [config] [calls] [bf16|e4m3|bare|stats]
  (env AMUN_SENTENCES, AMUN_PAIRS; bare / stats: amun_bench_variant 2 / 3)"""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "beam"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = synth.CONFIGS[name]
if os.environ.get("AMUN_SENTENCES"):
    w = dataclasses.replace(w, S=int(os.environ["AMUN_SENTENCES"]))
dev = torch.device("cuda", 0)
X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w, device=dev), synth.gen_b(w).to(dev)
pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
if prec == "e4m3":
    X8, xs = amun.quantize_e4m3(X)
    W8, ws = amun.quantize_e4m3(W)
    ol = amun.OutputLayer(w.H, w.V, dtype="e4m3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    for _ in range(calls):
        ol.call_e4m3(X8, xs, W8, ws, b, pc, off, w.k)
elif prec in ("bare", "stats"):
    ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    for _ in range(calls):
        ol.bench_variant(X, W, b, 2 if prec == "bare" else 3)
else:
    ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    for _ in range(calls):
        ol(X, W, b, pc, off, w.k)
torch.cuda.synchronize()
print("ok", name, w.N)
