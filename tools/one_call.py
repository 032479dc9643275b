"""Run the fused output layer a few times eagerly (for ncu captures).
  python tools/one_call.py [config] [calls]   (env AMUN_SENTENCES, AMUN_PAIRS)"""
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
ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
for _ in range(calls):
    ol(X, W, b, pc, off, w.k)
torch.cuda.synchronize()
print("ok", name, w.N)
