"""One-call driver for ncu launch lists of the one-shot path (NEXT f3):
three amun_output_layer calls and three amun_output_layer_oneshot calls
(world 1, IPC buffer) on a BASELINE config (default greedy).

  ncu --metrics gpu__time_duration.sum --csv --log-file L.csv python tools/os_one.py greedy
  python tools/os_ncu_parse.py L.csv
"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_09863_b200.sharded import ShardedOutputLayer
dev = torch.device("cuda", 0)
w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "greedy"]
X, pc, off = synth.gen_X(w).to(dev), synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
W, b = synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
sh = ShardedOutputLayer(w.H, w.V, 1, 0, k_max=w.k, max_rows=w.N, max_sentences=w.S, exchange="oneshot")
for _ in range(3):
    sh.ol(X, W, b, pc, off, w.k)
    sh(X, W, b, pc, off, w.k)
torch.cuda.synchronize()
print("ok")
