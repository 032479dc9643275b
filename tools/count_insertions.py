"""Instrumentation (AMUN_EXP=4 build, passed as AMUN_LIB): per-config counts of
row-chunks, candidate row-chunks, top-k insertions (total / into a filling
list) and warp-chunks with a candidate, for one fused call.
  AMUN_LIB=variants/e4.so python tools/count_insertions.py [config]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402
from paper_1805_09863_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "beam"
w = synth.CONFIGS[name]
dev = torch.device("cuda", 0)
X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
ol = amun.OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=w.N, max_sentences=w.S)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
ol.scores(X, W, b)
torch.cuda.synchronize()
lib.amun_debug_counters(buf, 1)
ol.scores(X, W, b)
torch.cuda.synchronize()
lib.amun_debug_counters(buf, 1)
c = list(buf)
print(f"{name}: rows {w.N}  row-chunks {c[0]}  cand row-chunks {c[1]} ({c[1]/max(c[0],1):.3f})  "
      f"insertions {c[2]} ({c[2]/w.N:.0f}/row, filling {c[3]})  warp-chunks w/ cand {c[4]}")
