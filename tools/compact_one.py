"""One amun_compact call (for ncu captures): N rows of the cfg4 state, the
given survival probability p (0 = none alive), S = N / 5.
  python tools/compact_one.py [N] [p] [calls]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 6400
p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
S = N // 5
cols = [torch.randn(N, 1024, device=dev).to(torch.bfloat16), torch.randn(N, 2048, device=dev),
        torch.randn(N, device=dev), torch.arange(N, dtype=torch.int64, device=dev)]
dst = [torch.empty_like(c) for c in cols]
off = torch.arange(S + 1, dtype=torch.int32, device=dev) * 5
alive = (synth.gen_alive(10, N, p) if p > 0 else torch.zeros(N, dtype=torch.uint8)).to(dev)
for _ in range(calls):
    out = amun.compact(list(zip(cols, dst)), alive, off, sync=False)
torch.cuda.synchronize()
print("ok", N, p)
if os.environ.get("AMUN_CP_EXP") in ("9", "10", "11", "12"):
    print("CTA0 phase ns:", out[3][:8].tolist())
