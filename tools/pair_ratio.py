"""Per-FLOP speed of the CTA-pair kernel vs the single-CTA kernel at the cfg
beam shape (H=1024, V=90000) for N rows: the fused kernel (scores) and the
bare GEMM (bench variant 2), CUDA-graph timed. Run once with AMUN_PAIRS=off
and once with AMUN_PAIRS=force (the plan reads the variable at creation).

  AMUN_PAIRS=force python tools/pair_ratio.py 512 640 1024
"""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402
from tools.sweep_n import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    base = synth.CONFIGS["beam"]
    W, b = synth.gen_W(base).to(dev), synth.gen_b(base).to(dev)
    for N in [int(a) for a in sys.argv[1:]] or [512, 640]:
        w = dataclasses.replace(base, S=N // base.B)
        X = synth.gen_X(w).to(dev)[:N].contiguous()
        ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=N, max_sentences=w.S)
        t_f = graph_time(lambda: ol.scores(X, W, b))
        t_g = graph_time(lambda: ol.bench_variant(X, W, b, 2))
        print(json.dumps({"pairs": os.environ.get("AMUN_PAIRS", "auto"), "N": N,
                          "fused_us": round(t_f, 2), "bare_us": round(t_g, 2),
                          "bare_tflops": round(2 * N * w.H * w.V / t_g / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
