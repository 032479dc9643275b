"""Device time per launch of the fused kernel's benchmark variants
(amun_bench_variant: 2 bare GEMM, 3 + softmax stats, 5 bare GEMM whose MMAs
re-read the first stages: the MMA issue rate without TMA traffic) and the
full kernel (amun_ol_scores), CUDA graphs of 30 launches, W rotated so L2
does not serve it, 1 s cool-down between measurements (burst clocks).
  python tools/variant_times.py [workload]   (JSON lines)"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402
from tools.ab_path import graph_us  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "beam"
    w = synth.CONFIGS[name]
    if os.environ.get("VT_S"):   # another batch: S sentences (x beam B)
        import dataclasses
        w = dataclasses.replace(w, S=int(os.environ["VT_S"]), B=int(os.environ.get("VT_B", w.B)))
    dev = torch.device("cuda", 0)
    X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
    if os.environ.get("VT_XOFF"):   # X placed at a byte offset inside a larger buffer
        off = int(os.environ["VT_XOFF"]) // X.element_size()
        buf = torch.empty(X.numel() + off + 4096, dtype=X.dtype, device=dev)
        Xo = buf[off:off + X.numel()].view(X.shape)
        Xo.copy_(X)
        X = Xo
    nc = max(2, -(-2 * 126 * 2 ** 20 // (W.numel() * W.element_size())))
    Ws = [W] + [W.clone() for _ in range(nc - 1)]
    ol = amun.OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    K = 30
    for rnd in range(2):
        for v in [int(x) if x.isdigit() else x
                  for x in os.environ.get("VT_VARIANTS", "full,2,3,5,6,7").split(",")]:
            def fn(i, v=v):
                if v == "full":
                    ol.scores(X, Ws[i % nc], b)
                else:
                    ol.bench_variant(X, Ws[i % nc], b, v)
            time.sleep(1.0)
            us = graph_us(fn, K, reps=3)
            flops = 2.0 * w.N * w.H * w.V
            print(json.dumps({"workload": name, "N": w.N, "xoff": os.environ.get("VT_XOFF"),
                              "xptr_mod_2m": X.data_ptr() % (1 << 21),
                              "round": rnd, "variant": v, "us_min": min(us),
                              "tflops": flops / (min(us) * 1e-6) / 1e12}), flush=True)


if __name__ == "__main__":
    main()
