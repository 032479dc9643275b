"""Per-CTA timeline of the fused kernel (amun_debug_timeline): %globaltimer
stamps at the kernel's phase boundaries, for the last of K graph-replayed
calls (W rotated so L2 does not serve it). Prints, per probe point, the
median / max over CTAs of (stamp - earliest entry) in microseconds, and the
launch-to-launch gap.

  python tools/timeline.py [workload] [tail|sep|scores|bare|stats] [taper] [prepass]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402
from paper_1805_09863_b200 import _L, check  # noqa: E402

NAMES = ["entry", "setup", "tma0", "full0", "mma_end", "epi_last", "epi_end", "barrier",
         "released", "tail_end"] + [f"tile{i}" for i in range(14)] + [f"mma{i}" for i in range(14)]
TL_N = 40


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "greedy"
    variant = sys.argv[2] if len(sys.argv) > 2 else "tail"
    os.environ["AMUN_TAIL"] = "off" if variant in ("sep", "scores", "bare", "stats", "mmaonly") else "on"
    if len(sys.argv) > 3:   # taper on / off (1 / 0)
        os.environ["AMUN_TAPER"] = sys.argv[3]
    if len(sys.argv) > 4:   # first-tile pre-pass on / off (1 / 0)
        os.environ["AMUN_PREPASS"] = sys.argv[4]
    w = synth.CONFIGS[name]
    if os.environ.get("AMUN_TL_V"):   # (experiment: another vocabulary size)
        import dataclasses
        w = dataclasses.replace(w, V=int(os.environ["AMUN_TL_V"]))
    dev = torch.device("cuda", 0)
    X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
    pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
    nc = max(2, -(-2 * 126 * 2 ** 20 // (W.numel() * W.element_size())))
    if os.environ.get("AMUN_TL_COPIES"):   # (experiment: 1 = W may stay in L2)
        nc = int(os.environ["AMUN_TL_COPIES"])
    Ws = [W] + [W.clone() for _ in range(nc - 1)]
    ol = amun.OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    tl = torch.zeros((nsm, TL_N), dtype=torch.int64, device=dev)
    check(_L.amun_debug_timeline(ol._h, tl.data_ptr()))
    oi = torch.empty((w.S, w.k), dtype=torch.int64, device=dev)
    oc = torch.empty((w.S, w.k), dtype=torch.float32, device=dev)

    def step(i):
        if variant == "scores":
            ol.scores(X, Ws[i % nc], b)
        elif variant in ("bare", "stats", "mmaonly"):   # amun_bench_variant 2 / 3 / 5
            ol.bench_variant(X, Ws[i % nc], b, {"bare": 2, "stats": 3, "mmaonly": 5}[variant])
        else:
            ol(X, Ws[i % nc], b, pc, off, w.k, out_idx=oi, out_cost=oc)
    K = 20
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        step(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(K):
                step(i)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        tl.zero_()
        g.replay()
        torch.cuda.synchronize()
    t = tl.cpu().numpy().astype(np.float64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    out = {"workload": name, "variant": variant, "ctas": int(used.sum()), "V": w.V, "copies": nc,
           "env": {k: os.environ.get(k) for k in ("AMUN_TAPER", "AMUN_PREPASS")}}
    for j, n in enumerate(NAMES):
        col = t[:, j]
        col = col[col > 0]
        if len(col) == 0:
            continue
        rel = (col - t0) / 1e3
        out[n] = {"med": round(float(np.median(rel)), 2), "max": round(float(rel.max()), 2),
                  "min": round(float(rel.min()), 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
