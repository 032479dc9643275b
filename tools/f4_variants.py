"""MXFP4 vs E4M3 fused-kernel device times by variant (0 full, 2 bare GEMM,
3 no k-best; mxfp4 also 5/6/7: bare GEMM whose MMAs re-read the first
stages, with only X / only W copied again) at the greedy and beam shapes: a CUDA graph of K launches, W
rotated over enough copies to defeat L2 (as bench.py).

  python tools/f4_variants.py        (JSON lines)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

dev = torch.device("cuda", 0)
K = int(os.environ.get("F4_K", "50"))


def graph_us(fn):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(K):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            g.replay()
            e.record(st)
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / K * 1e3)
    return best


def main():
    for name in os.environ.get("F4_CFG", "greedy,beam").split(","):
        w = synth.CONFIGS[name]
        X = synth.gen_X(w).to(dev)
        W = synth.gen_W(w).to(dev)
        b = synth.gen_b(w).to(dev)
        X8, xs = amun.quantize_e4m3(X)
        q4 = amun.quantize_mxfp4(W)
        q8 = amun.quantize_e4m3(W)
        n = max(2, -(-2 * 126 * 2 ** 20 // (q4[0].numel())))
        c4 = [q4] + [(q4[0].clone(), q4[1].clone()) for _ in range(n - 1)]
        n8 = max(2, -(-2 * 126 * 2 ** 20 // (q8[0].numel())))
        c8 = [q8] + [(q8[0].clone(), q8[1].clone()) for _ in range(n8 - 1)]
        o4 = amun.OutputLayer(w.H, w.V, dtype="mxfp4", k_max=w.k, max_rows=w.N, max_sentences=w.S)
        o8 = amun.OutputLayer(w.H, w.V, dtype="e4m3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
        for v in (0, 2, 3, 5, 6, 7):
            t4 = graph_us(lambda i: o4.scores_mxfp4(X8, xs, c4[i % n][0], c4[i % n][1], b, variant=v))
            t8 = (graph_us(lambda i: o8.scores_e4m3(X8, xs, c8[i % n8][0], c8[i % n8][1], b,
                                                    variant=v)) if v < 5 else None)
            print(json.dumps({"cfg": name, "variant": v, "mxfp4_us": round(t4, 2),
                              "e4m3_us": t8 and round(t8, 2)}), flush=True)
        del c4, c8, q4, q8, W
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
