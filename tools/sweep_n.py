"""Speed vs batch size (the Fig. 3 analogue, PAPER.md
P:340 "batches above 1000"): the full output-layer path (fused kernel + merge,
one CUDA graph) on the cfg beam shape (H=1024, V=90000, beam 5) for S
sentences, next to an UNFUSED B200 comparator in the style of the paper's
Table 4 baseline: cuBLAS GEMM with the logits in HBM, then torch
bias add, log_softmax and a per-sentence top-k over B*V costs.

  python tools/sweep_n.py [S ...]   -> one JSON line per S (rows/s, frac)
"""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def graph_time(fn, reps=5, iters=20):
    """Device time per call: `reps` calls captured in one CUDA graph, replayed."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (iters * reps) * 1e3


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1, 4, 16, 32, 64, 128, 256, 512, 1024, 2048]
    peaks = {"hbm_gbs": 6454.3, "bf16_tflops": 1642.7}
    pk = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks.update({k: v for k, v in json.load(open(pk)).items() if k in peaks})
    base = synth.CONFIGS["beam"]
    dev = torch.device("cuda", 0)
    W = synth.gen_W(base).to(dev)
    b = synth.gen_b(base).to(dev)
    Wt = W.t()
    for S in sizes:
        w = dataclasses.replace(base, S=S)
        N, H, V, B, k = w.N, w.H, w.V, w.B, w.k
        X = synth.gen_X(w).to(dev)
        pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
        ol = amun.OutputLayer(H, V, dtype=w.dtype, k_max=k, max_rows=N, max_sentences=S)
        oi = torch.empty((S, k), dtype=torch.int64, device=dev)
        oc = torch.empty((S, k), dtype=torch.float32, device=dev)
        t_ours = graph_time(lambda: ol(X, W, b, pc, off, k, out_idx=oi, out_cost=oc))

        def unfused():
            logits = torch.mm(X, Wt).float() + b                 # GEMM, logits in HBM, + bias
            logp = torch.log_softmax(logits, dim=1)              # softmax (3 passes)
            cost = (pc[:, None] + logp).view(S, B * V)           # beam cost
            return torch.topk(cost, k, dim=1)                    # k-best per sentence
        t_unf = graph_time(unfused)
        flops = 2.0 * N * H * V
        alg_bytes = V * H * 2 + N * H * 2 + V * 4 + N * 4 + (S + 1) * 4 + S * k * 12
        t_roof = max(flops / (peaks["bf16_tflops"] * 1e12), alg_bytes / (peaks["hbm_gbs"] * 1e9)) * 1e6
        print(json.dumps({
            "S": S, "B": B, "N": N, "H": H, "V": V, "k": k,
            "bound": "tensor" if flops / (peaks["bf16_tflops"] * 1e12) > alg_bytes / (peaks["hbm_gbs"] * 1e9)
            else "hbm",
            "t_roof_us": round(t_roof, 2),
            "ours_us": round(t_ours, 2), "ours_rows_per_s": round(N / (t_ours * 1e-6)),
            "ours_frac": round(t_roof / t_ours, 3),
            "unfused_us": round(t_unf, 2), "unfused_rows_per_s": round(N / (t_unf * 1e-6)),
            "speedup_vs_unfused": round(t_unf / t_ours, 2)}), flush=True)
        del ol


if __name__ == "__main__":
    main()
