"""fp32 output layer: the 3xTF32 tensor-core plan
(dtype="tf32x3") vs the SIMT fp32 plan (dtype="f32") vs an
unfused fp32 comparator (cuBLAS fp32 GEMM with TF32 disabled + bias +
log_softmax + per-sentence top-k), on the cfg beam shape with fp32 inputs.
Per step the tf32x3 time includes splitting X (amun_split_tf32x3); W is split
once (a weight, like the e4m3 quantization). Device time per call from CUDA
graph replays.

  python tools/tf32_bench.py [S ...]   -> one JSON line per S
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
    sizes = [int(a) for a in sys.argv[1:]] or [1, 16, 128, 256]
    torch.backends.cuda.matmul.allow_tf32 = False
    base = dataclasses.replace(synth.CONFIGS["beam"], dtype="f32")
    dev = torch.device("cuda", 0)
    W = synth.gen_W(base).to(dev)
    b = synth.gen_b(base).to(dev)
    Ws = amun.split_tf32x3(W, "W")
    for S in sizes:
        w = dataclasses.replace(base, S=S)
        N, H, V, k = w.N, w.H, w.V, w.k
        X = synth.gen_X(w).to(dev)
        pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
        Xs = torch.empty((N, 3 * H), dtype=torch.float32, device=dev)
        oi = torch.empty((S, k), dtype=torch.int64, device=dev)
        oc = torch.empty((S, k), dtype=torch.float32, device=dev)
        t3 = amun.OutputLayer(H, V, dtype="tf32x3", k_max=k, max_rows=N, max_sentences=S)
        f32 = amun.OutputLayer(H, V, dtype="f32", k_max=k, max_rows=N, max_sentences=S)

        def run_t3():
            amun.split_tf32x3(X, "X", out=Xs)
            t3(Xs, Ws, b, pc, off, k, out_idx=oi, out_cost=oc)
        t_t3 = graph_time(run_t3)
        t_t3_ol = graph_time(lambda: t3(Xs, Ws, b, pc, off, k, out_idx=oi, out_cost=oc))
        t_f32 = graph_time(lambda: f32(X, W, b, pc, off, k, out_idx=oi, out_cost=oc))

        def unfused():
            logits = torch.mm(X, W.t()) + b
            cost = (pc[:, None] + torch.log_softmax(logits, dim=1)).view(S, -1)
            return torch.topk(cost, k, dim=1)
        t_unf = graph_time(unfused)
        print(json.dumps({"S": S, "N": N, "H": H, "V": V, "k": k,
                          "tf32x3_us": round(t_t3, 2), "tf32x3_ol_only_us": round(t_t3_ol, 2),
                          "simt_f32_us": round(t_f32, 2), "unfused_fp32_us": round(t_unf, 2),
                          "tf32x3_rows_per_s": round(N / (t_t3 * 1e-6)),
                          "speedup_vs_simt": round(t_f32 / t_t3, 2),
                          "speedup_vs_unfused": round(t_unf / t_t3, 2)}), flush=True)
        del t3, f32


if __name__ == "__main__":
    main()
