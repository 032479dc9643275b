"""A few MXFP4 output-layer calls on a config shape, for ncu captures of
the ELT=3 fused kernel (ol_tc_kernel<KB, 0, 2, 3>).

  python tools/f4_one.py [greedy|beam]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402


def main():
    w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "greedy"]
    dev = torch.device("cuda", 0)
    X = synth.gen_X(w).to(dev)
    W4, sf = amun.quantize_mxfp4(synth.gen_W(w).to(dev))
    b, pc, off = synth.gen_b(w).to(dev), synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w, dev)
    ol = amun.OutputLayer(w.H, w.V, dtype="mxfp4", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    for _ in range(5):
        X8, xs = amun.quantize_e4m3(X)
        ol.call_mxfp4(X8, xs, W4, sf, b, pc, off, w.k)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
