"""Prototype (experiment): cfg beam as CTA PAIRS for the first 4 M-tiles
(rows 0-511, cta_group::2) on P SMs and single CTAs for the fifth (rows
512-639) on S = 148 - P SMs, the two fused kernels concurrently on two streams
(each emits one record per row, amun_output_layer_partial), then one sentence
merge over the [1][N][stride] records. Device time per step from CUDA graphs.
  python tools/hybrid_bench.py [P ...]"""
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
    dev = torch.device("cuda", 0)
    w = synth.CONFIGS["beam"]
    X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
    pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
    Ws = [W, W.clone()]
    ref = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    ri, rc = ref(X, W, b, pc, off, w.k)
    for P in [int(a) for a in sys.argv[1:]] or [118, 124, 126, 128]:
        S = 148 - P
        os.environ["AMUN_PAIRS"] = "force"
        os.environ["AMUN_SMS"] = str(P)
        olp = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=512, max_sentences=w.S)
        os.environ["AMUN_PAIRS"] = "off"
        os.environ["AMUN_SMS"] = str(S)
        ols = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=128, max_sentences=w.S)
        os.environ.pop("AMUN_SMS")
        os.environ.pop("AMUN_PAIRS")
        part = torch.empty((1, w.N, olp.stride), dtype=torch.float32, device=dev)
        oi = torch.empty((w.S, w.k), dtype=torch.int64, device=dev)
        oc = torch.empty((w.S, w.k), dtype=torch.float32, device=dev)
        side = torch.cuda.Stream(dev)
        e0, e1 = torch.cuda.Event(), torch.cuda.Event()

        def step(i):
            main = torch.cuda.current_stream(dev)
            e0.record(main)
            side.wait_event(e0)
            with torch.cuda.stream(side):
                ols.partial(X[512:], Ws[i % 2], b, out=part[0, 512:])
                e1.record(side)
            olp.partial(X[:512], Ws[i % 2], b, out=part[0, :512])
            main.wait_event(e1)
            ref.merge(part, pc, off, w.k, out_idx=oi, out_cost=oc)
        step(0)
        torch.cuda.synchronize()
        same = bool(torch.equal(oi, ri))
        time.sleep(1)
        us = graph_us(step, 30, reps=3)
        time.sleep(1)
        us_p = graph_us(lambda i: olp.partial(X[:512], Ws[i % 2], b, out=part[0, :512]), 30, reps=3)
        time.sleep(1)
        us_s = graph_us(lambda i: ols.partial(X[512:], Ws[i % 2], b, out=part[0, 512:]), 30, reps=3)
        print(json.dumps({"P": P, "S": S, "step_us": min(us), "pairs_alone_us": min(us_p),
                          "singles_alone_us": min(us_s), "same_idx_as_single_plan": same}), flush=True)
    time.sleep(1)
    us_ref = graph_us(lambda i: ref(X, Ws[i % 2], b, pc, off, w.k, out_idx=oi, out_cost=oc), 30, reps=3)
    print(json.dumps({"reference_amun_output_layer_us": min(us_ref)}))


if __name__ == "__main__":
    main()
