"""Compaction fixed cost and scan scaling.

Per call device time (CUDA graph of 50 calls) of amun_compact with NO row
surviving (the fixed cost: flag scan, new offsets, sentence count, launch)
and with p = 0.1 survival, at N in {6400 (cfg4), 16384, 65536} rows of the
cfg4 state (10,252 B/row; small N' so the gather does not hide the scan),
S = N / 5. AMUN_CP_EXP (read once per process) compiles nothing out but skips
parts at run time: 1 no sentence count, 2 + no new offsets, 3 scan only.
A one-element torch kernel in the same graph form gives the launch floor.

  AMUN_CP_EXP=e python tools/compact_fixed.py     (JSON lines)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

dev = torch.device("cuda", 0)


def graph_us(fn, reps=50):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            g.replay()
            e.record(st)
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / reps * 1e3)
    return best


def main():
    exp = int(os.environ.get("AMUN_CP_EXP", "0"))
    one = torch.zeros(1, device=dev)
    floor = graph_us(lambda: one.add_(1.0))
    for N in (6400, 16384, 65536):
        B = 5
        S = N // B
        cols = [torch.randn(N, 1024, device=dev).to(torch.bfloat16), torch.randn(N, 2048, device=dev),
                torch.randn(N, device=dev), torch.arange(N, dtype=torch.int64, device=dev)]
        dst = [torch.empty_like(c) for c in cols]
        off = torch.arange(S + 1, dtype=torch.int32, device=dev) * B
        new_off = torch.empty_like(off)
        src_row = torch.empty(N, dtype=torch.int32, device=dev)
        counts = torch.empty(2, dtype=torch.int32, device=dev)
        for name, alive in (("none", torch.zeros(N, dtype=torch.uint8, device=dev)),
                            ("p=0.1", synth.gen_alive(10, N, 0.1).to(dev))):
            us = graph_us(lambda: amun.compact(list(zip(cols, dst)), alive, off, new_off, src_row,
                                               counts, sync=False))
            print(json.dumps({"exp": exp, "N": N, "S": S, "mask": name,
                              "N_alive": int(alive.sum().item()), "us": round(us, 2),
                              "launch_floor_us": round(floor, 2)}), flush=True)
        del cols, dst


if __name__ == "__main__":
    main()
