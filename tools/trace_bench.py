"""Config 4 (BASELINE.json 'mini-batching decode trace'): 1280 sentences x beam 5,
V = 90k, H = 1024 (assumed), seeded ragged EOS schedule; dynamic mini-batching
(Alg. 2, compaction) vs naive constant batch (Alg. 1). Prints one JSON line.
  python tools/trace_bench.py [--sentences S] [--out file]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1805_09863_b200.trace import DecodeTrace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sentences", type=int, default=1280)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    w = synth.CONFIGS["trace"]
    S, B = a.sentences, w.B
    dev = torch.device("cuda", 0)
    wl = synth.Workload("trace", H=w.H, V=w.V, S=S, B=B, k=B, seed=w.seed)
    X, W, b, pc = synth.gen_X(wl), synth.gen_W(wl, device=dev), synth.gen_b(wl).to(dev), synth.gen_prev_cost(wl)
    f = synth.eos_schedule(w.seed, S, B)
    tr = DecodeTrace(w.H, w.V, S, B, device=dev)
    tr.run(X, W, b, pc, f, mode="dynamic")        # warm-up
    dyn = tr.run(X, W, b, pc, f, mode="dynamic")
    nai = tr.run(X, W, b, pc, f, mode="naive")
    gr = tr.run_graph(X, W, b, pc, f)
    assert gr.rows[:len(dyn.rows)] == dyn.rows, "graph mode must decode the same rows per step"
    useful = int(f.sum())
    out = {"workload": f"trace: H={w.H}, V={w.V}, {S} sentences x beam {B}, geometric lengths "
                       f"(p=1/20, cap 60), hypothesis j finishes at L_s + j",
           "useful_rows": useful, "T_max": int(f.max()),
           "dynamic": dyn.summary(useful), "naive": nai.summary(useful),
           "dynamic_graph": {"total_ms": gr.total_ms, "steps": gr.steps,
                             "useful_rows_per_s": useful / (gr.total_ms * 1e-3),
                             "note": "Alg. 2 with N on the device (amun_output_layer_dev + "
                                     "amun_compact), all steps in one CUDA graph"},
           "speedup_dynamic_vs_naive": nai.total_ms / dyn.total_ms,
           "speedup_dynamic_graph_vs_naive": nai.total_ms / gr.total_ms}
    line = json.dumps(out)
    print(json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items()
                                                            if kk not in ("step_ms", "rows_per_step")})
                      for k, v in out.items()}))
    if a.out:
        open(a.out, "w").write(line + "\n")


if __name__ == "__main__":
    main()
