"""Throughput vs clocks/power for a GEMM variant run back to back ~1.5 s
(CUDA-graph replays) while nvidia-smi samples clocks.sm, power.draw and the
throttle reasons. Shows whether a kernel is power-capped (sw_power_cap) and
at what SM clock it actually ran.
  python tools/power_probe.py [config] [variant: fused|gemm|stats|cublas]"""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "beam"
    var = sys.argv[2] if len(sys.argv) > 2 else "gemm"
    w = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    X = synth.gen_X(w).to(dev)
    W = synth.gen_W(w, device=dev)
    b = synth.gen_b(w).to(dev)
    ol = amun.OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    Wt = W.t()
    fn = {"fused": lambda: ol.scores(X, W, b), "gemm": lambda: ol.bench_variant(X, W, b, 2),
          "stats": lambda: ol.bench_variant(X, W, b, 3), "cublas": lambda: torch.mm(X, Wt)}[var]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    per = s.elapsed_time(e) / 10
    reps = max(1, int(1500 / (per * 10)))
    lines = []
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    threading.Thread(target=lambda: [lines.append(l.strip()) for l in p.stdout], daemon=True).start()
    time.sleep(0.3)
    n0 = len(lines)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    n1 = len(lines)
    p.terminate()
    ms = s.elapsed_time(e) / (reps * 10)
    samp = [l.split(",") for l in lines[n0:n1] if l.count(",") == 2]
    clk = sorted(float(x[0]) for x in samp) or [0]
    pw = sorted(float(x[1]) for x in samp) or [0]
    reasons = sorted({x[2].strip() for x in samp})
    flops = 2.0 * w.N * w.H * w.V
    print(f"{name} {var} pairs={os.environ.get('AMUN_PAIRS', 'auto')}: "
          f"{ms * 1e3:.1f} us/call, {flops / ms / 1e9:.0f} TF/s, sm clock median "
          f"{clk[len(clk) // 2]:.0f} MHz (min {clk[0]:.0f}), power median {pw[len(pw) // 2]:.0f} W, "
          f"reasons {reasons}, samples {len(samp)}")


if __name__ == "__main__":
    main()
