"""Per-stage device times of the output-layer path (CUDA events, warm L2):
fused kernel alone, select (merge) alone, both, and an empty-launch floor.
  python tools/stage_times.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402


def timeit(fn, iters=200, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def graph_time(fn, reps=20, iters=20):
    """Pure device time per call: `reps` calls captured in one CUDA graph."""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "beam"
    w = synth.CONFIGS[name]
    if os.environ.get("AMUN_SENTENCES"):   # same config with another batch size
        import dataclasses
        w = dataclasses.replace(w, S=int(os.environ["AMUN_SENTENCES"]))
        name = f"{name}(S={w.S})"
    dev = torch.device("cuda", 0)
    X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
    pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
    ol = amun.OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    oi = torch.empty((w.S, w.k), dtype=torch.int64, device=dev)
    oc = torch.empty((w.S, w.k), dtype=torch.float32, device=dev)
    ol.scores(X, W, b)
    t_sel = timeit(lambda: ol.select(w.N, pc, off, w.k, out_idx=oi, out_cost=oc))
    t_sc = timeit(lambda: ol.scores(X, W, b), iters=50)
    t_all = timeit(lambda: ol(X, W, b, pc, off, w.k, out_idx=oi, out_cost=oc), iters=50)
    z = torch.empty(1, device=dev)
    t_empty = timeit(lambda: z.add_(1.0))
    print(f"{name}: scores {t_sc:.1f} us | select {t_sel:.1f} us | both {t_all:.1f} us | "
          f"torch tiny-kernel launch {t_empty:.1f} us  (eager, host-launch bound)")
    g_sel = graph_time(lambda: ol.select(w.N, pc, off, w.k, out_idx=oi, out_cost=oc))
    g_sc = graph_time(lambda: ol.scores(X, W, b), reps=5)
    g_all = graph_time(lambda: ol(X, W, b, pc, off, w.k, out_idx=oi, out_cost=oc), reps=5)
    g_empty = graph_time(lambda: z.add_(1.0))
    g_v2 = graph_time(lambda: ol.bench_variant(X, W, b, 2), reps=5)
    g_v3 = graph_time(lambda: ol.bench_variant(X, W, b, 3), reps=5)
    Wt = W.t()
    g_cublas = graph_time(lambda: torch.mm(X, Wt), reps=5)
    print(f"{name}: GRAPH cuBLAS torch.mm bf16 (logits to HBM, no softmax/k-best) {g_cublas:.1f} us")
    print(f"{name}: GRAPH bare GEMM {g_v2:.1f} us | GEMM+bias+softmax stats {g_v3:.1f} us | "
          f"+k-best (full fused) {g_sc:.1f} us")
    print(f"{name}: GRAPH scores {g_sc:.1f} us | select {g_sel:.1f} us | both {g_all:.1f} us | "
          f"tiny kernel {g_empty:.1f} us")
    if w.dtype == "bf16":
        ot = torch.empty(w.N, dtype=torch.int64, device=dev)
        ob = torch.empty(w.N, dtype=torch.float32, device=dev)
        g_am = graph_time(lambda: ol.argmax(X, W, b, out_token=ot, out_logit=ob), reps=5)
        g_v4 = graph_time(lambda: ol.bench_variant(X, W, b, 4), reps=5)
        print(f"{name}: GRAPH argmax-only path (Alg. 5: fused kernel without exp + row argmax) "
              f"{g_am:.1f} us | its fused kernel alone {g_v4:.1f} us")
        # FP8 (E4M3, NEXT f4): same shapes, X / W quantised per row on the GPU
        X8, xs = amun.quantize_e4m3(X)
        W8, ws = amun.quantize_e4m3(W)
        o8 = amun.OutputLayer(w.H, w.V, dtype="e4m3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
        f8 = {v: graph_time(lambda v=v: o8.scores_e4m3(X8, xs, W8, ws, b, v), reps=5) for v in (2, 3, 0)}
        f8_all = graph_time(lambda: o8.call_e4m3(X8, xs, W8, ws, b, pc, off, w.k, out_idx=oi,
                                                 out_cost=oc), reps=5)
        g_q = graph_time(lambda: amun.quantize_e4m3(X, out=X8, scale=xs), reps=5)
        print(f"{name}: GRAPH e4m3 bare GEMM {f8[2]:.1f} us | + stats {f8[3]:.1f} us | full fused "
              f"{f8[0]:.1f} us | path (fused + select) {f8_all:.1f} us | X quantise {g_q:.1f} us")


if __name__ == "__main__":
    main()
