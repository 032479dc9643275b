"""Decode-chain timing (NEXT f1): T steps of [output layer -> beam advance]
on the cfg beam shape (H=1024, V=90k, S sentences, beam 5), EOS = token 0
(the most likely token under the zipf prior, so beams shrink).
  eager_host_n : amun_output_layer with N read back to the host every step
                 (one sync per step), then amun_beam_advance;
  graph_dev_n  : amun_output_layer_dev + amun_beam_advance, N' never leaves
                 the device, all T steps captured in ONE CUDA graph.
  python tools/chain_bench.py [S] [T]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses  # noqa: E402
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = dataclasses.replace(synth.CONFIGS["beam"], S=S)
H, V, B, k = w.H, w.V, w.B, w.k
M = S * k
dev = torch.device("cuda", 0)
W, b = synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
ol = amun.OutputLayer(H, V, k_max=k, max_rows=M, max_sentences=S)
X0 = torch.zeros(M, H, dtype=torch.bfloat16, device=dev)
X0[:S * B] = synth.gen_X(w).to(dev)
pc0 = torch.zeros(M, device=dev)
pc0[:S * B] = synth.gen_prev_cost(w).to(dev)
off0 = synth.gen_offsets(w).to(dev)
EOS = 0
st = {"X": [X0.clone(), torch.zeros_like(X0)], "pc": [pc0.clone(), torch.zeros_like(pc0)],
      "off": [off0.clone(), torch.zeros_like(off0)],
      "n": [torch.zeros(2, dtype=torch.int32, device=dev) for _ in range(2)],
      "src": torch.zeros(M, dtype=torch.int32, device=dev), "tok": torch.zeros(M, dtype=torch.int32, device=dev),
      "ws": torch.zeros(max(amun._L.amun_beam_advance_workspace_bytes(S, k), 256), dtype=torch.uint8, device=dev),
      "idx": torch.zeros((S, k), dtype=torch.int64, device=dev),
      "cost": torch.zeros((S, k), dtype=torch.float32, device=dev)}


def reset():
    st["X"][0].copy_(X0); st["pc"][0].copy_(pc0); st["off"][0].copy_(off0)
    st["n"][0][0] = S * B


def adv(a, c):
    amun.beam_advance(st["idx"], st["cost"], V, EOS, M, [(st["X"][a], st["X"][c])], sync=False,
                      out={"new_offsets": st["off"][c], "src_row": st["src"], "new_token": st["tok"],
                           "new_cost": st["pc"][c], "counts": st["n"][c], "workspace": st["ws"]})


def eager():
    rows = []
    for t in range(T):
        a, c = t % 2, (t + 1) % 2
        n = int(st["n"][a][0].item())                      # host sync
        rows.append(n)
        ol(st["X"][a][:n].contiguous(), W, b, st["pc"][a][:n].contiguous(), st["off"][a], k,
           out_idx=st["idx"], out_cost=st["cost"])
        adv(a, c)
    return rows


def dev_steps():
    for t in range(T):
        a, c = t % 2, (t + 1) % 2
        ol.call_dev(st["X"][a], W, b, st["pc"][a], st["off"][a], st["n"][a][:1], k,
                    out_idx=st["idx"], out_cost=st["cost"])
        adv(a, c)


def timed(fn):
    reset()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e), out


timed(eager)
t_eager, rows = timed(eager)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    reset()
    dev_steps()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        dev_steps()
timed(g.replay)
t_graph, _ = timed(g.replay)
print(json.dumps({"S": S, "beam": B, "T": T, "rows_per_step": rows, "useful_rows": sum(rows),
                  "eager_host_n_ms": round(t_eager, 3), "graph_dev_n_ms": round(t_graph, 3),
                  "speedup": round(t_eager / t_graph, 3)}))
