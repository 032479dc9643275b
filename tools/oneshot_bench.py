"""NVLink one-shot exchange on ONE GPU: G vocab-shard
ranks emulated (amun_output_layer_oneshot_emulated: the G fused kernels in
sequence + one cooperative one-shot kernel with a grid row per rank) against
the same G shards through the collective path emulated on one GPU (G x
amun_output_layer_partial, a torch.stack standing in for the all-gather,
amun_merge_partials). "post" = the total minus the G fused kernels alone, i.e.
everything after the GEMMs: for the one-shot path ONE kernel doing all G
ranks' row phase, exchange and merge at once (an upper bound on one rank's
tail on real GPUs, where each rank does 1/G of the row phase). Also the
real-mode entry point at G = 1 (IPC-exported buffer, self-signal) against
amun_output_layer. Device time per call from CUDA graph replays. No NVLink
is exercised: these are not multi-GPU numbers.

  python tools/oneshot_bench.py   -> one JSON line per (config, G)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402
from paper_1805_09863_b200.sharded import EmulatedOneShot, ShardedOutputLayer, shard_range  # noqa: E402
from tools.sweep_n import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    todo = [("greedy", [2, 8]), ("beam", [2, 8]), ("shard", [8])]
    if len(sys.argv) > 1:
        todo = [t for t in todo if t[0] in sys.argv[1:]]
    for name, Gs in todo:
        w = synth.CONFIGS[name]
        X, pc, off = synth.gen_X(w).to(dev), synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
        for G in Gs:
            layers, Ws, bs = [], [], []
            for g in range(G):
                v0, v1 = shard_range(w.V, G, g)
                layers.append(amun.OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, k_max=w.k,
                                               max_rows=w.N, max_sentences=w.S))
                Ws.append(synth.gen_W(w, v0, v1 - v0).to(dev))
                bs.append(synth.gen_b(w, v0, v1 - v0).to(dev))
            P = torch.empty((G, w.N, layers[0].stride), dtype=torch.float32, device=dev)

            def collective():
                for g in range(G):
                    layers[g].partial(X, Ws[g], bs[g], out=P[g])
                layers[0].merge(P, pc, off, w.k)

            em = EmulatedOneShot(layers)
            outs = [layers[0]._outputs(w.S, w.k, None, None) for _ in range(G)]
            t_fused = graph_time(lambda: [layers[g].scores(X, Ws[g], bs[g]) for g in range(G)])
            t_coll = graph_time(collective)
            t_os = graph_time(lambda: em(X, Ws, bs, pc, off, w.k, outs=outs))
            em.close()
            print(json.dumps({"config": name, "G": G, "N": w.N, "S": w.S, "V": w.V, "k": w.k,
                              "fused_x_G_us": round(t_fused, 2),
                              "collective_emulated_us": round(t_coll, 2),
                              "oneshot_emulated_us": round(t_os, 2),
                              "collective_post_us": round(t_coll - t_fused, 2),
                              "oneshot_post_us": round(t_os - t_fused, 2)}), flush=True)
            del layers, Ws, bs
        # real mode, G = 1
        sh = ShardedOutputLayer(w.H, w.V, 1, 0, k_max=w.k, max_rows=w.N, max_sentences=w.S,
                                exchange="oneshot")
        W, b = synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
        oi = torch.empty((w.S, w.k), dtype=torch.int64, device=dev)
        oc = torch.empty((w.S, w.k), dtype=torch.float32, device=dev)
        t_plain = graph_time(lambda: sh.ol(X, W, b, pc, off, w.k, out_idx=oi, out_cost=oc))
        t_real = graph_time(lambda: sh(X, W, b, pc, off, w.k, out_idx=oi, out_cost=oc))
        sh.oneshot.close()
        print(json.dumps({"config": name, "G": 1, "mode": "real (IPC buffer, rank 0 of 1)",
                          "output_layer_us": round(t_plain, 2), "oneshot_us": round(t_real, 2)}),
              flush=True)
        del sh, W, b


if __name__ == "__main__":
    main()
