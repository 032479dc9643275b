"""A/B device times of the whole output-layer path (amun_output_layer) under
plan-creation switches (env read by amun_ol_create): the fused tail
(AMUN_TAIL=off: separate merge kernel), the tail experiments, taper,
pre-pass, PDL and W box size. (The entry L2 prefetch of W that "+pf" once
measured was removed after it measured slower.) CUDA graph of K calls, W rotated over enough copies that
L2 never serves W across calls (as bench.py). Interleaved repetitions.

  python tools/ab_path.py [workload ...]     (JSON lines)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1805_09863_b200 as amun  # noqa: E402

VARIANTS = {
    "tail": {"AMUN_TAIL": "on"},
    "sep": {"AMUN_TAIL": "off"},
    "tailwait": {"AMUN_TAIL": "wait"},     # tail without merge work
    "tailnocoop": {"AMUN_TAIL": "nocoop"},
}
VARIANTS["tailfence"] = {"AMUN_TAIL": "fence"}
VARIANTS["tailsleep"] = {"AMUN_TAIL": "sleep"}
VARIANTS["waitnocoop"] = {"AMUN_TAIL": "waitnocoop"}
VARIANTS["arriveonly"] = {"AMUN_TAIL": "arriveonly"}
VARIANTS["scores"] = {"AMUN_TAIL": "off"}   # the fused kernel alone
# final-tile taper (TileIter) on (default off), the first-tile k-best bound
# pre-pass off (default on)
VARIANTS["tail_t1"] = {"AMUN_TAIL": "on", "AMUN_TAPER": "1"}
VARIANTS["sep_t1"] = {"AMUN_TAIL": "off", "AMUN_TAPER": "1"}
VARIANTS["scores_t1"] = {"AMUN_TAIL": "off", "AMUN_TAPER": "1"}
VARIANTS["tail_pp0"] = {"AMUN_TAIL": "on", "AMUN_PREPASS": "0"}
VARIANTS["sep_pp0"] = {"AMUN_TAIL": "off", "AMUN_PREPASS": "0"}
VARIANTS["scores_pp0"] = {"AMUN_TAIL": "off", "AMUN_PREPASS": "0"}
for _p in (0, 1):
    VARIANTS[f"tail_pdl{_p}"] = {"AMUN_TAIL": "on", "AMUN_PDL": str(_p)}
    VARIANTS[f"sep_pdl{_p}"] = {"AMUN_TAIL": "off", "AMUN_PDL": str(_p)}
    VARIANTS[f"scores_pdl{_p}"] = {"AMUN_TAIL": "off", "AMUN_PDL": str(_p)}
for _m in (0, 2, 4, 5, 6):   # W multicast clusters of the M-tiles of a split (experiment)
    VARIANTS[f"tail_mc{_m}"] = {"AMUN_TAIL": "on", "AMUN_MC": str(_m)}
for _n in (0, 1):   # narrow remainder tiles load 64-row W boxes
    VARIANTS[f"tail_wn{_n}"] = {"AMUN_TAIL": "on", "AMUN_WNARROW": str(_n)}
for _g in (2, 4):   # epilogue warpgroups (4 needs a -DAMUN_WITH_NG4 build, AMUN_LIB)
    VARIANTS[f"tail_ng{_g}"] = {"AMUN_TAIL": "on", "AMUN_NG": str(_g)}
for _b in (64, 256):
    VARIANTS[f"sep_box{_b}"] = {"AMUN_TAIL": "off", "AMUN_WBOX": str(_b)}
    VARIANTS[f"scores_box{_b}"] = {"AMUN_TAIL": "off", "AMUN_WBOX": str(_b)}
for _v in VARIANTS.values():
    _v.setdefault("AMUN_TAPER", "0")
    _v.setdefault("AMUN_PREPASS", "1")
    _v.setdefault("AMUN_MC", "0")
    _v.setdefault("AMUN_NG", "2")
    _v.setdefault("AMUN_WNARROW", "1")
NOCHECK = {v for v in VARIANTS if v.startswith("scores")} | {"tailwait", "waitnocoop", "arriveonly"}


def graph_us(fn, K, reps=5):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(K):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        out = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            out.append(s.elapsed_time(e) * 1e3 / K)
    return out


def main():
    names = sys.argv[1:] or ["greedy", "beam"]
    variants = os.environ.get("AB_VARIANTS", ",".join(VARIANTS)).split(",")
    dev = torch.device("cuda", 0)
    for name in names:
        # "beam@176": the cfg with S overridden (N = S x B)
        w = synth.CONFIGS[name.split("@")[0]]
        if "@" in name:
            import dataclasses
            w = dataclasses.replace(w, S=int(name.split("@")[1]))
        X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
        pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
        wbytes = W.numel() * W.element_size()
        ncopy = max(2, -(-2 * 126 * 2 ** 20 // wbytes))
        Ws = [W] + [W.clone() for _ in range(ncopy - 1)]
        K = int(os.environ.get("AB_K", "100" if w.N < 2000 else "10"))
        layers = {}
        for v in variants:
            os.environ.update(VARIANTS[v])
            layers[v] = amun.OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=w.N,
                                         max_sentences=w.S)
        ref = {}   # bit-identical outputs within one taper / NG setting (the
        # tile widths and warpgroup count decide which warpgroup sums which
        # chunk, so they differ in the last bits of the sums)
        res = {v: [] for v in variants}
        for rnd in range(3):
            for v in variants:
                ol = layers[v]
                oi = torch.empty((w.S, w.k), dtype=torch.int64, device=dev)
                oc = torch.empty((w.S, w.k), dtype=torch.float32, device=dev)

                def fn(i, ol=ol, oi=oi, oc=oc, v=v):
                    if v.startswith("scores"):
                        ol.scores(X, Ws[i % ncopy], b)
                    else:
                        ol(X, Ws[i % ncopy], b, pc, off, w.k, out_idx=oi, out_cost=oc)
                if os.environ.get("AB_SLEEP"):   # cool down between measurements (burst clocks)
                    import time
                    time.sleep(float(os.environ["AB_SLEEP"]))
                res[v] += graph_us(fn, K)
                if v in NOCHECK:
                    pass
                else:
                    t = (VARIANTS[v]["AMUN_TAPER"], VARIANTS[v]["AMUN_NG"])
                    if t not in ref:
                        ref[t] = (oi.clone(), oc.clone())
                    assert torch.equal(ref[t][0], oi) and torch.equal(ref[t][1], oc), v
        for v in variants:
            xs = sorted(res[v])
            print(json.dumps({"workload": name, "variant": v, "us_min": xs[0],
                              "us_med": xs[len(xs) // 2], "K": K, "w_copies": ncopy}), flush=True)


if __name__ == "__main__":
    main()
