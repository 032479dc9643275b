"""amun_output_layer_dev (row count in device memory, NEXT f1): bit-identical
to the host-N path on the same (single-CTA) kernel, and a decode chain
output layer -> beam advance -> output layer ... with N' never leaving the
device, captured in ONE CUDA graph and replayed, equal to the eager chain."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests.compare import compare_kbest

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def amun():
    import paper_1805_09863_b200 as m
    return m


@pytest.mark.parametrize("N,B,M,pairs", [
    (0, 5, 1024, "off"), (1, 1, 1024, "off"), (127, 1, 1024, "off"), (128, 4, 1024, "off"),
    (200, 5, 1024, "off"), (640, 5, 1024, "off"), (1000, 4, 1024, "off"),
    # max_rows >= 9 M-tiles: the _dev path runs CTA pairs (host reference forced to pairs)
    (300, 5, 1280, "force"), (1000, 4, 1280, "force"), (1280, 5, 1280, "force"), (0, 5, 1280, "force"),
])
def test_device_n_equals_host_n(N, B, M, pairs, monkeypatch):
    monkeypatch.setenv("AMUN_PAIRS", pairs)          # same kernel + schedule on both paths
    H, V, k = 256, 30000, 4
    S = max(N // B, 1) if N else 1
    w = synth.Workload("dn", H=H, V=V, S=S, B=B if N else 1, k=k, seed=synth.BASE_SEED + 500 + N)
    ol = amun().OutputLayer(H, V, k_max=k, max_rows=M, max_sentences=S)
    W, b = synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV)
    Xf = torch.randn(M, H, device=DEV).to(torch.bfloat16) * 7          # garbage beyond N
    pcf = torch.randn(M, device=DEV) * 100
    rows = S * B if N else 0
    if rows:
        Xf[:rows] = synth.gen_X(w).to(DEV)
        pcf[:rows] = synth.gen_prev_cost(w).to(DEV)
    off = (torch.arange(S + 1, dtype=torch.int32) * (B if N else 0)).to(DEV)
    n_dev = torch.tensor([rows], dtype=torch.int32, device=DEV)
    i_d, c_d = ol.call_dev(Xf, W, b, pcf, off, n_dev, k)
    i_h, c_h = ol(Xf[:rows].contiguous(), W, b, pcf[:rows].contiguous(), off, k)
    torch.cuda.synchronize()
    assert torch.equal(i_d, i_h)
    assert torch.equal(c_d.view(torch.int32), c_h.view(torch.int32))
    if rows == 640:    # and against the oracle
        L = O.add_bias(O.gemm(O.as_f64(Xf[:rows].cpu()), O.as_f64(W.cpu())), O.as_f64(b.cpu()))
        logp = O.log_softmax(L)
        pcd = O.as_f64(pcf[:rows].cpu())
        oi, oc32, oc64, nxt = O.kbest_sentences(logp, pcd, off.cpu().numpy(), k)
        compare_kbest(i_d.cpu().numpy(), c_d.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                      oc64, np.full(S, k), "bf16", V, o_next=nxt)


def test_decode_chain_in_one_graph(monkeypatch):
    monkeypatch.setenv("AMUN_PAIRS", "off")
    H, V, S, B, k, T = 256, 8000, 40, 4, 4, 4
    M = S * k
    w = synth.Workload("chain", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + 600)
    W, b = synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV)
    ol = amun().OutputLayer(H, V, k_max=k, max_rows=M, max_sentences=S)
    eos = 0                                            # the most likely token (zipf prior): beams shrink
    X0 = torch.zeros(M, H, dtype=torch.bfloat16, device=DEV)
    X0[:S * B] = synth.gen_X(w).to(DEV)
    pc0 = torch.zeros(M, device=DEV)
    pc0[:S * B] = synth.gen_prev_cost(w).to(DEV)
    off0 = synth.gen_offsets(w).to(DEV)

    def make_state():
        return {"X": [X0.clone(), torch.zeros_like(X0)], "pc": [pc0.clone(), torch.zeros_like(pc0)],
                "off": [off0.clone(), torch.zeros_like(off0)],
                "n": [torch.tensor([S * B], dtype=torch.int32, device=DEV),
                      torch.zeros(2, dtype=torch.int32, device=DEV)],
                "src": torch.zeros(M, dtype=torch.int32, device=DEV),
                "tok": torch.zeros(M, dtype=torch.int32, device=DEV),
                "ws": torch.zeros(4096, dtype=torch.uint8, device=DEV),
                "idx": torch.zeros((S, k), dtype=torch.int64, device=DEV),
                "cost": torch.zeros((S, k), dtype=torch.float32, device=DEV),
                "log": []}

    def step(st, t, eager):
        a, c = t % 2, (t + 1) % 2
        if eager:    # host N: the reference chain (syncs every step)
            n = int(st["n"][a][0].item())
            ol(st["X"][a][:n].contiguous(), W, b, st["pc"][a][:n].contiguous(), st["off"][a], k,
               out_idx=st["idx"], out_cost=st["cost"])
        else:
            ol.call_dev(st["X"][a], W, b, st["pc"][a], st["off"][a], st["n"][a][:1], k,
                        out_idx=st["idx"], out_cost=st["cost"])
        amun().beam_advance(st["idx"], st["cost"], V, eos, M, [(st["X"][a], st["X"][c])], sync=False,
                            out={"new_offsets": st["off"][c], "src_row": st["src"], "new_token": st["tok"],
                                 "new_cost": st["pc"][c], "counts": st["n"][c], "workspace": st["ws"]})
        st["log"].append((st["idx"].clone(), st["cost"].clone()))

    ref = make_state()
    for t in range(T):
        step(ref, t, eager=True)
    torch.cuda.synchronize()

    g_state = make_state()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step(make_state(), 0, eager=False)             # warm-up (plans, maps) outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        logs = []
        with torch.cuda.graph(g, stream=s):
            for t in range(T):
                a, c = t % 2, (t + 1) % 2
                ol.call_dev(g_state["X"][a], W, b, g_state["pc"][a], g_state["off"][a],
                            g_state["n"][a][:1], k, out_idx=g_state["idx"], out_cost=g_state["cost"])
                logs.append((g_state["idx"].clone(), g_state["cost"].clone()))
                amun().beam_advance(g_state["idx"], g_state["cost"], V, eos, M,
                                    [(g_state["X"][a], g_state["X"][c])], sync=False,
                                    out={"new_offsets": g_state["off"][c], "src_row": g_state["src"],
                                         "new_token": g_state["tok"], "new_cost": g_state["pc"][c],
                                         "counts": g_state["n"][c], "workspace": g_state["ws"]})
    g.replay()
    torch.cuda.synchronize()
    sizes = []
    for t in range(T):
        assert torch.equal(logs[t][0], ref["log"][t][0]), t
        assert torch.equal(logs[t][1].view(torch.int32), ref["log"][t][1].view(torch.int32)), t
    n_final = int(g_state["n"][T % 2][0].item())
    assert n_final == int(ref["n"][T % 2][0].item())
    assert n_final < S * B        # EOS winners left the batch
