"""Small-shape runs of every kernel of the path, for compute-sanitizer
(SURVEY.md §4 test tiers: memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Shapes are cfg1/cfg2-like and a small cfg3 (several M-tiles, ragged V and N,
so the vocabulary tail, the row tail and the multi-CTA merge are exercised).
Each case runs the C-ABI path once and checks the result against the oracle
(so a sanitizer-clean run is also a correct one). Prints one line per case.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from tests.compare import compare_kbest  # noqa: E402

DEV = torch.device("cuda", 0)


def amun():
    import paper_1805_09863_b200 as m
    return m


def check_beam(w, idx, cost, dtype="bf16"):
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))),
                   O.as_f64(synth.gen_b(w)))
    logp = O.log_softmax(L)
    pcd = O.as_f64(synth.gen_prev_cost(w))
    _, _, oc64, nxt = O.kbest_sentences(logp, pcd, synth.gen_offsets(w).numpy(), w.k)
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                  oc64, np.full(w.S, w.k), dtype, w.V, o_next=nxt)


def inputs(w):
    return (synth.gen_X(w).to(DEV), synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV),
            synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV))


def case_beam(pairs, tail="on"):
    os.environ["AMUN_PAIRS"] = pairs
    os.environ["AMUN_TAIL"] = tail
    w = synth.Workload("san", H=256, V=3001, S=52, B=5, k=5, seed=synth.BASE_SEED + 900)
    X, W, b, pc, off = inputs(w)
    ol = amun().OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X, W, b, pc, off, w.k)
    torch.cuda.synchronize()
    check_beam(w, idx, cost)
    # determinism (a race would show as run-to-run differences): bit-equal again
    for _ in range(3):
        i2, c2 = ol(X, W, b, pc, off, w.k)
        torch.cuda.synchronize()
        assert torch.equal(i2, idx) and torch.equal(c2, cost), "nondeterministic output"
    os.environ.pop("AMUN_PAIRS")
    os.environ.pop("AMUN_TAIL")


def case_beam_single():
    case_beam("off")


def case_beam_pairs():
    case_beam("force")


def case_beam_sep():
    """The two-kernel form (fused kernel, then the separate merge kernel)."""
    case_beam("off", tail="off")


def case_oneshot_real():
    """The one-shot exchange in the fused kernel's tail, real mode at world 1
    (IPC-exported buffer, self-signal), equal to the single-GPU path."""
    from paper_1805_09863_b200.sharded import ShardedOutputLayer
    w = synth.Workload("san", H=256, V=3001, S=30, B=5, k=5, seed=synth.BASE_SEED + 908)
    X, W, b, pc, off = inputs(w)
    sh = ShardedOutputLayer(w.H, w.V, 1, 0, k_max=w.k, max_rows=w.N, max_sentences=w.S,
                            exchange="oneshot")
    ref = sh.ol(X, W, b, pc, off, w.k)
    for _ in range(3):
        i2, c2 = sh(X, W, b, pc, off, w.k)
        torch.cuda.synchronize()
        assert torch.equal(i2, ref[0]) and torch.equal(c2, ref[1])
    assert not sh.oneshot.error()
    sh.oneshot.close()


def case_greedy():
    w = synth.Workload("san", H=512, V=6000, S=100, B=1, k=1, seed=synth.BASE_SEED + 901)
    X, W, b, pc, off = inputs(w)
    ol = amun().OutputLayer(w.H, w.V, k_max=1, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X, W, b, pc, off, 1)
    tok, logit = ol.argmax(X, W, b)
    torch.cuda.synchronize()
    check_beam(w, idx, cost)
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))),
                   O.as_f64(synth.gen_b(w)))
    lo = L[np.arange(w.N), tok.cpu().numpy()]
    assert np.all(L.max(1) - lo <= 1e-3 * np.abs(L).max()), "argmax off"


def case_dev():
    w = synth.Workload("san", H=256, V=3001, S=30, B=5, k=5, seed=synth.BASE_SEED + 902)
    X, W, b, pc, off = inputs(w)
    ol = amun().OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    n_dev = torch.tensor([w.N], dtype=torch.int32, device=DEV)
    idx, cost = ol.call_dev(X, W, b, pc, off, n_dev, w.k)
    torch.cuda.synchronize()
    check_beam(w, idx, cost)


def case_shards():
    from paper_1805_09863_b200.sharded import shard_range
    w = synth.Workload("san", H=256, V=3001, S=30, B=5, k=5, seed=synth.BASE_SEED + 903)
    X, _, _, pc, off = inputs(w)
    G = 2
    layers, Ws, bs = [], [], []
    for g in range(G):
        v0, v1 = shard_range(w.V, G, g)
        layers.append(amun().OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, k_max=w.k,
                                         max_rows=w.N, max_sentences=w.S))
        Ws.append(synth.gen_W(w, v0, v1 - v0).to(DEV))
        bs.append(synth.gen_b(w, v0, v1 - v0).to(DEV))
    parts = torch.stack([ol.partial(X, Wg, bg) for ol, Wg, bg in zip(layers, Ws, bs)])
    idx, cost = layers[0].merge(parts, pc, off, w.k)
    torch.cuda.synchronize()
    check_beam(w, idx, cost)
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    em = EmulatedOneShot(layers)
    outs = em(X, Ws, bs, pc, off, w.k)
    torch.cuda.synchronize()
    for i2, c2 in outs:
        assert torch.equal(i2, idx) and torch.equal(c2, cost)
    em.close()


def case_e4m3():
    w = synth.Workload("san", H=256, V=3001, S=30, B=5, k=5, seed=synth.BASE_SEED + 904)
    X, W, b, pc, off = inputs(w)
    X8, xs = amun().quantize_e4m3(X)
    W8, ws = amun().quantize_e4m3(W)
    ol = amun().OutputLayer(w.H, w.V, dtype="e4m3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol.call_e4m3(X8, xs, W8, ws, b, pc, off, w.k)
    torch.cuda.synchronize()
    assert (idx >= 0).all()


def case_mxfp4():
    """MXFP4 W: both tile widths (256 / 128), 3 M-tiles, k = 5 and the k = 1
    argmax; 3 bit-determinism repeats."""
    w = synth.Workload("san", H=256, V=30001, S=60, B=5, k=5, seed=synth.BASE_SEED + 907)
    X, W, b, pc, off = inputs(w)
    X8, xs = amun().quantize_e4m3(X)
    W4, sf = amun().quantize_mxfp4(W)
    ol = amun().OutputLayer(w.H, w.V, dtype="mxfp4", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    ref = None
    for _ in range(3):
        idx, cost = ol.call_mxfp4(X8, xs, W4, sf, b, pc, off, w.k)
        torch.cuda.synchronize()
        if ref is None:
            ref = (idx.clone(), cost.clone())
        assert torch.equal(ref[0], idx) and torch.equal(ref[1], cost)
    assert (idx >= 0).all()
    tok, logit = ol.argmax_mxfp4(X8, xs, W4, sf, b)
    torch.cuda.synchronize()
    assert (tok >= 0).all() and (tok < w.V).all()


def case_tf32x3():
    w = synth.Workload("san", H=128, V=2001, S=20, B=5, k=5, dtype="f32", seed=synth.BASE_SEED + 905)
    X, W, b, pc, off = inputs(w)
    X3 = amun().split_tf32x3(X, "X")
    W3 = amun().split_tf32x3(W, "W")
    ol = amun().OutputLayer(w.H, w.V, dtype="tf32x3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X3, W3, b, pc, off, w.k)
    torch.cuda.synchronize()
    check_beam(w, idx, cost, "f32")


def case_simt():
    w = synth.Workload("san", H=64, V=1000, S=4, B=2, k=2, dtype="f32", seed=synth.BASE_SEED + 906)
    X, W, b, pc, off = inputs(w)
    ol = amun().OutputLayer(w.H, w.V, dtype="f32", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X, W, b, pc, off, w.k)
    torch.cuda.synchronize()
    check_beam(w, idx, cost, "f32")


def case_compact():
    N, S = 1003, 201
    off = torch.tensor(np.linspace(0, N, S + 1).astype(np.int32), device=DEV)
    alive = synth.gen_alive(11, N, 0.6).to(DEV)
    state = synth.gen_bytes(12, synth.S_STATE, N * 52).view(N, 52).to(DEV)
    dst = torch.empty_like(state)
    n, s_alive, new_off, src_row, _ = amun().compact([(state, dst)], alive, off)
    cols, no, src, n_ref, s_ref = O.compact([state.cpu().numpy()], alive.cpu().numpy(),
                                            off.cpu().numpy())
    assert n == n_ref and np.array_equal(dst[:n].cpu().numpy(), cols[0])


def case_beam_advance():
    w = synth.Workload("san", H=256, V=3001, S=30, B=5, k=5, seed=synth.BASE_SEED + 907)
    X, W, b, pc, off = inputs(w)
    ol = amun().OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X, W, b, pc, off, w.k)
    state = synth.gen_bytes(13, synth.S_STATE, w.N * 64).view(w.N, 64).to(DEV)
    dst = torch.empty((w.S * w.k, 64), dtype=state.dtype, device=DEV)
    eos = int((idx[0, 0] % w.V).item())
    amun().beam_advance(idx, cost, w.V, eos, w.N, [(state, dst)])
    torch.cuda.synchronize()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_") and callable(v)
         and k not in ("case_beam",)}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n}: ok", flush=True)
