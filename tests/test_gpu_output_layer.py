"""GPU parity of the output-layer path (fused tcgen05/SIMT kernel + merge)
against the CPU oracle, element by element on the same seeded inputs.
All calls go through the C-ABI (libamun.so) via the thin binding."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests.compare import compare_kbest, compare_row_topk

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def amun():
    import paper_1805_09863_b200 as m
    return m


def run_case(w: synth.Workload, k_s=None, X=None, W=None, b=None, pc=None, off=None,
             exact_idx=False):
    X = synth.gen_X(w) if X is None else X
    W = synth.gen_W(w) if W is None else W
    b = synth.gen_b(w) if b is None else b
    pc = synth.gen_prev_cost(w) if pc is None else pc
    off = synth.gen_offsets(w) if off is None else off
    S = off.numel() - 1
    ol = amun().OutputLayer(w.H, w.V, dtype=w.dtype, k_max=w.k, max_rows=max(X.shape[0], 1),
                            max_sentences=max(S, 1))
    ks_t = None if k_s is None else torch.as_tensor(k_s, dtype=torch.int32).to(DEV)
    idx, cost = ol(X.to(DEV), W.to(DEV), b.to(DEV), pc.to(DEV), off.to(DEV), w.k, ks_t)
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    logp = O.log_softmax(L) if L.shape[0] else L
    oi, oc32, oc64, nxt = O.kbest_sentences(logp, O.as_f64(pc), off.numpy(), w.k,
                                            None if k_s is None else np.asarray(k_s))
    pcd = O.as_f64(pc)
    ks = np.full(S, w.k) if k_s is None else np.minimum(np.asarray(k_s), w.k)
    rep = compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(),
                        lambda s, r, v: pcd[r] + logp[r, v], oc64, ks, w.dtype, w.V, o_next=nxt)
    if exact_idx:
        assert np.array_equal(idx.cpu().numpy(), oi)
    return rep, idx.cpu().numpy(), oi


# ------------------------------------------------------------------ configs
def test_cfg_tiny_f32():
    """BASELINE cfg 'tiny': H=64, V=1000, 4 x 2, k=2, fp32 (SIMT, 1e-4 rel)."""
    rep, gi, oi = run_case(synth.CONFIGS["tiny"])
    assert rep["sentences_checked"] == 4


@pytest.mark.parametrize("H,V,S,B,k", [
    (256, 1009, 37, 5, 5),      # 2 M-tiles (185 rows, ragged), V not a multiple of 16
    (128, 3000, 3, 1, 1),       # greedy-like
    (512, 65521, 9, 3, 7),      # prime vocab, many tiles per CTA
    (64, 200, 60, 4, 16),       # k = 16 bucket, 240 rows
    (1024, 5000, 130, 2, 3),    # 260 rows -> 3 M-tiles, H = 1024
    (72, 777, 5, 3, 2),         # H not a multiple of 64 (TMA zero-fills K)
])
def test_bf16_shapes(H, V, S, B, k):
    w = synth.Workload("t", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + H + V)
    run_case(w)


def test_bf16_flat_distribution_near_ties():
    w = synth.Workload("flat", H=256, V=20000, S=20, B=4, k=8, dist="flat",
                       seed=synth.BASE_SEED + 11)
    run_case(w)


def test_f32_larger():
    w = synth.Workload("f32", H=96, V=3001, S=11, B=3, k=4, dtype="f32", seed=synth.BASE_SEED + 12)
    run_case(w)


def test_cfg_greedy_full():
    """BASELINE cfg 'greedy' at full size: H=512, V=60000, 128 x 1, k=1."""
    rep, gi, oi = run_case(synth.CONFIGS["greedy"])
    assert rep["sentences_checked"] == 128


@pytest.mark.slow
def test_cfg_beam_full():
    """BASELINE cfg 'beam' at full size (the bench workload, same launch):
    H=1024, V=90000, 128 x 5, k=5; every sentence checked."""
    rep, gi, oi = run_case(synth.CONFIGS["beam"])
    assert rep["sentences_checked"] == 128
    assert rep["max_abs_dcost"] < 1e-3


# ------------------------------------------------------------------ exact cases
def test_gex1_exact_with_ties():
    """SURVEY.md §8(c) GEX1, H padded to 8 with zeros; exact incl. tie order."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gex1.json")))
    X = torch.zeros(2, 8); X[:, :2] = torch.tensor(g["X"], dtype=torch.float32)
    W = torch.zeros(4, 8); W[:, :2] = torch.tensor(g["W"], dtype=torch.float32)
    b = torch.tensor(g["b"], dtype=torch.float32)
    pc = torch.tensor(g["prev_cost"], dtype=torch.float32)
    off = torch.tensor([0, 2], dtype=torch.int32)
    for dtype in ["bf16", "f32"]:
        for case in g["cases"]:
            w = synth.Workload("gex1", H=8, V=4, S=1, B=2, k=case["k"], dtype=dtype)
            Xd = X.to(torch.bfloat16) if dtype == "bf16" else X
            Wd = W.to(torch.bfloat16) if dtype == "bf16" else W
            rep, gi, oi = run_case(w, X=Xd, W=Wd, b=b, pc=pc, off=off, exact_idx=True)
            assert gi[0].tolist() == case["idx"]


def test_integer_regime_logits_bit_exact():
    """|x|,|w| <= 8 integers, H <= 256: products and sums are exact in bf16 x
    bf16 -> fp32, so the GEMM's biased logits must equal the oracle's exactly."""
    rng = np.random.default_rng(0)
    for (N, V, H) in [(130, 1000, 256), (7, 4099, 64), (300, 513, 128)]:
        X = torch.from_numpy(rng.integers(-8, 9, (N, H)).astype(np.float32)).to(torch.bfloat16)
        W = torch.from_numpy(rng.integers(-8, 9, (V, H)).astype(np.float32)).to(torch.bfloat16)
        b = torch.from_numpy(rng.integers(-4, 5, V).astype(np.float32))
        ol = amun().OutputLayer(H, V, k_max=4, max_rows=N, max_sentences=N)
        L = ol.debug_logits(X.to(DEV), W.to(DEV), b.to(DEV)).cpu().numpy()
        ref = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
        assert np.array_equal(L.astype(np.float64), ref), (N, V, H)


def test_f32_logits_close():
    rng = np.random.default_rng(1)
    N, V, H = 40, 700, 96
    X = torch.from_numpy(rng.standard_normal((N, H)).astype(np.float32))
    W = torch.from_numpy(rng.standard_normal((V, H)).astype(np.float32))
    b = torch.from_numpy(rng.standard_normal(V).astype(np.float32))
    ol = amun().OutputLayer(H, V, dtype="f32", k_max=2, max_rows=N, max_sentences=N)
    L = ol.debug_logits(X.to(DEV), W.to(DEV), b.to(DEV)).cpu().numpy()
    ref = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    assert np.abs(L - ref).max() < 1e-4


def test_unit_vector_rows():
    """X rows = e_j: L[r][v] = W[v][j] + b[v] exactly."""
    w = synth.Workload("u", H=64, V=2000, S=3, B=2, k=3)
    W = synth.gen_W(w)
    X = torch.zeros(6, 64)
    for r, j in enumerate([0, 5, 63, 17, 17, 40]):
        X[r, j] = 1.0
    X = X.to(torch.bfloat16)
    ol = amun().OutputLayer(64, 2000, k_max=3, max_rows=6, max_sentences=3)
    b = synth.gen_b(w)
    L = ol.debug_logits(X.to(DEV), W.to(DEV), b.to(DEV)).cpu()
    ref = (W.float()[:, [0, 5, 63, 17, 17, 40]] + b[:, None]).T
    assert torch.equal(L, ref)


# ------------------------------------------------------------------ adversarial
def _zero_w(H, V):
    return torch.zeros(V, H, dtype=torch.bfloat16)


def test_ascending_logits_every_element_inserts():
    """W = 0, b ascending in v: every logit beats the current k-th best."""
    H, V, S, B, k = 64, 9000, 4, 3, 16
    w = synth.Workload("asc", H=H, V=V, S=S, B=B, k=k)
    b = torch.arange(V, dtype=torch.float32) * 1e-3
    rep, gi, oi = run_case(w, W=_zero_w(H, V), b=b, exact_idx=True)


def test_duplicated_maxima_across_tiles_and_splits():
    H, V, S, B, k = 64, 50000, 2, 2, 4
    w = synth.Workload("dup", H=H, V=V, S=S, B=B, k=k)
    b = torch.zeros(V)
    for v in [7, 300, 12345, 49999, 25000]:
        b[v] = 3.0
    pc = torch.tensor([-1.0, -1.0, -2.0, -2.0])
    rep, gi, oi = run_case(w, W=_zero_w(H, V), b=b, pc=pc, exact_idx=True)
    assert [int(i) % V for i in gi[0]] == [7, 300, 12345, 25000]


def test_all_equal_rows_and_large_offset():
    H, V, S, B, k = 64, 90000, 2, 3, 5
    w = synth.Workload("eq", H=H, V=V, S=S, B=B, k=k)
    b = torch.full((V,), 1000.0)
    pc = torch.zeros(6)
    rep, gi, oi = run_case(w, W=_zero_w(H, V), b=b, pc=pc, exact_idx=True)
    assert gi[0].tolist() == [0, 1, 2, 3, 4]
    _, cost = None, None


def test_ragged_sentences_and_k_per_sentence():
    """Empty sentences, single-row sentences, k_s < k and k_s = 0."""
    H, V, k = 128, 4000, 6
    sizes = [0, 1, 5, 0, 2, 7, 1, 3]
    off = torch.tensor(np.concatenate([[0], np.cumsum(sizes)]), dtype=torch.int32)
    N = int(off[-1])
    w = synth.Workload("rag", H=H, V=V, S=len(sizes), B=1, k=k)
    X = synth.gen_X(synth.Workload("rag", H=H, V=V, S=N, B=1, k=k))
    pc = -torch.arange(N, dtype=torch.float32) * 0.1
    run_case(w, X=X, pc=pc, off=off, k_s=[6, 1, 3, 6, 0, 6, 2, 5])


def test_k_equals_all_candidates():
    """k = B*V (16) on a tiny vocabulary: every candidate, probs sum to 1."""
    H, V, S, B, k = 64, 8, 3, 2, 16
    w = synth.Workload("all", H=H, V=V, S=S, B=B, k=k)
    rep, gi, oi = run_case(w)
    X = synth.gen_X(w); pc = synth.gen_prev_cost(w)
    ol = amun().OutputLayer(H, V, k_max=k, max_rows=6, max_sentences=3)
    idx, cost = ol(X.to(DEV), synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV), pc.to(DEV),
                   synth.gen_offsets(w).to(DEV), k)
    idx, cost = idx.cpu().numpy(), cost.cpu().numpy()
    for s in range(S):
        assert sorted(idx[s].tolist()) == list(range(2 * s * V, 2 * s * V + 16))
        rows = idx[s] // V
        assert abs(np.exp(cost[s] - pc.numpy()[rows]).sum() - 2.0) < 1e-4


def test_empty_batch():
    ol = amun().OutputLayer(64, 100, k_max=2, max_rows=8, max_sentences=4)
    X = torch.empty(0, 64, dtype=torch.bfloat16, device=DEV)
    W = torch.zeros(100, 64, dtype=torch.bfloat16, device=DEV)
    b = torch.zeros(100, device=DEV)
    off = torch.zeros(4, dtype=torch.int32, device=DEV)
    idx, cost = ol(X, W, b, torch.empty(0, device=DEV), off, 2)
    torch.cuda.synchronize()
    assert (idx == -1).all() and torch.isneginf(cost).all()


# ------------------------------------------------------------------ shards
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_vocab_shard_emulation(G):
    """One-GPU emulation of the vocab-sharded path: G plans over V/G slices of
    the same global W (each slice regenerated from its global indices), their
    per-row partials stacked like an all-gather, then the exact merge.
    Must equal the oracle on the full vocabulary."""
    w = synth.Workload("shard", H=256, V=30000, S=16, B=4, k=6, seed=synth.BASE_SEED + 99)
    X, pc, off = synth.gen_X(w).to(DEV), synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    bounds = [0]
    per = -(-w.V // G)
    per = -(-per // 256) * 256
    while bounds[-1] < w.V:
        bounds.append(min(w.V, bounds[-1] + per))
    parts = []
    plans = []
    for g in range(len(bounds) - 1):
        v0, v1 = bounds[g], bounds[g + 1]
        ol = amun().OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, k_max=w.k,
                                max_rows=w.N, max_sentences=w.S)
        plans.append(ol)
        parts.append(ol.partial(X, synth.gen_W(w, v0, v1 - v0).to(DEV), synth.gen_b(w, v0, v1 - v0).to(DEV)))
    P = torch.stack(parts)
    idx, cost = plans[0].merge(P, pc, off, w.k)
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))), O.as_f64(synth.gen_b(w)))
    logp = O.log_softmax(L)
    oi, _, oc64, nxt = O.kbest_sentences(logp, O.as_f64(synth.gen_prev_cost(w)), off.cpu().numpy(), w.k)
    pcd = O.as_f64(synth.gen_prev_cost(w))
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                  oc64, np.full(w.S, w.k), "bf16", w.V, o_next=nxt)
    # the per-shard partial records themselves against the oracle's shard_partial
    Pn = P.cpu().numpy()
    for g in range(len(bounds) - 1):
        v0, v1 = bounds[g], bounds[g + 1]
        m, s, l, v = O.shard_partial(L[:, v0:v1], w.k, v_offset=v0)
        assert np.allclose(Pn[g, :, 0], m, atol=1e-4)
        assert np.allclose(Pn[g, :, 1], s, rtol=1e-4)
        compare_row_topk(Pn[g, :, 2:2 + w.k], Pn[g, :, 2 + w.k:].view(np.int32), L[:, v0:v1],
                         w.k, band=1e-4, v_offset=v0)


def test_partial_record_layout():
    """Partial of the whole vocabulary: m = max logit, s = sum exp(l - m),
    top-k ids; compared with oracle shard_partial."""
    w = synth.Workload("p", H=128, V=5000, S=10, B=3, k=5)
    X, W, b = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w)
    ol = amun().OutputLayer(w.H, w.V, k_max=5, max_rows=w.N, max_sentences=w.S)
    P = ol.partial(X.to(DEV), W.to(DEV), b.to(DEV)).cpu().numpy()
    L = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    m, s, l, v = O.shard_partial(L, 5)
    assert P.shape == (w.N, 12)
    assert np.abs(P[:, 0] - m).max() < 1e-4
    assert np.allclose(P[:, 1], s, rtol=1e-4)
    assert np.abs(P[:, 2:7] - l).max() < 1e-4
    compare_row_topk(P[:, 2:7], P[:, 7:12].view(np.int32), L, 5, band=1e-4)


def test_invalid_k_rejected():
    ol = amun().OutputLayer(64, 100, k_max=2, max_rows=8, max_sentences=4)
    X = torch.zeros(2, 64, dtype=torch.bfloat16, device=DEV)
    W = torch.zeros(100, 64, dtype=torch.bfloat16, device=DEV)
    b = torch.zeros(100, device=DEV)
    with pytest.raises(amun().AmunError):
        ol(X, W, b, torch.zeros(2, device=DEV), torch.tensor([0, 2], dtype=torch.int32, device=DEV), 3)


# ------------------------------------------------------------------ CTA-pair kernel
@pytest.mark.parametrize("N,V,H,k", [(300, 4099, 128, 5), (640, 9000, 256, 5), (130, 1000, 64, 3)])
def test_pair_kernel_forced(N, V, H, k, monkeypatch):
    """The tcgen05 cta_group::2 kernel on odd M-tile counts (a padded pair) and
    small cases, forced with AMUN_PAIRS=force (read at plan creation)."""
    monkeypatch.setenv("AMUN_PAIRS", "force")
    S = N // 5 if N % 5 == 0 else N
    B = N // S
    w = synth.Workload("pairs", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + N)
    run_case(w)
    # integer regime bit-exact through the pair kernel
    rng = np.random.default_rng(N)
    X = torch.from_numpy(rng.integers(-8, 9, (N, H)).astype(np.float32)).to(torch.bfloat16)
    W = torch.from_numpy(rng.integers(-8, 9, (V, H)).astype(np.float32)).to(torch.bfloat16)
    b = torch.from_numpy(rng.integers(-4, 5, V).astype(np.float32))
    ol = amun().OutputLayer(H, V, k_max=4, max_rows=N, max_sentences=N)
    L = ol.debug_logits(X.to(DEV), W.to(DEV), b.to(DEV)).cpu().numpy()
    ref = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    assert np.array_equal(L.astype(np.float64), ref)


# ------------------------------------------------------------------ CUDA graphs
@pytest.mark.parametrize("N", [640, 250])
def test_graph_replay_with_new_inputs(N):
    """The path is CUDA-graph capturable; each replay must see fresh cross-CTA
    k-th-best hints (a device-side launch generation), so replaying the same
    graph on NEW X contents stays exact."""
    H, V, B, k = 256, 20000, 5, 5
    S = N // B
    dev = DEV
    ol = amun().OutputLayer(H, V, k_max=k, max_rows=N, max_sentences=S)
    base = synth.Workload("g", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + 500)
    W, b = synth.gen_W(base).to(dev), synth.gen_b(base).to(dev)
    pc, off = synth.gen_prev_cost(base).to(dev), synth.gen_offsets(base).to(dev)
    Xbuf = torch.empty(N, H, dtype=torch.bfloat16, device=dev)
    oi = torch.empty(S, k, dtype=torch.int64, device=dev)
    oc = torch.empty(S, k, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        Xbuf.copy_(synth.gen_X(base).to(dev))
        ol(Xbuf, W, b, pc, off, k, out_idx=oi, out_cost=oc)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            ol(Xbuf, W, b, pc, off, k, out_idx=oi, out_cost=oc)
    Wo, bo = O.as_f64(synth.gen_W(base)), O.as_f64(synth.gen_b(base))
    pcd = O.as_f64(synth.gen_prev_cost(base))
    for rep in range(3):
        w = synth.Workload("g", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + 600 + rep)
        Xh = synth.gen_X(w)
        Xbuf.copy_(Xh.to(dev))
        g.replay()
        torch.cuda.synchronize()
        logp = O.log_softmax(O.add_bias(O.gemm(O.as_f64(Xh), Wo), bo))
        _, _, oc64, nxt = O.kbest_sentences(logp, pcd, off.cpu().numpy(), k)
        compare_kbest(oi.cpu().numpy(), oc.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                      oc64, np.full(S, k), "bf16", V, o_next=nxt)


# ------------------------------------------------------------------ full-size sampled parity
def _sampled_oracle_check(w, idx, cost, sentences, V_total):
    """Oracle on the sampled sentences only (all their rows, full vocabulary)."""
    Xh, pch, offh = synth.gen_X(w), synth.gen_prev_cost(w), synth.gen_offsets(w)
    rows = np.concatenate([np.arange(int(offh[s]), int(offh[s + 1])) for s in sentences])
    Wo, bo = O.as_f64(synth.gen_W(w)), O.as_f64(synth.gen_b(w))
    L = O.add_bias(O.gemm(O.as_f64(Xh[torch.from_numpy(rows)]), Wo), bo)
    logp = O.log_softmax(L)
    pcs = O.as_f64(pch)[rows]
    sub_off = np.concatenate([[0], np.cumsum([int(offh[s + 1] - offh[s]) for s in sentences])])
    _, _, oc64, nxt = O.kbest_sentences(logp, pcs, sub_off, w.k)
    pos = {int(r): i for i, r in enumerate(rows)}
    gi = idx.cpu().numpy()[sentences]
    gc = cost.cpu().numpy()[sentences]
    # GPU indices are r * V_total + v with global r; the oracle sees the sampled rows
    return compare_kbest(gi, gc, lambda s, r, v: pcs[pos[r]] + logp[pos[r], v], oc64,
                         np.full(len(sentences), w.k), "bf16", V_total, o_next=nxt)


@pytest.mark.slow
def test_cfg_shard_full_size_sampled():
    """BASELINE cfg 'shard' at full size on one GPU (H=1024, V=256000, 1024 x 12,
    k=12; 96 M-tiles -> the CTA-pair kernel): every 64th sentence (16 sentences,
    192 rows, full vocabulary) against the oracle."""
    w = synth.CONFIGS["shard"]
    dev = DEV
    ol = amun().OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    X, W, b = synth.gen_X(w).to(dev), synth.gen_W(w).to(dev), synth.gen_b(w).to(dev)
    pc, off = synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
    idx, cost = ol(X, W, b, pc, off, w.k)
    torch.cuda.synchronize()
    del W
    rep = _sampled_oracle_check(w, idx, cost, list(range(0, w.S, 64)), w.V)
    assert rep["sentences_checked"] == 16


@pytest.mark.slow
def test_cfg_shard_vocab_sharded_8_sampled():
    """The 8-way vocab-sharded path at cfg 'shard' size, emulated on one GPU:
    8 plans over V/8 slices (partial records), stacked like the all-gather,
    exact merge; every 128th sentence against the oracle."""
    from paper_1805_09863_b200.sharded import shard_range
    w = synth.CONFIGS["shard"]
    dev = DEV
    X, pc, off = synth.gen_X(w).to(dev), synth.gen_prev_cost(w).to(dev), synth.gen_offsets(w).to(dev)
    parts, plans = [], []
    for g in range(8):
        v0, v1 = shard_range(w.V, 8, g)
        ol = amun().OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, k_max=w.k,
                                max_rows=w.N, max_sentences=w.S)
        plans.append(ol)
        parts.append(ol.partial(X, synth.gen_W(w, v0, v1 - v0).to(dev),
                                synth.gen_b(w, v0, v1 - v0).to(dev)))
    idx, cost = plans[0].merge(torch.stack(parts), pc, off, w.k)
    torch.cuda.synchronize()
    rep = _sampled_oracle_check(w, idx, cost, list(range(0, w.S, 128)), w.V)
    assert rep["sentences_checked"] == 8
