"""GPU parity of the fp32 tensor-core path (dtype="tf32x3", SURVEY.md §8(f)
f2 "fp32 path"): the output layer (steps 1-4, P:152-200,
Alg. 4) computed on tcgen05 kind::tf32 with the 3xTF32 split
x.w ~= hi(x).hi(w) + hi(x).lo(w) + lo(x).hi(w), against the fp64 oracle on the
ORIGINAL fp32 values, at the fp32 tolerance of tests/compare.py (1e-4 rel,
north_star).

The split is one GEMM over K = 3H: X rows [hi | hi | lo], W rows
[hi | lo | hi] (amun_split_tf32x3). The dropped lo.lo term and the tf32
rounding of lo bound each product's relative error by ~2^-21, the same order
as fp32 accumulation itself."""
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


def split(X, W):
    m = amun()
    return m.split_tf32x3(X.to(DEV).contiguous(), "X"), m.split_tf32x3(W.to(DEV).contiguous(), "W")


def low13_zero(t):
    return bool(((t.view(torch.int32) & 0x1FFF) == 0).all())


@pytest.mark.parametrize("R,H", [(1, 4), (37, 96), (300, 1024), (5, 1028)])
def test_split_layout_and_precision(R, H):
    """hi, lo carry tf32 mantissas (13 low bits zero); |x - hi - lo| <=
    2^-21 |x|-ish; X rows are [hi | hi | lo], W rows [hi | lo | hi]."""
    g = torch.Generator().manual_seed(R * 1000 + H)
    x = (torch.randn(R, H, generator=g) * torch.exp(torch.randn(R, H, generator=g) * 3)).to(DEV)
    m = amun()
    sx, sw = m.split_tf32x3(x, "X"), m.split_tf32x3(x, "W")
    hi, hi2, lo = sx[:, :H], sx[:, H:2 * H], sx[:, 2 * H:]
    assert torch.equal(hi, hi2)
    assert torch.equal(sw[:, :H], hi) and torch.equal(sw[:, H:2 * H], lo) and torch.equal(sw[:, 2 * H:], hi)
    assert low13_zero(hi) and low13_zero(lo)
    # hi is x rounded to 10 mantissa bits: |x - hi| <= 2^-11 |x|
    assert ((x - hi).abs() <= x.abs() * 2.0 ** -11).all()
    # hi + lo reproduces x to ~21 bits
    assert ((x.double() - hi.double() - lo.double()).abs() <= x.abs().double() * 2.0 ** -21).all()


def test_split_special_values():
    x = torch.tensor([[0.0, -0.0, 1.0, -1.0, 3.0e38, 1e-40, 2.0 ** -126, 1.0 + 2.0 ** -23]], device=DEV)
    s = amun().split_tf32x3(x, "X")
    hi, lo = s[0, :8].cpu(), s[0, 16:].cpu()
    assert hi[2] == 1.0 and lo[2] == 0.0 and hi[3] == -1.0
    assert hi[0] == 0.0 and lo[0] == 0.0
    assert torch.isfinite(hi).all() and torch.isfinite(lo).all()
    assert float(hi[7]) + float(lo[7]) == 1.0 + 2.0 ** -23 or float(hi[7]) == 1.0


def run_case(w: synth.Workload, k_s=None, check_exact=False):
    X, W, b = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w)
    pc, off = synth.gen_prev_cost(w), synth.gen_offsets(w)
    S = off.numel() - 1
    Xs, Ws = split(X, W)
    ol = amun().OutputLayer(w.H, w.V, dtype="tf32x3", k_max=w.k, max_rows=max(X.shape[0], 1),
                            max_sentences=max(S, 1))
    ks_t = None if k_s is None else torch.as_tensor(k_s, dtype=torch.int32).to(DEV)
    idx, cost = ol(Xs, Ws, b.to(DEV), pc.to(DEV), off.to(DEV), w.k, ks_t)
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    logp = O.log_softmax(L) if L.shape[0] else L
    oi, oc32, oc64, nxt = O.kbest_sentences(logp, O.as_f64(pc), off.numpy(), w.k,
                                            None if k_s is None else np.asarray(k_s))
    pcd = O.as_f64(pc)
    ks = np.full(S, w.k) if k_s is None else np.minimum(np.asarray(k_s), w.k)
    return compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(),
                         lambda s, r, v: pcd[r] + logp[r, v], oc64, ks, "f32", w.V, o_next=nxt)


@pytest.mark.parametrize("H,V,S,B,k", [
    (64, 1000, 4, 2, 2),        # cfg tiny (BASELINE configs[0]) on the tensor cores
    (96, 3001, 11, 3, 4),       # V ragged, H = 3 K-blocks of 32
    (256, 1009, 37, 5, 5),      # 2 M-tiles, ragged rows
    (512, 65521, 9, 3, 7),      # prime vocab, many tiles per CTA
    (1024, 5000, 130, 2, 3),    # 3 M-tiles
    (68, 777, 5, 3, 2),         # 3H = 204: K not a multiple of 32 (TMA zero-fill)
    (64, 200, 60, 4, 16),       # k = 16 bucket
])
def test_output_layer_parity(H, V, S, B, k):
    w = synth.Workload("t3", H=H, V=V, S=S, B=B, k=k, dtype="f32", seed=synth.BASE_SEED + 40 + H + S)
    rep = run_case(w)
    assert rep["sentences_checked"] == S


def test_ragged_k_per_sentence():
    w = synth.Workload("t3", H=128, V=2000, S=9, B=4, k=6, dtype="f32", seed=synth.BASE_SEED + 77)
    run_case(w, k_s=[1, 6, 3, 0, 6, 2, 5, 6, 1])


def test_cfg_beam_shape_sampled():
    """cfg 'beam' shape (H=1024, V=90000, 128 x 5, k=5) with fp32 inputs."""
    w = synth.Workload("t3beam", H=1024, V=90000, S=128, B=5, k=5, dtype="f32",
                       seed=synth.BASE_SEED + 3)
    rep = run_case(w)
    assert rep["sentences_checked"] == 128


def test_integer_regime_logits_bit_exact():
    """|x|,|w| <= 8 integers: hi = x, lo = 0 and every product / sum is exact,
    so the biased logits equal the oracle's exactly."""
    rng = np.random.default_rng(3)
    for (N, V, H) in [(130, 1000, 256), (7, 4099, 64), (300, 513, 132)]:
        X = torch.from_numpy(rng.integers(-8, 9, (N, H)).astype(np.float32))
        W = torch.from_numpy(rng.integers(-8, 9, (V, H)).astype(np.float32))
        b = torch.from_numpy(rng.integers(-4, 5, V).astype(np.float32))
        Xs, Ws = split(X, W)
        ol = amun().OutputLayer(H, V, dtype="tf32x3", k_max=4, max_rows=N, max_sentences=N)
        L = ol.debug_logits(Xs, Ws, b.to(DEV)).cpu().numpy()
        ref = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
        assert np.array_equal(L.astype(np.float64), ref), (N, V, H)


@pytest.mark.parametrize("N,V,H", [(40, 700, 96), (200, 3000, 1024)])
def test_logits_fp32_accuracy(N, V, H):
    """Beyond the tf32 (10-bit) regime: the split must reach fp32-level error
    (single-pass tf32 would miss 1e-4 by ~100x at H = 1024)."""
    rng = np.random.default_rng(N)
    X = torch.from_numpy(rng.standard_normal((N, H)).astype(np.float32))
    W = torch.from_numpy(rng.standard_normal((V, H)).astype(np.float32))
    b = torch.from_numpy(rng.standard_normal(V).astype(np.float32))
    Xs, Ws = split(X, W)
    ol = amun().OutputLayer(H, V, dtype="tf32x3", k_max=2, max_rows=N, max_sentences=N)
    L = ol.debug_logits(Xs, Ws, b.to(DEV)).cpu().numpy()
    ref = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    scale = np.abs(O.as_f64(X)) @ np.abs(O.as_f64(W)).T      # sum |x w|
    assert (np.abs(L - ref) <= 1e-5 * scale + 1e-6).all(), np.abs(L - ref).max()


def test_argmax_parity():
    """Greedy (Alg. 5) on the tf32x3 plan: the token's oracle logit is within
    the fp32 accumulation band of the oracle maximum; integer regime exact."""
    rng = np.random.default_rng(5)
    N, V, H = 133, 7001, 512
    X = torch.from_numpy(rng.standard_normal((N, H)).astype(np.float32))
    W = torch.from_numpy((rng.standard_normal((V, H)) * 0.05).astype(np.float32))
    b = torch.from_numpy(rng.standard_normal(V).astype(np.float32))
    Xs, Ws = split(X, W)
    ol = amun().OutputLayer(H, V, dtype="tf32x3", k_max=1, max_rows=N, max_sentences=1)
    tok, logit = ol.argmax(Xs, Ws, b.to(DEV))
    tok, logit = tok.cpu().numpy(), logit.cpu().numpy()
    P = O.gemm(O.as_f64(X), O.as_f64(W))
    L = O.add_bias(P, O.as_f64(b))
    band = 1e-5 * (np.abs(O.as_f64(X)) @ np.abs(O.as_f64(W)).T).max(axis=1) + 1e-6
    best = L.max(axis=1)
    assert (L[np.arange(N), tok] >= best - 2 * band).all()
    assert np.allclose(logit, L[np.arange(N), tok], atol=1e-4)
    Xi = torch.from_numpy(rng.integers(-8, 9, (N, H)).astype(np.float32))
    Wi = torch.from_numpy(rng.integers(-8, 9, (V, H)).astype(np.float32))
    bi = torch.from_numpy(rng.integers(-4, 5, V).astype(np.float32))
    Xs, Ws = split(Xi, Wi)
    tok, _ = ol.argmax(Xs, Ws, bi.to(DEV))
    Pi = O.gemm(O.as_f64(Xi), O.as_f64(Wi))
    ref = np.array([O.argmax_1best(Pi[r], O.as_f64(bi)) for r in range(N)])
    assert np.array_equal(tok.cpu().numpy(), ref)


def test_device_n_and_partial_merge():
    """call_dev (row count on the device) and the vocab-shard partial + merge
    on the tf32x3 plan agree with the fused call."""
    w = synth.Workload("t3d", H=256, V=4000, S=20, B=3, k=4, dtype="f32", seed=synth.BASE_SEED + 91)
    X, W, b = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w)
    pc, off = synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    Xs, Ws = split(X, W)
    m = amun()
    ol = m.OutputLayer(w.H, w.V, dtype="tf32x3", k_max=w.k, max_rows=w.N, max_sentences=w.S)
    i0, c0 = ol(Xs, Ws, b.to(DEV), pc, off, w.k)
    nd = torch.tensor([w.N], dtype=torch.int32, device=DEV)
    i1, c1 = ol.call_dev(Xs, Ws, b.to(DEV), pc, off, nd, w.k)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(c0, c1)


@pytest.mark.parametrize("G", [2, 3])
def test_vocab_shards_partial_merge_and_oneshot(G):
    """tf32x3 plans on vocab shards: per-shard partial records + merge (the
    collective path) and the one-shot emulation give the same result, which
    passes the oracle comparator at the fp32 tolerance."""
    from paper_1805_09863_b200.sharded import EmulatedOneShot, shard_range
    w = synth.Workload("t3s", H=128, V=7001, S=10, B=3, k=4, dtype="f32", seed=synth.BASE_SEED + 120 + G)
    X, W, b = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w)
    pc, off = synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    m = amun()
    Xs = m.split_tf32x3(X.to(DEV), "X")
    layers, Ws, bs = [], [], []
    for g in range(G):
        v0, v1 = shard_range(w.V, G, g)
        layers.append(m.OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, dtype="tf32x3",
                                    k_max=w.k, max_rows=w.N, max_sentences=w.S))
        Ws.append(m.split_tf32x3(W[v0:v1].contiguous().to(DEV), "W"))
        bs.append(b[v0:v1].contiguous().to(DEV))
    parts = torch.stack([ol.partial(Xs, Wg, bg) for ol, Wg, bg in zip(layers, Ws, bs)])
    idx, cost = layers[0].merge(parts, pc, off, w.k)
    em = EmulatedOneShot(layers)
    for i, c in em(Xs, Ws, bs, pc, off, w.k):
        assert torch.equal(i, idx) and torch.equal(c, cost)
    em.close()
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.as_f64(X), O.as_f64(W)), O.as_f64(b))
    logp = O.log_softmax(L)
    _, _, oc64, nxt = O.kbest_sentences(logp, O.as_f64(synth.gen_prev_cost(w)), off.cpu().numpy(), w.k)
    pcd = O.as_f64(synth.gen_prev_cost(w))
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                  oc64, np.full(w.S, w.k), "f32", w.V, o_next=nxt)
