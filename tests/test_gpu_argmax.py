"""GPU parity of the greedy argmax path (Alg. 5; amun_argmax)
against the oracle (oracle.argmax_1best: argmax of p + b, lowest index on
ties), element by element through the C-ABI.

Where floating point decides the integer (the argmax), the GPU decides in
its own precision (bf16 products, fp32 accumulation) and the oracle in fp64;
away from the integer regime a GPU token is accepted iff its oracle logit is
within the a-priori fp32 accumulation bound of the oracle maximum:
  |L32 - L64| <= band = H 2^-24 max_v sum_h |x_h w_vh| + |L| 2^-24
(standard recursive-summation bound; bf16 x bf16 products are exact in fp32),
so two candidates closer than 2 band may legitimately swap (G16).
In the integer regime every value is exact and the token must match."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def amun():
    import paper_1805_09863_b200 as m
    return m


def run_argmax(H, V, X, W, b, dtype="bf16", exact=False):
    N = X.shape[0]
    ol = amun().OutputLayer(H, V, dtype=dtype, k_max=1, max_rows=max(N, 1), max_sentences=1)
    tok, logit = ol.argmax(X.to(DEV), W.to(DEV), b.to(DEV))
    torch.cuda.synchronize()
    tok, logit = tok.cpu().numpy(), logit.cpu().numpy()
    X64, W64, b64 = O.as_f64(X), O.as_f64(W), O.as_f64(b)
    P = O.gemm(X64, W64)
    L = O.add_bias(P, b64)
    ref = np.array([O.argmax_1best(P[r], b64) for r in range(N)], dtype=np.int64)
    if exact:
        assert np.array_equal(tok, ref)
        assert np.array_equal(logit.astype(np.float64), L[np.arange(N), ref])
        return tok, ref
    ulp = 2.0 ** -24
    terms = 1 if dtype == "bf16" else 2      # f32: the products are rounded too
    band = terms * H * ulp * (np.abs(X64) @ np.abs(W64).T).max(axis=1) + np.abs(L).max(axis=1) * ulp
    rows = np.arange(N)
    assert (tok >= 0).all() and (tok < V).all()
    gap = L[rows, ref] - L[rows, tok]
    assert (gap <= 2 * band).all(), (np.max(gap / band), np.argmax(gap - 2 * band))
    assert np.all(np.abs(logit - L[rows, tok]) <= band + 1e-7), np.max(np.abs(logit - L[rows, tok]))
    return tok, ref


def test_argmax_cfg_greedy_full():
    """BASELINE cfg 'greedy' (H=512, V=60k, 128 rows) in argmax-only mode."""
    w = synth.CONFIGS["greedy"]
    tok, ref = run_argmax(w.H, w.V, synth.gen_X(w), synth.gen_W(w), synth.gen_b(w))
    assert (tok == ref).mean() > 0.99


@pytest.mark.parametrize("H,V,N", [
    (256, 1009, 185),      # 2 M-tiles, ragged, V not a multiple of 16
    (64, 200, 5),          # one CTA range per row, tiny vocab
    (256, 30000, 640),     # 5 M-tiles, >= 4 tiles per CTA range: cross-CTA hints on
    (72, 777, 300),        # H not a multiple of 64
])
def test_argmax_shapes(H, V, N):
    w = synth.Workload("am", H=H, V=V, S=N, B=1, k=1, seed=synth.BASE_SEED + 31 + H + V)
    run_argmax(H, V, synth.gen_X(w), synth.gen_W(w), synth.gen_b(w))


def test_argmax_integer_regime_exact_and_ties():
    """Integer |x|,|w| <= 8, H <= 256: every logit exact; many exact ties
    (small integer range) must resolve to the lowest token id, across tiles
    and vocab splits."""
    rng = np.random.default_rng(5)
    for N, H, V in [(130, 64, 40000), (7, 32, 999), (640, 128, 20000)]:
        X = torch.from_numpy(rng.integers(-2, 3, (N, H)).astype(np.float32)).to(torch.bfloat16)
        W = torch.from_numpy(rng.integers(-2, 3, (V, H)).astype(np.float32)).to(torch.bfloat16)
        b = torch.from_numpy(rng.integers(-1, 2, V).astype(np.float32))
        run_argmax(H, V, X, W, b, exact=True)


def test_argmax_duplicated_maxima_lowest_id():
    H, V, N = 64, 50000, 3
    X = torch.zeros(N, H, dtype=torch.bfloat16)
    W = torch.zeros(V, H, dtype=torch.bfloat16)
    b = torch.zeros(V)
    for v in [49999, 25000, 12345, 300, 7]:
        b[v] = 3.0
    tok, ref = run_argmax(H, V, X, W, b, exact=True)
    assert tok.tolist() == [7, 7, 7]


def test_argmax_f32_simt():
    w = synth.CONFIGS["tiny"]
    run_argmax(w.H, w.V, synth.gen_X(w), synth.gen_W(w), synth.gen_b(w), dtype="f32")


def test_argmax_pair_kernel_forced(monkeypatch):
    monkeypatch.setenv("AMUN_PAIRS", "force")
    rng = np.random.default_rng(9)
    N, H, V = 300, 128, 4099
    X = torch.from_numpy(rng.integers(-3, 4, (N, H)).astype(np.float32)).to(torch.bfloat16)
    W = torch.from_numpy(rng.integers(-3, 4, (V, H)).astype(np.float32)).to(torch.bfloat16)
    b = torch.from_numpy(rng.integers(-2, 3, V).astype(np.float32))
    run_argmax(H, V, X, W, b, exact=True)


def test_argmax_agrees_with_k1_beam_path():
    """Alg. 5 = Alg. 4 with k = 1: the argmax token equals the
    k = 1 winner of the full softmax path (one row per sentence, prev_cost 0)."""
    w = synth.Workload("agree", H=256, V=20000, S=96, B=1, k=1, seed=synth.BASE_SEED + 77)
    X, W, b = synth.gen_X(w).to(DEV), synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV)
    ol = amun().OutputLayer(w.H, w.V, k_max=1, max_rows=w.N, max_sentences=w.S)
    tok, logit = ol.argmax(X, W, b)
    idx, cost = ol(X, W, b, torch.zeros(w.N, device=DEV), synth.gen_offsets(w).to(DEV), 1)
    torch.cuda.synchronize()
    assert torch.equal(tok.cpu(), (idx[:, 0] % w.V).cpu())


def test_argmax_empty_batch():
    ol = amun().OutputLayer(64, 100, k_max=1, max_rows=4, max_sentences=1)
    tok, logit = ol.argmax(torch.zeros(0, 64, dtype=torch.bfloat16, device=DEV),
                           torch.zeros(100, 64, dtype=torch.bfloat16, device=DEV),
                           torch.zeros(100, device=DEV))
    assert tok.numel() == 0 and logit.numel() == 0
