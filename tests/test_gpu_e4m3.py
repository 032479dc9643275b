"""FP8 (E4M3) output layer (NEXT f4; amun_output_layer_e4m3, amun_quantize_e4m3)
against the oracle: the GPU quantiser bit-exact, and the k-best of the
e4m3 x e4m3 -> fp32 kernel against the oracle run on the exactly
dequantised values (oracle.dequant_rows_e4m3), with the same comparator and
tolerance as the bf16 path (both accumulate exact products in fp32)."""
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


@pytest.mark.parametrize("src_dtype", [torch.float32, torch.bfloat16])
def test_quantize_bit_exact(src_dtype):
    rng = np.random.default_rng(4)
    R, H = 300, 1040
    x = (rng.normal(size=(R, H)) * np.exp(rng.normal(size=(R, 1)) * 4)).astype(np.float32)
    x[7] = 0.0                                        # all-zero row -> scale 1
    x[8, ::3] = 0.0
    x[9, 5] = 1e30                                    # huge dynamic range in one row
    xt = torch.from_numpy(x).to(src_dtype)
    codes, scale = amun().quantize_e4m3(xt.to(DEV))
    rc, rs = O.quantize_rows_e4m3(xt.float().numpy())
    assert np.array_equal(scale.cpu().numpy().view(np.uint32), rs.view(np.uint32))
    assert np.array_equal(codes.cpu().numpy(), rc)


def run_e4m3(H, V, S, B, k, X=None, W=None, b=None, exact_idx=False, seed=0, dist="zipf"):
    w = synth.Workload("f8", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + 700 + seed, dist=dist)
    X = synth.gen_X(w).float() if X is None else X
    W = synth.gen_W(w).float() if W is None else W
    b = synth.gen_b(w) if b is None else b
    pc, off = synth.gen_prev_cost(w), synth.gen_offsets(w)
    X8, xs = O.quantize_rows_e4m3(X.numpy())
    W8, ws = O.quantize_rows_e4m3(W.numpy())
    ol = amun().OutputLayer(H, V, dtype="e4m3", k_max=k, max_rows=w.N, max_sentences=S)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    idx, cost = ol.call_e4m3(t(X8), t(xs), t(W8), t(ws), b.to(DEV), pc.to(DEV), off.to(DEV), k)
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.dequant_rows_e4m3(X8, xs), O.dequant_rows_e4m3(W8, ws)), O.as_f64(b))
    logp = O.log_softmax(L)
    pcd = O.as_f64(pc)
    oi, oc32, oc64, nxt = O.kbest_sentences(logp, pcd, off.numpy(), k)
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v], oc64,
                  np.full(S, k), "bf16", V, o_next=nxt)
    if exact_idx:
        assert np.array_equal(idx.cpu().numpy(), oi)
    return idx


@pytest.mark.parametrize("H,V,S,B,k", [
    (256, 1009, 37, 5, 5),      # 2 M-tiles, ragged vocab
    (128, 3000, 3, 1, 1),       # greedy-like
    (1040, 20000, 130, 2, 3),   # H not a multiple of 128 (TMA zero-fills K), 3 M-tiles
    (64, 200, 60, 4, 16),       # k = 16 bucket
])
def test_e4m3_shapes(H, V, S, B, k):
    run_e4m3(H, V, S, B, k, seed=H + V)


def test_e4m3_flat_near_ties():
    run_e4m3(256, 20000, 20, 4, 8, dist="flat", seed=11)


def test_e4m3_cfg_shapes_full():
    """cfg greedy and cfg beam shapes end to end in FP8 (W quantised on the GPU)."""
    for name in ("greedy", "beam"):
        w = synth.CONFIGS[name]
        Wf = synth.gen_W(w).float()
        W8, ws = amun().quantize_e4m3(Wf.to(DEV))
        rc, rs = O.quantize_rows_e4m3(Wf.numpy())
        assert np.array_equal(W8.cpu().numpy(), rc)
        run_e4m3(w.H, w.V, w.S, w.B, w.k, X=synth.gen_X(w).float(), W=Wf, b=synth.gen_b(w))


def test_e4m3_integer_regime_exact():
    """Integer codes (|x|, |w| <= 8 are exact in E4M3) and unit scales: exact
    integer logits, so the index sets (ties: lowest id) must match exactly."""
    rng = np.random.default_rng(12)
    N, H, V, S, B, k = 40, 64, 5000, 10, 4, 4
    X = torch.from_numpy(rng.integers(-8, 9, (N, H)).astype(np.float32))
    W = torch.from_numpy(rng.integers(-8, 9, (V, H)).astype(np.float32))
    X[:, 0] = 448.0    # row max 448 -> scale exactly 1
    W[:, 0] = 448.0
    b = torch.from_numpy(rng.integers(-4, 5, V).astype(np.float32))
    run_e4m3(H, V, S, B, k, X=X, W=W, b=b, exact_idx=True)


def test_e4m3_plan_rejects_bf16_entry_points():
    ol = amun().OutputLayer(64, 100, dtype="e4m3", k_max=2, max_rows=4, max_sentences=2)
    X = torch.zeros(4, 64, dtype=torch.uint8, device=DEV)
    W = torch.zeros(100, 64, dtype=torch.uint8, device=DEV)
    with pytest.raises(amun().AmunError if hasattr(amun(), "AmunError") else Exception):
        ol.scores(X, W, torch.zeros(100, device=DEV))


@pytest.mark.parametrize("G", [2, 3])
def test_e4m3_vocab_shard_emulation(G):
    """FP8 vocab shards (amun_output_layer_partial_e4m3 per shard, stacked like
    an all-gather, amun_merge_partials): equal to the oracle on the full
    dequantised vocabulary. W's per-row scales do not depend on the split."""
    w = synth.Workload("f8shard", H=256, V=30000, S=16, B=4, k=6, seed=synth.BASE_SEED + 98)
    X, W, b = synth.gen_X(w).float(), synth.gen_W(w).float(), synth.gen_b(w)
    pc, off = synth.gen_prev_cost(w), synth.gen_offsets(w)
    X8, xs = O.quantize_rows_e4m3(X.numpy())
    W8, ws = O.quantize_rows_e4m3(W.numpy())
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    per = -(-w.V // G)
    per = -(-per // 256) * 256
    bounds = [0]
    while bounds[-1] < w.V:
        bounds.append(min(w.V, bounds[-1] + per))
    parts, plans = [], []
    for g in range(len(bounds) - 1):
        v0, v1 = bounds[g], bounds[g + 1]
        ol = amun().OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, dtype="e4m3", k_max=w.k,
                                max_rows=w.N, max_sentences=w.S)
        plans.append(ol)
        parts.append(ol.partial_e4m3(t(X8), t(xs), t(W8[v0:v1]), t(ws[v0:v1]), b[v0:v1].to(DEV)))
    idx, cost = plans[0].merge(torch.stack(parts), pc.to(DEV), off.to(DEV), w.k)
    torch.cuda.synchronize()
    L = O.add_bias(O.gemm(O.dequant_rows_e4m3(X8, xs), O.dequant_rows_e4m3(W8, ws)), O.as_f64(b))
    logp = O.log_softmax(L)
    pcd = O.as_f64(pc)
    oi, _, oc64, nxt = O.kbest_sentences(logp, pcd, off.numpy(), w.k)
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                  oc64, np.full(w.S, w.k), "bf16", w.V, o_next=nxt)


def test_e4m3_argmax():
    """FP8 greedy argmax (Alg. 5) vs oracle.argmax_1best on the dequantised
    logits: exact in the integer regime (unit scales, lowest id on ties);
    otherwise within the fp32 accumulation band (reading G16)."""
    rng = np.random.default_rng(21)
    N, H, V = 130, 64, 20000
    X = rng.integers(-3, 4, (N, H)).astype(np.float32)
    W = rng.integers(-3, 4, (V, H)).astype(np.float32)
    X[:, 0] = 448.0
    W[:, 0] = 448.0
    b = rng.integers(-2, 3, V).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    for Xf, Wf, exact in [(X, W, True),
                          (synth.gen_X(synth.CONFIGS["greedy"]).float().numpy()[:N, :H],
                           synth.gen_W(synth.CONFIGS["greedy"]).float().numpy()[:V, :H], False)]:
        N = Xf.shape[0]
        X8, xs = O.quantize_rows_e4m3(Xf)
        W8, ws = O.quantize_rows_e4m3(Wf)
        ol = amun().OutputLayer(H, V, dtype="e4m3", k_max=1, max_rows=N, max_sentences=1)
        tok, logit = ol.argmax_e4m3(t(X8), t(xs), t(W8), t(ws), t(b))
        torch.cuda.synchronize()
        P = O.gemm(O.dequant_rows_e4m3(X8, xs), O.dequant_rows_e4m3(W8, ws))
        L = O.add_bias(P, O.as_f64(b))
        ref = np.array([O.argmax_1best(P[r], O.as_f64(b)) for r in range(N)])
        tok, logit = tok.cpu().numpy(), logit.cpu().numpy()
        rows = np.arange(N)
        if exact:
            assert np.array_equal(tok, ref)
            assert np.array_equal(logit.astype(np.float64), L[rows, ref])
        else:
            band = H * 2.0 ** -24 * (np.abs(O.dequant_rows_e4m3(X8, xs)) @
                                     np.abs(O.dequant_rows_e4m3(W8, ws)).T).max(axis=1) \
                + np.abs(L).max(axis=1) * 2.0 ** -22
            assert (L[rows, ref] - L[rows, tok] <= 2 * band).all()
            assert (tok == ref).mean() > 0.99
