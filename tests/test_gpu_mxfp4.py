"""Block-scaled 4-bit W (NEXT f4; amun_*_mxfp4, amun_quantize_mxfp4) against
the oracle: the GPU quantiser bit-exact against oracle.quantize_rows_mxfp4
(codes and E8M0 scales, unpacked from the device layouts amun.h defines),
the raw logits of the kind::mxf8f6f4.block_scale GEMM exact in an integer
regime, and the k-best / argmax of the full path against the oracle run on
the exactly dequantised values (oracle.dequant_rows_mxfp4 x
dequant_rows_e4m3), with the bf16 comparator (exact products, fp32
accumulation, as the e4m3 path)."""
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


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


# --------------------------------------------------- device layouts (amun.h)
def sf_offsets(R, H):
    """Byte offset of the E8M0 code of (row r, block j) in the atom layout."""
    r = np.arange(R)[:, None]
    j = np.arange(H // 32)[None, :]
    return ((j // 4) * (-(-R // 128)) + r // 128) * 512 + 16 * (r % 32) + 4 * ((r % 128) // 32) + j % 4


def to_device(codes, sexp):
    """Oracle (unpacked codes, E8M0 codes) -> (W4 [R, H/2], sf bytes)."""
    R, H = codes.shape
    packed = ((codes[:, 0::2] & 0xF) | ((codes[:, 1::2] & 0xF) << 4)).astype(np.uint8)
    sf = np.full(-(-R // 128) * (H // 128) * 512, 127, np.uint8)
    sf[sf_offsets(R, H)] = sexp
    return packed, sf


def from_device(W4, sf, R, H):
    W4 = W4.cpu().numpy()
    codes = np.empty((R, H), np.uint8)
    codes[:, 0::2] = W4 & 0xF
    codes[:, 1::2] = W4 >> 4
    return codes, sf.cpu().numpy()[sf_offsets(R, H)]


def test_layout_helpers_round_trip():
    rng = np.random.default_rng(1)
    codes = rng.integers(0, 16, (300, 256)).astype(np.uint8)
    sexp = rng.integers(0, 255, (300, 8)).astype(np.uint8)
    W4, sf = to_device(codes, sexp)
    assert len(sf) == amun().mxfp4_sf_bytes(300, 256)
    c2, s2 = from_device(torch.from_numpy(W4), torch.from_numpy(sf), 300, 256)
    assert np.array_equal(c2, codes) and np.array_equal(s2, sexp)


@pytest.mark.parametrize("src_dtype", [torch.float32, torch.bfloat16])
def test_quantize_bit_exact(src_dtype):
    rng = np.random.default_rng(4)
    R, H = 300, 1024
    x = (rng.normal(size=(R, H)) * np.exp(rng.normal(size=(R, 1)) * 4)).astype(np.float32)
    x[7] = 0.0                                        # all-zero blocks -> code 127
    x[8, ::3] = 0.0
    x[9, 5] = 1e30                                    # huge value: its block saturates the rest to 0
    x[10, 32:64] = -1e-3                              # small negatives beside a large value -> -0
    x[10, 40] = 5.0
    x[11, :32] = 0.75                                 # exact ties (0.75 / 2^-2 = 3: on the grid)
    x[12, :32] = np.float32(5.0)                      # tie 4 | 6 -> 4
    xt = torch.from_numpy(x).to(src_dtype)
    W4, sf = amun().quantize_mxfp4(xt.to(DEV))
    torch.cuda.synchronize()
    rc, rs = O.quantize_rows_mxfp4(xt.float().numpy())
    gc, gs = from_device(W4, sf, R, H)
    assert np.array_equal(gs, rs)
    assert np.array_equal(gc, rc)
    # the padding rows of the last 128-row atom carry code 127
    pad = np.setdiff1d(np.arange(len(sf)), sf_offsets(R, H).ravel())
    assert (sf.cpu().numpy()[pad] == 127).all()


def oracle_logits(X8, xs, codes, sexp, b):
    return O.add_bias(O.gemm(O.dequant_rows_e4m3(X8, xs), O.dequant_rows_mxfp4(codes, sexp)),
                      O.as_f64(b))


@pytest.mark.parametrize("N,V", [
    (200, 1000),     # 2 M-tiles (ragged), V not a multiple of 128
    (128, 94720),    # one M-tile: CTA ranges of 640 = tiles 256 | 128 | 256
    (300, 5000),     # 3 M-tiles, flattened schedule, ranges across M-tiles
])
def test_logits_integer_regime_exact(N, V):
    """Integer E4M3 X (x_scale exactly 1) and W on the E2M1 grid with block
    exponents in [-2, 2]: every product and partial sum is a small multiple of
    1/8, exact in fp32, so the biased logits equal the oracle's bit for bit.
    Pins the nibble order, the scale-atom layout, the sf ids and both tile
    widths (256 in accumulator 0, 128 in accumulator 1)."""
    rng = np.random.default_rng(12)
    H = 256
    X = rng.integers(-8, 9, (N, H)).astype(np.float32)
    X[:, 0] = 448.0
    X8, xs = O.quantize_rows_e4m3(X)
    assert (xs == 1.0).all()
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    Wv = rng.choice(grid, (V, H)) * rng.choice([-1.0, 1.0], (V, H))
    Wv = Wv * np.repeat(2.0 ** rng.integers(-2, 3, (V, H // 32)), 32, axis=1)
    codes, sexp = O.quantize_rows_mxfp4(Wv.astype(np.float32))
    assert np.array_equal(O.dequant_rows_mxfp4(codes, sexp), Wv)   # W on the grid: exact
    b = rng.integers(-4, 5, V).astype(np.float32)
    W4, sf = to_device(codes, sexp)
    ol = amun().OutputLayer(H, V, dtype="mxfp4", k_max=4, max_rows=N, max_sentences=N)
    L = ol.debug_logits_mxfp4(t(X8), t(xs), t(W4), t(sf), t(b))
    torch.cuda.synchronize()
    want = oracle_logits(X8, xs, codes, sexp, b)
    assert np.array_equal(L.cpu().numpy().astype(np.float64), want)


def run_mxfp4(H, V, S, B, k, X=None, W=None, b=None, seed=0, dist="zipf", gpu_quant=False):
    w = synth.Workload("f4", H=H, V=V, S=S, B=B, k=k, seed=synth.BASE_SEED + 900 + seed, dist=dist)
    X = synth.gen_X(w).float() if X is None else X
    W = synth.gen_W(w).float() if W is None else W
    b = synth.gen_b(w) if b is None else b
    pc, off = synth.gen_prev_cost(w), synth.gen_offsets(w)
    X8, xs = O.quantize_rows_e4m3(X.numpy())
    codes, sexp = O.quantize_rows_mxfp4(W.numpy())
    if gpu_quant:   # the GPU quantiser's output, checked equal to the oracle's first
        W4d, sfd = amun().quantize_mxfp4(W.to(DEV))
        gc, gs = from_device(W4d, sfd, V, H)
        assert np.array_equal(gc, codes) and np.array_equal(gs, sexp)
    else:
        W4, sf = to_device(codes, sexp)
        W4d, sfd = t(W4), t(sf)
    ol = amun().OutputLayer(H, V, dtype="mxfp4", k_max=k, max_rows=w.N, max_sentences=S)
    idx, cost = ol.call_mxfp4(t(X8), t(xs), W4d, sfd, b.to(DEV), pc.to(DEV), off.to(DEV), k)
    torch.cuda.synchronize()
    L = oracle_logits(X8, xs, codes, sexp, b)
    logp = O.log_softmax(L)
    pcd = O.as_f64(pc)
    oi, oc32, oc64, nxt = O.kbest_sentences(logp, pcd, off.numpy(), k)
    compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v], oc64,
                  np.full(S, k), "bf16", V, o_next=nxt)
    return ol, (X8, xs, W4d, sfd, b, L)


@pytest.mark.parametrize("H,V,S,B,k", [
    (256, 1009, 37, 5, 5),      # 2 M-tiles, ragged vocab (tail tile of 113 columns)
    (128, 3000, 3, 1, 1),       # greedy-like, one K block
    (1024, 20000, 130, 2, 3),   # 3 M-tiles
    (384, 200, 60, 4, 16),      # k = 16 bucket, vocab smaller than one CTA range
])
def test_mxfp4_shapes(H, V, S, B, k):
    run_mxfp4(H, V, S, B, k, seed=H + V)


def test_mxfp4_flat_near_ties():
    run_mxfp4(256, 20000, 20, 4, 8, dist="flat", seed=11)


def test_mxfp4_argmax():
    """Alg. 5 on the MXFP4 GEMM: the token is the oracle's argmax unless the
    top two oracle logits are within the fp32 band; the logit within it."""
    ol, (X8, xs, W4d, sfd, b, L) = run_mxfp4(512, 30000, 100, 1, 1, seed=5)
    tok, logit = ol.argmax_mxfp4(t(X8), t(xs), W4d, sfd, b.to(DEV))
    torch.cuda.synchronize()
    tok, logit = tok.cpu().numpy(), logit.cpu().numpy()
    top2 = np.sort(L, axis=1)[:, -2:]
    band = 1e-4 * np.maximum(1.0, np.abs(top2[:, 1]))
    clear = top2[:, 1] - top2[:, 0] > band
    assert np.array_equal(tok[clear], L.argmax(axis=1)[clear])
    assert np.allclose(logit, L[np.arange(len(tok)), tok], rtol=1e-5, atol=1e-4)


@pytest.mark.slow
def test_mxfp4_cfg_shapes_full():
    """cfg greedy and cfg beam shapes end to end with W quantised on the GPU
    (bit-exact against the oracle quantiser over all of W)."""
    for name in ("greedy", "beam"):
        w = synth.CONFIGS[name]
        run_mxfp4(w.H, w.V, w.S, w.B, w.k, X=synth.gen_X(w).float(), W=synth.gen_W(w).float(),
                  b=synth.gen_b(w), gpu_quant=True)


def test_mxfp4_entry_point_checks():
    A = amun()
    ol = A.OutputLayer(256, 100, dtype="mxfp4", k_max=2, max_rows=4, max_sentences=2)
    X8 = torch.zeros(4, 256, dtype=torch.uint8, device=DEV)
    W = torch.zeros(100, 256, dtype=torch.uint8, device=DEV)
    with pytest.raises(A.AmunError):                  # bf16 entry points refuse scaled plans
        ol.scores(X8, W, torch.zeros(100, device=DEV))
    with pytest.raises(A.AmunError):                  # H % 128 != 0
        A.OutputLayer(192, 100, dtype="mxfp4", k_max=2, max_rows=4, max_sentences=2)
    bf = A.OutputLayer(256, 100, dtype="bf16", k_max=2, max_rows=4, max_sentences=2)
    W4 = torch.zeros(100, 128, dtype=torch.uint8, device=DEV)
    sf = torch.zeros(A.mxfp4_sf_bytes(100, 256), dtype=torch.uint8, device=DEV)
    with pytest.raises(A.AmunError):                  # an mxfp4 call on a bf16 plan
        bf.argmax_mxfp4(X8, torch.ones(4, device=DEV), W4, sf, torch.zeros(100, device=DEV))
