"""Pins for the CPU oracle (oracle/). Each test fixes a function by something
other than the function itself: values printed in the paper or its SPEC,
closed forms, brute force on tiny inputs, exact integer arithmetic, library
routines, and invariants. A plausible mistake (dropped bias, wrong sign,
transposed operand, wrong tie rule, wrong rescale) fails at least one.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ GEX1
def test_gex1_closed_form_and_oracle():
    g = _load("gex1.json")
    X = np.array(g["X"], float)
    W = np.array(g["W"], float)
    b = np.array(g["b"], float)
    L = O.add_bias(O.gemm(X, W), b)
    assert np.array_equal(L, np.array(g["logits"], float))          # exact integers
    # closed-form lse, recomputed with the math module
    lse = [math.log(sum(math.exp(x) for x in row)) for row in g["logits"]]
    assert np.allclose(lse, g["lse"], atol=1e-9)
    for case in g["cases"]:
        k = case["k"]
        # the stored costs must equal the closed form prev + l - lse
        for i, c in zip(case["idx"], case["cost"]):
            r, v = divmod(i, g["V"])
            cf = g["prev_cost"][r] + g["logits"][r][v] - lse[r]
            assert abs(cf - c) < 1e-9
        idx, c32, c64, nxt = O.output_layer(X, W, b, g["prev_cost"], [0, 2], k)
        assert idx[0].tolist() == case["idx"]                       # incl. exact-tie order
        assert np.allclose(c64[0], case["cost"], atol=1e-9)


def test_gex1_shards_and_greedy():
    g = _load("gex1.json")
    L = np.array(g["logits"], float)
    p0 = O.shard_partial(L[:, 0:2], 2, v_offset=0)
    p1 = O.shard_partial(L[:, 2:4], 2, v_offset=2)
    for r, key in enumerate(["row0", "row1"]):
        for p, exp in zip([p0, p1], g["shards_2"][key]):
            assert p[0][r] == exp[0]
            assert abs(p[1][r] - exp[1]) < 1e-9
            assert p[3][r].tolist() == exp[2]
    M, S, l, v = O.combine_partials([p0, p1], 2)
    assert np.allclose(M + np.log(S), g["lse"], atol=1e-9)
    gr = g["greedy"]
    W = np.array(g["W"], float)
    Lg = O.add_bias(O.gemm(np.array([gr["x"]]), W), g["b"])
    assert np.allclose(Lg[0], gr["logits"])
    idx, _, c64, _ = O.output_layer(np.array([gr["x"]]), W, g["b"], [0.0], [0, 1], 1)
    assert idx[0, 0] == gr["idx"] and abs(c64[0, 0] - gr["cost"]) < 1e-9


# ------------------------------------------------------------------ SPEC examples
def _val(x):
    return math.log(3) if x == "ln3" else float(x)


def test_spec_softmax_examples():
    ex = _load("spec_examples.json")
    for e in ex["softmax_3pass"]:
        p = np.array([[_val(x) for x in e["p"]]])
        probs = np.exp(O.log_softmax(p))[0]
        assert np.allclose(probs, e["probs"], atol=1e-12), e["line"]
        assert np.isfinite(probs).all()


def test_spec_find_best_and_argmax():
    ex = _load("spec_examples.json")
    for e in ex["find_best"]:
        mx, best = O.find_best(e["p"])
        assert best == e["best"] and mx == e["max"], e["line"]
    for e in ex["argmax_1best"]:
        assert O.argmax_1best(e["p"], e["b"]) == e["best"], e["line"]
    for e in ex["argmax_1best_parallel"]:
        assert O.argmax_1best_parallel(e["p"], e["b"], e["shards"]) == e["best"], e["line"]


def test_spec_output_examples():
    ex = _load("spec_examples.json")
    for e in ex["baseline_output"] + ex["fused_output"]:
        p = np.array([e["p"]], float)
        idx, _, c64, _ = O.kbest_sentences(O.log_softmax(O.add_bias(p, e["b"])), [0.0], [0, 1], e["k"])
        assert idx[0].tolist() == e["idx"], e["line"]
        if "prob" in e:
            assert np.allclose(np.exp(c64[0]), e["prob"], atol=e["tol"]), e["line"]
    for e in ex["fused_output"]:
        inv_sum, best, _, _ = O.online_stats(e["p"], e["b"])
        assert best == e["idx"][0] and abs(inv_sum - e["prob"][0]) < e["tol"], e["line"]


def test_spec_expand_beam():
    e = _load("spec_examples.json")["expand_beam"][0]
    logp = np.array(e["slot_costs"])
    idx, _, c64, _ = O.kbest_sentences(logp, [0.0, 0.0], [0, 2], 2)
    assert sorted(c64[0].tolist(), reverse=True) == e["keep"]
    assert idx[0].tolist() == [0, 2]                     # (r0, v0), (r1, v0)


def test_beam_advance_spec_and_hand_example():
    """SPEC S:331 (beam 2 keeps {-1.0, -1.5}) and S:332 (an EOS winner
    finishes its hypothesis and frees its slot), then a hand-worked batch:
    EOS in the middle, padding, and one parent chosen twice."""
    V, eos = 10, 2
    cols = [np.arange(4 * 8, dtype=np.uint8).reshape(4, 8)]
    # winners (slot0, v0) -1.0 and (slot1, v0) -1.5 -> both continue
    out = O.beam_advance([[0 * V + 0, 1 * V + 0]], [[-1.0, -1.5]], V, eos, cols)
    ncols, off, src, tok, cost, n, s_alive, fin = out
    assert src.tolist() == [0, 1] and tok.tolist() == [0, 0] and cost.tolist() == [-1.0, -1.5]
    assert off.tolist() == [0, 2] and n == 2 and s_alive == 1 and fin == []
    # the best candidate is EOS at beam 1 -> the sentence finishes
    out = O.beam_advance([[0 * V + eos]], [[-0.5]], V, eos, cols)
    assert out[5] == 0 and out[6] == 0 and out[1].tolist() == [0, 0]
    assert out[7] == [(0, 0, 0, eos, -0.5)]
    # hand example: 3 sentences, k = 3
    idx = [[1 * V + 7, 0 * V + eos, 1 * V + 3],     # s0 rows 0-1: (1,7), EOS, (1,3): parent 1 twice
           [-1, -1, -1],                             # s1: no candidates
           [3 * V + 5, 2 * V + eos, -1]]             # s2 rows 2-3: (3,5), EOS, pad
    cst = [[-1.0, -2.0, -3.0], [-np.inf] * 3, [-0.5, -0.7, -np.inf]]
    ncols, off, src, tok, cost, n, s_alive, fin = O.beam_advance(idx, cst, V, eos, cols)
    assert src.tolist() == [1, 1, 3] and tok.tolist() == [7, 3, 5]
    assert cost.tolist() == [-1.0, -3.0, -0.5]
    assert off.tolist() == [0, 2, 2, 3] and n == 3 and s_alive == 2
    assert [f[:4] for f in fin] == [(0, 1, 0, eos), (2, 1, 2, eos)]
    assert np.array_equal(ncols[0], cols[0][[1, 1, 3]])


def test_beam_advance_reduces_to_compact():
    """Invariant tying the two Alg. 2 oracles together: when sentence s's i-th
    winner continues its own slot (parent = o_s + i), advancing the beam is
    exactly the stable compaction by the non-EOS mask (compact is pinned by
    SPEC S:339-341 independently)."""
    rng = np.random.default_rng(3)
    V, eos, S, k = 50, 7, 40, 4
    N = S * k
    tok = rng.integers(0, V, N)
    tok[rng.random(N) < 0.3] = eos
    idx = (np.arange(N) * V + tok).reshape(S, k)
    cst = rng.normal(size=(S, k)).astype(np.float32)
    cols = [rng.integers(0, 256, (N, 24), dtype=np.uint8)]
    ncols, off, src, t2, c2, n, s_alive, fin = O.beam_advance(idx, cst, V, eos, cols)
    alive = (tok != eos).astype(np.uint8)
    ccols, coff, csrc, cn, cs_alive = O.compact(cols, alive, np.arange(S + 1) * k)
    assert np.array_equal(ncols[0], ccols[0]) and np.array_equal(src, csrc)
    assert np.array_equal(off, coff) and n == cn and s_alive == cs_alive
    assert np.array_equal(t2, tok[alive == 1]) and np.array_equal(c2, cst.reshape(-1)[alive == 1])
    assert len(fin) == N - n


def test_spec_compact_examples():
    for e in _load("spec_examples.json")["compact_states"]:
        rows = np.array([[ord(c)] * 16 for c in e["rows"]], np.uint8)
        cols, off, src, n, s_alive = O.compact([rows], e["alive"], [0, 3])
        assert [chr(r[0]) for r in cols[0]] == e["out"], e["line"]
        assert src.tolist() == e["src_row"]
        assert n == len(e["out"]) and off.tolist() == [0, n]
        assert s_alive == (1 if n else 0)


def test_spec_decode_work():
    for e in _load("spec_examples.json")["decode_work"]:
        assert O.decode_work(e["finish"], e["beam"], "naive") == e["naive"], e["line"]
        assert O.decode_work(e["finish"], e["beam"], "dynamic") == e["dynamic"], e["line"]


# ------------------------------------------------------------------ brute force
def _brute_kbest(L, prev, offsets, k):
    """Independent O(n^2) route: probabilities from the textbook definition
    exp(l)/sum(exp(l)) with math.fsum (no max shift; inputs are small), and
    ranks by COUNTING strictly better candidates instead of sorting."""
    out = []
    for s in range(len(offsets) - 1):
        cands = []
        for r in range(offsets[s], offsets[s + 1]):
            z = math.fsum(math.exp(x) for x in L[r])
            for v, x in enumerate(L[r]):
                cands.append((prev[r] + math.log(math.exp(x) / z), r, v))

        def better(a, b):  # a ranks before b
            return a[0] > b[0] or (a[0] == b[0] and (a[1], a[2]) < (b[1], b[2]))

        ranked = [None] * len(cands)
        for a in cands:
            rank = sum(1 for b in cands if better(b, a))
            ranked[rank] = a
        out.append(ranked[:k])
    return out


@pytest.mark.parametrize("seed", range(12))
def test_kbest_brute_force_tiny(seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(1, 9))
    Bs = [int(x) for x in rng.integers(0, 4, size=3)]     # includes empty sentences
    off = np.concatenate([[0], np.cumsum(Bs)]).astype(int)
    N = int(off[-1])
    H = 8
    X = rng.standard_normal((N, H))
    W = rng.standard_normal((V, H))
    b = rng.standard_normal(V)
    prev = -rng.uniform(0, 5, N)
    L = O.add_bias(O.gemm(X, W), b)
    kmax = max(1, max(Bs) * V)
    for k in sorted({1, 2, 3, kmax}):
        idx, c32, c64, nxt = O.kbest_sentences(O.log_softmax(L), prev, off, k)
        ref = _brute_kbest(L.tolist(), prev.tolist(), off.tolist(), k)
        for s in range(len(Bs)):
            got = [(int(i) // V, int(i) % V) for i in idx[s] if i >= 0]
            exp = [(r, v) for _, r, v in ref[s]]
            assert got == exp
            n = len(exp)
            assert np.allclose(c64[s, :n], [c for c, _, _ in ref[s]], atol=1e-12)
            assert (idx[s, n:] == -1).all() and np.isneginf(c64[s, n:]).all()


def test_k_equals_all_candidates_sum_to_one():
    rng = np.random.default_rng(5)
    L = rng.standard_normal((3, 5)) * 3
    prev = np.array([-1.0, -2.0, -0.5])
    idx, c32, c64, nxt = O.kbest_sentences(O.log_softmax(L), prev, [0, 3], 15)
    assert sorted(idx[0].tolist()) == list(range(15))
    rows = idx[0] // 5
    tot = sum(math.exp(c - prev[r]) for c, r in zip(c64[0], rows))
    assert abs(tot - 3.0) < 1e-12                       # each row's probs sum to 1
    assert np.isneginf(nxt[0])


# ------------------------------------------------------------------ invariants
def test_softmax_sums_to_one_and_shift_invariance():
    rng = np.random.default_rng(1)
    L = rng.standard_normal((7, 5000)) * 4
    lp = O.log_softmax(L)
    assert np.allclose(np.exp(lp).sum(axis=1), 1.0, atol=1e-12)
    lp2 = O.log_softmax(L + 123.25)
    assert np.allclose(lp, lp2, atol=1e-11)
    big = O.log_softmax(np.full((1, 4), 1000.0))
    assert np.allclose(big, -math.log(4))
    uni = O.log_softmax(np.zeros((1, 90000)))
    assert abs(uni[0, 0] + 11.407564949312402) < 1e-12   # -ln(90000)


def test_bias_shift_keeps_indices_and_prev_cost_shift():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((6, 16)); W = rng.standard_normal((50, 16)); b = rng.standard_normal(50)
    prev = -rng.uniform(0, 3, 6); off = [0, 3, 6]
    a = O.output_layer(X, W, b, prev, off, 4)
    c = O.output_layer(X, W, b + 7.5, prev, off, 4)
    assert np.array_equal(a[0], c[0]) and np.allclose(a[2], c[2], atol=1e-12)
    d = O.output_layer(X, W, b, prev + 2.0, off, 4)
    assert np.array_equal(a[0], d[0]) and np.allclose(a[2] + 2.0, d[2], atol=1e-12)


def test_log_softmax_vs_torch():
    rng = np.random.default_rng(3)
    L = rng.standard_normal((4, 3000)) * 5
    ref = torch.log_softmax(torch.from_numpy(L), dim=1).numpy()
    assert np.allclose(O.log_softmax(L), ref, atol=1e-12)


def test_greedy_is_argmax():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((9, 32)); W = rng.standard_normal((700, 32)); b = rng.standard_normal(700)
    off = np.arange(10)
    idx, _, c64, _ = O.output_layer(X, W, b, np.zeros(9), off, 1)
    L = X @ W.T + b
    assert (idx[:, 0] == np.arange(9) * 700 + np.argmax(L, axis=1)).all()
    ref = -np.log(np.exp(L - L.max(axis=1, keepdims=True)).sum(axis=1))
    assert np.allclose(c64[:, 0], ref, atol=1e-12)
    for r in range(9):  # Alg. 5 == Alg. 4 agreement
        assert O.argmax_1best(L[r] - b, b) == idx[r, 0] - 700 * r


def test_gemm_integer_regime_exact():
    rng = np.random.default_rng(6)
    X = rng.integers(-8, 9, (5, 40)); W = rng.integers(-8, 9, (13, 40))
    L = O.gemm(X.astype(float), W.astype(float))
    ref = [[sum(int(a) * int(c) for a, c in zip(X[r], W[v])) for v in range(13)] for r in range(5)]
    assert np.array_equal(L, np.array(ref, float))
    assert not np.array_equal(L, O.gemm(X.astype(float), W[::-1].astype(float)))


def test_unit_vector_rows_pick_columns():
    rng = np.random.default_rng(7)
    W = rng.standard_normal((30, 8)); b = rng.standard_normal(30)
    X = np.eye(8)[[3, 0, 7]]
    L = O.add_bias(O.gemm(X, W), b)
    assert np.array_equal(L, (W[:, [3, 0, 7]] + b[:, None]).T)


def test_bf16_widening_exact():
    t = torch.tensor([1.0, 0.1, -3.3, 1e-3]).to(torch.bfloat16)
    a = O.as_f64(t)
    bits = t.view(torch.int16).numpy().astype(np.int64) & 0xFFFF
    ref = (bits << 16).astype(np.uint32).view(np.float32).astype(np.float64)
    assert np.array_equal(a, ref)


# ------------------------------------------------------------------ partial-state monoid
@pytest.mark.parametrize("G", [1, 2, 3, 7, 64])
def test_partials_any_split(G):
    rng = np.random.default_rng(10 + G)
    L = rng.standard_normal((4, 640)) * 3
    L[1, 5] = L[1, 600] = L[1].max() + 1.0            # duplicated maxima across shards
    L[2, :] = 0.25                                      # all-equal row
    full = O.shard_partial(L, 5)
    cuts = np.linspace(0, 640, G + 1).round().astype(int)
    parts = [O.shard_partial(L[:, a:c], 5, v_offset=a) for a, c in zip(cuts[:-1], cuts[1:])]
    M, S, l, v = O.combine_partials(parts, 5)
    assert np.array_equal(M, full[0])
    assert np.allclose(S, full[1], rtol=1e-12)
    assert np.array_equal(v, full[3]) and np.array_equal(l, full[2])
    assert v[2].tolist() == [0, 1, 2, 3, 4]             # ties -> lower v
    assert v[1, :2].tolist() == [5, 600]


def test_online_stats_matches_3pass_under_permutation():
    rng = np.random.default_rng(11)
    p = rng.standard_normal(1000) * 4
    m, z = O.softmax_3pass_stats(p[None, :])
    for t in range(100):
        q = rng.permutation(p)
        inv, best, mx, sm = O.online_stats(q)
        assert mx == m[0] and abs(sm - z[0]) <= 1e-12 * z[0]
        assert q[best] == mx
    # the literal "Delta x sum" of P:176 would NOT reproduce the sum (reading G1)
    mx, sm = -np.inf, 0.0
    for x in p[:50]:
        if x > mx:
            sm, mx = (mx - x) * sm + 1.0 if np.isfinite(mx) else 1.0, x
        else:
            sm += math.exp(x - mx)
    assert abs(sm - O.softmax_3pass_stats(p[None, :50])[1][0]) > 1e-3


def test_argmax_parallel_shard_invariance():
    rng = np.random.default_rng(12)
    for t in range(200):
        p = rng.integers(0, 20, 300).astype(float)       # many duplicated maxima
        b = np.zeros(300)
        ref = O.argmax_1best(p, b)
        assert ref == int(np.argmax(p))
        for sh in [1, 2, 3, 7, 64]:
            assert O.argmax_1best_parallel(p, b, sh) == ref


# ------------------------------------------------------------------ compaction
@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.9, 1.0])
def test_compact_random(p):
    rng = np.random.default_rng(int(p * 10))
    N, S = 40, 9
    off = np.sort(np.concatenate([[0, N], rng.integers(0, N, S - 1)]))
    alive = (rng.random(N) < p).astype(np.uint8)
    c1 = rng.integers(0, 256, (N, 32), dtype=np.uint8)
    c2 = rng.integers(0, 256, (N, 4), dtype=np.uint8)
    cols, no, src, n, s_alive = O.compact([c1, c2], alive, off)
    keep = [r for r in range(N) if alive[r]]                       # list comprehension pin
    assert src.tolist() == keep and n == len(keep)
    assert np.array_equal(cols[0], c1[keep]) and np.array_equal(cols[1], c2[keep])
    assert no.tolist() == [sum(1 for r in keep if r < o) for o in off]
    assert s_alive == sum(1 for s in range(S) if any(alive[off[s]:off[s + 1]]))
    # idempotent under re-compaction with all-ones
    cols2, no2, src2, n2, _ = O.compact(cols, np.ones(n, np.uint8), no)
    assert np.array_equal(cols2[0], cols[0]) and src2.tolist() == list(range(n))
    assert no2.tolist() == no.tolist()


# ------------------------------------------------------------------ FP8 (f4)
def test_e4m3_decode_definition_points():
    """Values fixed by the OCP E4M3 definition: 1.0 = 0x38, max 448 = 0x7E,
    min normal 2^-6 = 0x08, min subnormal 2^-9 = 0x01, -0 = 0x80, NaN = 0x7F."""
    d = O.e4m3_decode(np.array([0x38, 0x7E, 0x08, 0x01, 0x80, 0x00, 0xFE, 0x3C, 0x07], np.uint8))
    assert d[:4].tolist() == [1.0, 448.0, 2.0 ** -6, 2.0 ** -9]
    assert d[4] == 0.0 and np.signbit(d[4]) and d[5] == 0.0
    assert d[6] == -448.0 and d[7] == 1.5 and d[8] == 7 / 8 * 2.0 ** -6
    assert np.isnan(O.e4m3_decode(np.array([0x7F, 0xFF], np.uint8))).all()


def test_e4m3_decode_matches_library_all_codes():
    import torch
    codes = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], np.uint8)
    lib = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    assert np.array_equal(O.e4m3_decode(codes), lib)


def test_quantize_rows_e4m3_is_nearest_by_brute_force():
    """Every code is the nearest of all 254 finite E4M3 values to x / scale
    (ties: even mantissa), the row scale maps the row max to 448 exactly,
    and representable inputs round-trip exactly."""
    rng = np.random.default_rng(8)
    x = (rng.normal(size=(6, 200)) * np.exp(rng.normal(size=(6, 1)) * 3)).astype(np.float32)
    x[5] = 0.0
    codes, scale = O.quantize_rows_e4m3(x)
    finite = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], np.uint8)
    vals = O.e4m3_decode(finite)
    y = (x / scale[:, None]).astype(np.float32).astype(np.float64)
    got = O.e4m3_decode(codes)
    for r in range(x.shape[0]):
        for h in range(x.shape[1]):
            dist = np.abs(vals - y[r, h])
            best = dist.min()
            assert abs(got[r, h] - y[r, h]) == best
            cands = finite[dist == best]
            if len(set(O.e4m3_decode(cands).tolist())) > 1:      # a true tie: even mantissa
                assert codes[r, h] & 1 == 0
    assert scale[5] == 1.0 and (codes[5] == 0).all()
    assert np.allclose(np.abs(O.dequant_rows_e4m3(codes, scale)[:5]).max(axis=1),
                       np.abs(x[:5]).max(axis=1), rtol=1e-6)
    rep = O.e4m3_decode(np.array([[0x38, 0x30, 0x7E, 0x01]], np.uint8)).astype(np.float32)
    c2, s2 = O.quantize_rows_e4m3(rep)
    assert np.array_equal(O.dequant_rows_e4m3(c2, s2), rep.astype(np.float64))


# ---------------------------------------------------------------- MXFP4 (f4)
def test_e2m1_decode_is_the_ocp_table():
    """The OCP MX v1.0 E2M1 table: codes 0-7 = 0, 0.5, 1, 1.5, 2, 3, 4, 6;
    codes 8-15 the same negated (8 = -0)."""
    d = O.e2m1_decode(np.arange(16, dtype=np.uint8))
    table = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]
    assert d[:8].tolist() == table
    assert d[8:].tolist() == [-t for t in table]
    assert np.signbit(d[8])
    # only the low nibble is a code
    assert O.e2m1_decode(np.array([0x37, 0xF9], np.uint8)).tolist() == [6.0, -0.5]


def test_quantize_rows_mxfp4_is_nearest_by_brute_force():
    """Per block: the scale puts the block max in [4, 8) x 2^e (the MX rule
    e = floor(log2 amax) - 2); every code is the nearest of the 15 distinct
    E2M1 values times 2^e to x (magnitudes above 6 x 2^e clamp to 6 x 2^e),
    ties to the even code; an all-zero block has scale code 127."""
    rng = np.random.default_rng(21)
    x = (rng.normal(size=(5, 128)) * np.exp(rng.normal(size=(5, 1)) * 2)).astype(np.float32)
    x[4, :32] = 0.0
    x[3, 32:64] = np.float32(-1e-3)          # small negatives beside a large value round to -0
    x[3, 40] = np.float32(5.0)
    codes, sexp = O.quantize_rows_mxfp4(x)
    assert codes.shape == x.shape and sexp.shape == (5, 4)
    assert sexp[4, 0] == 127 and (codes[4, :32] & 0x7 == 0).all()
    assert (np.delete(codes[3, 32:64], 8) == 0x8).all()
    mags = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    for r in range(5):
        for blk in range(4):
            v = x[r, 32 * blk:32 * blk + 32].astype(np.float64)
            amax = np.abs(v).max()
            if amax == 0:
                continue
            X = 2.0 ** (int(sexp[r, blk]) - 127)
            assert 4.0 <= amax / X < 8.0
            for j in range(32):
                a = min(abs(v[j]) / X, 6.0)
                c = int(codes[r, 32 * blk + j])
                dist = np.abs(mags - a)
                assert abs(mags[c & 7] - a) == dist.min()
                if (dist == dist.min()).sum() > 1:   # a true tie: even code
                    assert (c & 7) % 2 == 0
                assert bool(c & 8) == bool(np.signbit(v[j]))
    deq = O.dequant_rows_mxfp4(codes, sexp)
    # error bound: half the E2M1 spacing at the value (0.25 below 2, 0.5 below
    # 4, 1 up to 6) times 2^e; above 6 x 2^e the clamp
    X = np.repeat(2.0 ** (sexp.astype(np.float64) - 127), 32, axis=1)
    q = np.abs(x.astype(np.float64)) / X
    half = np.where(q < 2, 0.25, np.where(q < 4, 0.5, 1.0))
    err = np.abs(deq - x) / X
    assert (err <= np.maximum(half, q - 6.0) + 1e-12).all()


def test_quantize_rows_mxfp4_round_trip_and_special_blocks():
    """Values on the E2M1 grid whose block max is 4 or 6 x 2^e round-trip
    exactly; a constant block maps its value to code 6 (4 x 2^e) or 7."""
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    rng = np.random.default_rng(3)
    rows = []
    for e in (-9, -1, 0, 3):
        v = rng.choice(grid, size=32) * rng.choice([-1.0, 1.0], size=32)
        v[5] = 6.0
        rows.append(v * 2.0 ** e)
    x = np.concatenate([np.array(rows)], axis=1).astype(np.float32)
    codes, sexp = O.quantize_rows_mxfp4(x)
    assert np.array_equal(O.dequant_rows_mxfp4(codes, sexp), x.astype(np.float64))
    assert sexp[:, 0].tolist() == [127 - 9, 127 - 1, 127, 127 + 3]
    c1, s1 = O.quantize_rows_mxfp4(np.full((1, 32), 5.0, np.float32))   # 5 = 1.25 * 4: X = 1
    assert s1[0, 0] == 127 and (c1 == 6).all()                          # 5 -> tie(4, 6) -> 4 (even)
    c2, s2 = O.quantize_rows_mxfp4(np.full((1, 32), -7.0, np.float32))  # 7 / 1 -> clamp 6
    assert s2[0, 0] == 127 and (c2 == 0xF).all()
