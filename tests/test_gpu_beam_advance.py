"""GPU beam advance (amun_beam_advance; SPEC S:324-332 expand_beam + Alg. 2)
against oracle.beam_advance: bit-exact offsets, parent rows, tokens, costs,
N', S_alive and every gathered state column."""
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


def check(idx, cost, V, eos, N, row_bytes_list, seed=0):
    S, k = idx.shape
    cols_h = [synth.gen_bytes(seed + i, synth.S_STATE, max(N, 1) * rb).view(max(N, 1), rb)[:N]
              for i, rb in enumerate(row_bytes_list)]
    cols_d = [(c.contiguous().to(DEV), torch.full((max(S * k, 1), c.shape[1]), 0xAB, dtype=torch.uint8,
                                                  device=DEV)) for c in cols_h]
    n, s_alive, off, src, tok, cst, counts = amun().beam_advance(
        idx.to(DEV), cost.to(DEV), V, eos, N, cols_d)
    r = O.beam_advance(idx.numpy(), cost.numpy(), V, eos, [c.numpy() for c in cols_h])
    ncols, roff, rsrc, rtok, rcost, rn, rs, fin = r
    assert n == rn and s_alive == rs
    assert counts.cpu().tolist() == [rn, rs]
    assert np.array_equal(off.cpu().numpy(), roff)
    assert np.array_equal(src[:n].cpu().numpy(), rsrc)
    assert np.array_equal(tok[:n].cpu().numpy(), rtok)
    assert np.array_equal(cst[:n].cpu().numpy().view(np.uint32), rcost.view(np.uint32))
    for (_, dst), ref in zip(cols_d, ncols):
        assert np.array_equal(dst[:n].cpu().numpy(), ref)
        assert (dst[n:].cpu().numpy() == 0xAB).all()          # rows past N' untouched
    return n


def winners(rng, S, k, B, V, eos, p_eos, p_pad):
    """Random selection output: sentence s owns rows [s B, s B + B); winner i
    picks a parent row in it (repeats allowed) and a token; EOS / padding mixed in."""
    parent = np.arange(S)[:, None] * B + rng.integers(0, B, (S, k))
    tok = rng.integers(0, V, (S, k))
    tok[rng.random((S, k)) < p_eos] = eos
    idx = parent * V + tok
    idx[rng.random((S, k)) < p_pad] = -1
    cost = -rng.random((S, k)).astype(np.float32) * 20
    cost[idx < 0] = -np.inf
    return torch.from_numpy(idx.astype(np.int64)), torch.from_numpy(cost)


@pytest.mark.parametrize("S,k,p_eos,p_pad", [(128, 5, 0.1, 0.0), (1280, 5, 0.3, 0.05),
                                             (7, 12, 0.5, 0.2), (300, 1, 0.2, 0.0)])
def test_random_winners(S, k, p_eos, p_pad):
    rng = np.random.default_rng(S + k)
    V, eos, B = 90000, 2, k
    idx, cost = winners(rng, S, k, B, V, eos, p_eos, p_pad)
    check(idx, cost, V, eos, S * B, [2048, 8192, 4, 8], seed=S)


def test_all_eos_and_all_padding():
    rng = np.random.default_rng(1)
    V, eos, S, k = 1000, 0, 20, 3
    idx = torch.from_numpy((np.arange(S * k) * V + eos).reshape(S, k).astype(np.int64))
    cost = torch.from_numpy(-rng.random((S, k)).astype(np.float32))
    assert check(idx, cost, V, eos, S * k, [16]) == 0
    idx = torch.full((S, k), -1, dtype=torch.int64)
    cost = torch.full((S, k), -np.inf, dtype=torch.float32)
    assert check(idx, cost, V, eos, S * k, [16]) == 0


def test_empty_and_ragged_columns():
    rng = np.random.default_rng(2)
    idx, cost = winners(rng, 33, 4, 4, 777, 5, 0.25, 0.1)
    check(idx, cost, 777, 5, 33 * 4, [12, 20, 4])                # non-16-byte rows: word path
    idx0 = torch.zeros((0, 4), dtype=torch.int64)
    check(idx0, torch.zeros((0, 4)), 777, 5, 0, [16])


def test_chain_with_output_layer():
    """One decode step end to end on the device: output layer -> beam advance,
    then the next step's output layer on the advanced (gathered) X."""
    w = synth.Workload("adv", H=256, V=5000, S=24, B=4, k=4, seed=synth.BASE_SEED + 91)
    X, W, b = synth.gen_X(w).to(DEV), synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV)
    pc, off = synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ol = amun().OutputLayer(w.H, w.V, k_max=w.k, max_rows=w.N, max_sentences=w.S)
    idx, cost = ol(X, W, b, pc, off, w.k)
    eos = int((idx[0, 0] % w.V).item())                     # make sentence 0's best finish
    Xn = torch.empty_like(X)
    n, s_alive, noff, src, tok, ncost, _ = amun().beam_advance(idx, cost, w.V, eos, w.N, [(X, Xn)])
    ref = O.beam_advance(idx.cpu().numpy(), cost.cpu().numpy(), w.V, eos,
                         [X.cpu().view(torch.uint8).numpy().reshape(w.N, -1)])
    assert n == ref[5] and np.array_equal(noff.cpu().numpy(), ref[1])
    assert torch.equal(Xn[:n], X[src[:n].long()])
    idx2, cost2 = ol(Xn[:n], W, b, ncost[:n].contiguous(), noff, w.k)   # next step runs
    torch.cuda.synchronize()
    assert (idx2[noff[1:] > noff[:-1]] >= 0).all()
