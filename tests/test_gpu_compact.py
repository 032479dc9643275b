"""GPU compaction (Alg. 2 "Remove h from b") against the oracle: bit-exact
columns, N', S_alive, new offsets and the row map."""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def run(N, S_sizes, alive, row_bytes_list, seed=0, alive_shift=0):
    import paper_1805_09863_b200 as amun
    off = torch.tensor(np.concatenate([[0], np.cumsum(S_sizes)]), dtype=torch.int32)
    assert int(off[-1]) == N
    cols_h = [synth.gen_bytes(seed + i, synth.S_STATE, N * rb).view(N, rb) if N else
              torch.empty(0, rb, dtype=torch.uint8) for i, rb in enumerate(row_bytes_list)]
    cols_d = [(c.to(DEV), torch.full_like(c, 0xAB, device=DEV)) for c in cols_h]
    alive_d = alive.to(DEV)
    if alive_shift:   # flags at a non-16-byte-aligned address (byte path)
        buf = torch.zeros(N + alive_shift, dtype=torch.uint8, device=DEV)
        buf[alive_shift:] = alive_d
        alive_d = buf[alive_shift:]
    n, s_alive, new_off, src_row, counts = amun.compact(cols_d, alive_d, off.to(DEV))
    ref_cols, ref_off, ref_src, ref_n, ref_s = O.compact([c.numpy() for c in cols_h],
                                                          alive.numpy(), off.numpy())
    assert n == ref_n and s_alive == ref_s
    assert counts.cpu().tolist() == [ref_n, ref_s]
    assert np.array_equal(new_off.cpu().numpy(), ref_off)
    assert np.array_equal(src_row[:n].cpu().numpy(), ref_src)
    for (src, dst), ref in zip(cols_d, ref_cols):
        assert np.array_equal(dst[:n].cpu().numpy(), ref)
        if n < N:   # rows past N' untouched
            assert (dst[n:].cpu().numpy() == 0xAB).all()


@pytest.mark.parametrize("p", [0.0, 0.1, 0.5, 0.9, 0.99, 1.0])
def test_random_masks(p):
    N, B = 6400, 5
    alive = synth.gen_alive(int(p * 100), N, p)
    run(N, [B] * (N // B), alive, [2048, 8192, 4, 8])


def test_cfg4_state_row():
    """The cfg4 per-hypothesis state: x bf16 [1024] 2048 B + decoder state 2x1024
    fp32 8192 B + prev_cost 4 B + (sentence, slot) id 8 B = 10,252 B/row."""
    f = synth.eos_schedule(synth.BASE_SEED + 4, 1280, 5).reshape(-1)
    for t in [1, 5, 20, 40]:
        alive = (f > t).to(torch.uint8)
        run(6400, [5] * 1280, alive, [2048, 8192, 4, 8], seed=t)


@pytest.mark.parametrize("N", [0, 1, 31, 33, 257, 1000])
def test_small_and_ragged(N):
    rng = np.random.default_rng(N)
    sizes = []
    left = N
    while left > 0:
        s = int(min(left, rng.integers(0, 7)))
        sizes.append(s)
        left -= s
    sizes.append(0)
    alive = torch.from_numpy((rng.random(N) < 0.6).astype(np.uint8))
    run(N, sizes, alive, [16, 4, 48, 20])


def test_one_survivor_per_sentence_and_alternating():
    N, B = 1200, 6
    alive = torch.zeros(N, dtype=torch.uint8)
    alive[::B] = 1
    run(N, [B] * (N // B), alive, [64])
    alive = torch.tensor([i % 2 for i in range(N)], dtype=torch.uint8)
    run(N, [B] * (N // B), alive, [64, 12])


@pytest.mark.parametrize("shift", [1, 3, 8])
def test_unaligned_flags(shift):
    N = 1001
    rng = np.random.default_rng(shift)
    alive = torch.from_numpy((rng.random(N) < 0.5).astype(np.uint8))
    run(N, [7] * 143, alive, [32, 4], alive_shift=shift)


@pytest.mark.parametrize("N,B", [(70001, 1), (65536, 12), (16389, 3)])
def test_large_ragged(N, B):
    """Several 16-byte flag words per scan thread, S > 256 * grid-limit cases,
    flag counts that end mid-word (masked-tail path)."""
    rng = np.random.default_rng(N)
    sizes = [B] * (N // B) + ([N % B] if N % B else [])
    alive = torch.from_numpy((rng.random(N) < 0.3).astype(np.uint8))
    run(N, sizes, alive, [16, 4])


@pytest.mark.parametrize("S,B,p", [(1, 1, 0.0), (7, 3, 0.5), (300, 5, 0.3), (1280, 5, 0.9)])
def test_sentence_columns_follow_their_rows(S, B, p):
    """f1 (optional part): after the row compaction, the sentence-level
    columns (here an encoder context [S, 64, 32] bf16-sized bytes and a source
    length [S] int32) keep exactly the sentences with surviving rows, stably
    (amun_sentence_alive + amun_compact), bit-exact with the oracle's
    compaction under alive_s[s] = new_off[s+1] > new_off[s]."""
    import paper_1805_09863_b200 as m
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(S * 7 + B)
    N = S * B
    alive = (torch.rand(N, generator=g) >= p).to(torch.uint8)
    off = torch.arange(0, N + 1, B, dtype=torch.int32)
    ctx = torch.randint(0, 256, (S, 64 * 32 * 2), generator=g, dtype=torch.uint8)
    slen = torch.randint(1, 100, (S,), generator=g, dtype=torch.int32)
    x = torch.randint(0, 256, (N, 16), generator=g, dtype=torch.uint8)
    xd = torch.empty_like(x, device=dev)
    n_rows, s_alive, new_off, _, _ = m.compact([(x.to(dev), xd)], alive.to(dev), off.to(dev))
    ctx_d, slen_d = torch.empty_like(ctx, device=dev), torch.empty_like(slen, device=dev)
    S_kept, src_s, counts = m.compact_sentences([(ctx.to(dev), ctx_d), (slen.to(dev), slen_d)], new_off)
    torch.cuda.synchronize()
    _, o_new_off, _, _, o_S_alive = O.compact([x.numpy()], alive.numpy(), off.numpy())
    alive_s = (o_new_off[1:] > o_new_off[:-1]).astype(np.uint8)
    (o_ctx, o_slen), _, o_src, o_n, _ = O.compact([ctx.numpy(), slen.numpy().view(np.uint8).reshape(S, 4)],
                                                  alive_s, np.arange(S + 1))
    assert S_kept == o_n == o_S_alive == s_alive
    assert np.array_equal(src_s[:S_kept].cpu().numpy(), o_src)
    assert np.array_equal(ctx_d[:S_kept].cpu().numpy(), o_ctx)
    assert np.array_equal(slen_d[:S_kept].cpu().numpy().view(np.uint8).reshape(-1, 4), o_slen)
