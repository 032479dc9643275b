"""The seeded generator (synth/) against Python big-integer splitmix64 and
the recipe it claims (SURVEY.md §8(d) 'Synthetic inputs')."""
import math

import numpy as np
import torch

import synth


def test_splitmix_matches_bigint():
    for seed, stream, start in [(0, 0, 0), (synth.BASE_SEED, 2, 12345), (7, 5, 2**40)]:
        z = synth.raw64(seed, stream, start, 64)
        key = synth.stream_key(seed, stream)
        ref = [synth.mix64_int(key + i * synth.GOLDEN) for i in range(start, start + 64)]
        got = [int(a) & synth.MASK64 for a in z.tolist()]
        assert got == ref


def test_bf16_rne_matches_torch_cast():
    x = synth.normal(3, 9, 0, 100000) * 7.0
    a = synth.f32_to_bf16_rne(x)
    b = x.to(torch.bfloat16)  # torch's cast is RNE for finite values
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_slices_are_consistent():
    """A vocab shard regenerates exactly its slice of the global W."""
    w = synth.Workload("t", H=48, V=300, S=2, B=2, k=2)
    W = synth.gen_W(w)
    for v0, n in [(0, 300), (17, 100), (299, 1), (150, 150)]:
        assert torch.equal(synth.gen_W(w, v0, n).view(torch.int16), W[v0:v0 + n].view(torch.int16))
    X = synth.gen_X(w)
    assert torch.equal(synth.gen_X(w, 1, 2).view(torch.int16), X[1:3].view(torch.int16))


def test_recipe_moments():
    w = synth.Workload("t", H=1024, V=2000, S=4, B=5, k=5)
    W = synth.gen_W(w).float()
    assert abs(W.std().item() - 3.0 / math.sqrt(1024 / 3)) < 2e-3
    X = synth.gen_X(w).float()
    assert X.abs().max() <= 1.0 and abs(X.mean().item()) < 0.02
    b = synth.gen_b(w)
    assert b[0] == 0 and abs(b[99].item() + 0.5 * math.log(100)) < 1e-6
    pc = synth.gen_prev_cost(w).view(4, 5)
    assert (pc <= 0).all() and (pc >= -20).all()
    assert (pc[:, :-1] >= pc[:, 1:]).all()
    assert synth.gen_offsets(w).tolist() == [0, 5, 10, 15, 20]


def test_eos_schedule_shape():
    f = synth.eos_schedule(synth.BASE_SEED + 4, 1280, 5)
    assert f.shape == (1280, 5)
    assert (f[:, 1:] - f[:, :-1] == 1).all()
    assert f[:, 0].min() >= 1 and f[:, 0].max() <= 60
    assert 15 < f[:, 0].float().mean() < 22
