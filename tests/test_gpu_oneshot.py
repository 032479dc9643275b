"""GPU parity of the NVLink one-shot exchange + merge (
amun_output_layer_oneshot / _emulated, csrc/oneshot.cuh): the vocab-sharded
output layer (Alg. 6) with the per-row partial records pushed into
every rank's receive buffer by the library's own kernel, then merged.

One GPU: G ranks run as ONE cooperative kernel with a grid row per rank
(B200_PROFILING.md: ranks whose blocks wait on one another must not be
separate launches on one GPU); the real-mode entry point runs at G = 1
through the IPC-exported buffer. Checks: every rank's result is BIT-identical
to the collective path (per-shard partial + stacked all-gather +
amun_merge_partials, itself oracle-tested) and passes the oracle comparator;
repeated calls (epoch parity, monotonic counters) and CUDA-graph replays give
the same results; empty inputs pad."""
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


def shards(w, G, dtype="bf16"):
    from paper_1805_09863_b200.sharded import shard_range
    layers, Ws, bs = [], [], []
    for g in range(G):
        v0, v1 = shard_range(w.V, G, g)
        layers.append(amun().OutputLayer(w.H, v1 - v0, v_offset=v0, V_total=w.V, k_max=w.k,
                                         max_rows=max(w.N, 1), max_sentences=max(w.S, 1)))
        Ws.append(synth.gen_W(w, v0, v1 - v0).to(DEV))
        bs.append(synth.gen_b(w, v0, v1 - v0).to(DEV))
    return layers, Ws, bs


def collective(layers, X, Ws, bs, pc, off, k, ks=None):
    parts = [ol.partial(X, W, b) for ol, W, b in zip(layers, Ws, bs)]
    return layers[0].merge(torch.stack(parts), pc, off, k, ks)


def oracle_check(w, idx, cost, ks=None):
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))), O.as_f64(synth.gen_b(w)))
    logp = O.log_softmax(L)
    off = synth.gen_offsets(w).numpy()
    _, _, oc64, nxt = O.kbest_sentences(logp, O.as_f64(synth.gen_prev_cost(w)), off, w.k,
                                        None if ks is None else np.asarray(ks))
    pcd = O.as_f64(synth.gen_prev_cost(w))
    kk = np.full(w.S, w.k) if ks is None else np.minimum(np.asarray(ks), w.k)
    return compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: pcd[r] + logp[r, v],
                         oc64, kk, "bf16", w.V, o_next=nxt)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_emulated_ranks_equal_collective_path(G):
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    w = synth.Workload("os", H=256, V=30011, S=16, B=4, k=6, seed=synth.BASE_SEED + 200 + G)
    layers, Ws, bs = shards(w, G)
    X, pc, off = synth.gen_X(w).to(DEV), synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ref_i, ref_c = collective(layers, X, Ws, bs, pc, off, w.k)
    em = EmulatedOneShot(layers)
    for call in range(3):          # epochs 0, 1, 2: both receive halves, counters advance
        outs = em(X, Ws, bs, pc, off, w.k)
        torch.cuda.synchronize()
        for g, (i, c) in enumerate(outs):
            assert torch.equal(i, ref_i), (call, g)
            assert torch.equal(c, ref_c), (call, g)
    oracle_check(w, outs[0][0], outs[0][1])
    em.close()


def test_emulated_changing_inputs_and_ragged_k():
    """Successive calls with different X / prev_cost (a decode loop) and
    per-sentence k: each call equals the collective path on its inputs."""
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    w = synth.Workload("os2", H=128, V=9000, S=9, B=5, k=5, seed=synth.BASE_SEED + 301)
    layers, Ws, bs = shards(w, 4)
    em = EmulatedOneShot(layers)
    off = synth.gen_offsets(w).to(DEV)
    ks = torch.tensor([1, 5, 3, 0, 5, 2, 4, 5, 1], dtype=torch.int32, device=DEV)
    g = torch.Generator().manual_seed(5)
    for call in range(5):
        X = (torch.randn(w.N, w.H, generator=g) * 0.5).to(torch.bfloat16).to(DEV)
        pc = (torch.rand(w.N, generator=g) * -3).to(DEV)
        ref_i, ref_c = collective(layers, X, Ws, bs, pc, off, w.k, ks)
        outs = em(X, Ws, bs, pc, off, w.k, ks)
        torch.cuda.synchronize()
        for i, c in outs:
            assert torch.equal(i, ref_i) and torch.equal(c, ref_c), call
    em.close()


def test_emulated_cuda_graph_replay():
    """The cooperative one-shot launch captured in a CUDA graph: replays keep
    advancing the device epochs and give the eager result every time."""
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    w = synth.Workload("os3", H=256, V=20000, S=24, B=5, k=5, seed=synth.BASE_SEED + 302)
    layers, Ws, bs = shards(w, 2)
    X, pc, off = synth.gen_X(w).to(DEV), synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ref_i, ref_c = collective(layers, X, Ws, bs, pc, off, w.k)
    em = EmulatedOneShot(layers)
    outs = [(torch.empty_like(ref_i), torch.empty_like(ref_c)) for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        em(X, Ws, bs, pc, off, w.k, outs=outs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            em(X, Ws, bs, pc, off, w.k, outs=outs)
    torch.cuda.synchronize()
    for rep in range(4):
        for o in outs:
            o[0].fill_(-7)
        graph.replay()
        torch.cuda.synchronize()
        for i, c in outs:
            assert torch.equal(i, ref_i) and torch.equal(c, ref_c), rep
    em.close()


def test_emulated_empty():
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    w = synth.Workload("os4", H=64, V=3000, S=3, B=2, k=2, seed=synth.BASE_SEED + 303)
    layers, Ws, bs = shards(w, 2)
    em = EmulatedOneShot(layers)
    X = torch.empty((0, w.H), dtype=torch.bfloat16, device=DEV)
    pc = torch.empty(0, dtype=torch.float32, device=DEV)
    off = torch.zeros(4, dtype=torch.int32, device=DEV)           # 3 sentences, no rows
    outs = em(X, Ws, bs, pc, off, w.k)
    torch.cuda.synchronize()
    for i, c in outs:
        assert (i == -1).all() and torch.isneginf(c).all()
    # and the epochs stay consistent for a following non-empty call
    X, pc, off = synth.gen_X(w).to(DEV), synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ref_i, ref_c = collective(layers, X, Ws, bs, pc, off, w.k)
    outs = em(X, Ws, bs, pc, off, w.k)
    torch.cuda.synchronize()
    for i, c in outs:
        assert torch.equal(i, ref_i) and torch.equal(c, ref_c)
    em.close()


def test_real_mode_single_rank_ipc_buffer():
    """amun_output_layer_oneshot itself (rank parameter, IPC-exported buffer)
    at world 1 through ShardedOutputLayer(exchange="oneshot"): equals the
    single-GPU path over repeated calls. With the fused tail (default) the
    whole exchange runs inside the fused kernel (one launch); AMUN_TAIL=off
    gives the fused kernel + the separate one-shot kernel."""
    from paper_1805_09863_b200.sharded import ShardedOutputLayer
    w = synth.CONFIGS["beam"]
    sh = ShardedOutputLayer(w.H, w.V, 1, 0, k_max=w.k, max_rows=w.N, max_sentences=w.S,
                            exchange="oneshot")
    assert sh.launches_per_step == sh.ol.launches["call"]
    assert not sh.oneshot.error()
    X, W, b = synth.gen_X(w).to(DEV), synth.gen_W(w).to(DEV), synth.gen_b(w).to(DEV)
    pc, off = synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ref_i, ref_c = sh.ol(X, W, b, pc, off, w.k)
    for call in range(3):
        i, c = sh(X, W, b, pc, off, w.k)
        torch.cuda.synchronize()
        assert torch.equal(i, ref_i) and torch.equal(c, ref_c), call
    assert not sh.oneshot.error()
    sh.oneshot.close()


@pytest.mark.slow
def test_cfg_shard_8_ranks_emulated():
    """cfg 'shard' (H=1024, V=256000, 1024 x 12, k=12) over 8 emulated ranks
    (the CTA-pair fused kernel per shard): bit-identical to the collective
    path; every 128th sentence against the oracle."""
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    w = synth.CONFIGS["shard"]
    layers, Ws, bs = shards(w, 8)
    X, pc, off = synth.gen_X(w).to(DEV), synth.gen_prev_cost(w).to(DEV), synth.gen_offsets(w).to(DEV)
    ref_i, ref_c = collective(layers, X, Ws, bs, pc, off, w.k)
    em = EmulatedOneShot(layers)
    outs = em(X, Ws, bs, pc, off, w.k)
    torch.cuda.synchronize()
    for i, c in outs:
        assert torch.equal(i, ref_i) and torch.equal(c, ref_c)
    em.close()
    from tests.test_gpu_output_layer import _sampled_oracle_check
    rep = _sampled_oracle_check(w, outs[3][0], outs[3][1], list(range(0, w.S, 128)), w.V)
    assert rep["sentences_checked"] == 8


def test_invalid_arguments():
    from paper_1805_09863_b200.sharded import EmulatedOneShot
    m = amun()
    ol = m.OutputLayer(64, 1000, k_max=2, max_rows=8, max_sentences=4)
    X = torch.zeros((8, 64), dtype=torch.bfloat16, device=DEV)
    W = torch.zeros((1000, 64), dtype=torch.bfloat16, device=DEV)
    b = torch.zeros(1000, device=DEV)
    pc = torch.zeros(8, device=DEV)
    off = torch.tensor([0, 4, 8], dtype=torch.int32, device=DEV)
    with pytest.raises(m.AmunError):
        ol.oneshot(X, W, b, pc, off, 2, [], 0)                    # G = 0
    with pytest.raises(m.AmunError):
        ol.oneshot(X, W, b, pc, off, 2, [0], 0)                   # NULL buffer
    with pytest.raises(m.AmunError):
        ol.oneshot(X, W, b, pc, off, 2, [256] * 9, 0)             # G > 8
    em = EmulatedOneShot([ol])
    with pytest.raises(m.AmunError):
        ol.oneshot(X, W, b, pc, off, 2, em.bufs, 1)               # rank >= G
    em.close()
