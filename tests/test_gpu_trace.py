"""Decode trace (Alg. 1 naive vs Alg. 2 dynamic mini-batching) on the GPU:
every step's output layer matches the oracle, every compaction is bit-exact
against the oracle's, and the work accounting matches the analytic count
(S:321-322 style: dynamic rows = sum of per-hypothesis step counts)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from tests.compare import compare_kbest

pytestmark = pytest.mark.gpu


def test_trace_dynamic_and_naive():
    from paper_1805_09863_b200.trace import DecodeTrace
    S, B, H, V = 24, 5, 128, 3000
    w = synth.Workload("trace-small", H=H, V=V, S=S, B=B, k=B, seed=synth.BASE_SEED + 44)
    X, W, b, pc = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w), synth.gen_prev_cost(w)
    f = synth.eos_schedule(w.seed, S, B, p=1 / 3, cap=6)          # short sentences
    dev = torch.device("cuda", 0)
    tr = DecodeTrace(H, V, S, B, device=dev)
    Wd, bd = W.to(dev), b.to(dev)
    Wo, bo = O.as_f64(W), O.as_f64(b)
    seen = {"ol": 0, "compact": 0}

    def as_bytes(c):
        rb = c.element_size()
        for d in c.shape[1:]:
            rb *= int(d)
        return c.contiguous().view(torch.uint8).reshape(c.shape[0], rb).cpu().numpy()

    def check(t, inp, out):
        if inp[0] == "compact":
            _, src_cols, alive, off = inp
            dst_cols, new_off, src_row, counts = out
            ref = O.compact([as_bytes(c) for c in src_cols], alive.cpu().numpy(), off.cpu().numpy())
            rc, ro, rs, rn, rsa = ref
            assert counts.cpu().tolist() == [rn, rsa]
            assert np.array_equal(new_off.cpu().numpy(), ro)
            assert np.array_equal(src_row.cpu().numpy(), rs)
            for d, r in zip(dst_cols, rc):
                assert np.array_equal(as_bytes(d), r)
            seen["compact"] += 1
            return
        Xs, _, _, prev, off, k_s = inp
        idx, cost = out
        logp = O.log_softmax(O.add_bias(O.gemm(O.as_f64(Xs), Wo), bo))
        prevd = O.as_f64(prev)
        oi, _, oc64, nxt = O.kbest_sentences(logp, prevd, off.cpu().numpy(), B, k_s.cpu().numpy())
        compare_kbest(idx.cpu().numpy(), cost.cpu().numpy(), lambda s, r, v: prevd[r] + logp[r, v],
                      oc64, k_s.cpu().numpy(), "bf16", V, o_next=nxt)
        seen["ol"] += 1

    dyn = tr.run(X, Wd, bd, pc, f, mode="dynamic", check=check)
    assert seen["ol"] == dyn.steps and seen["compact"] == dyn.steps
    assert sum(dyn.rows) == int(f.sum())                     # Alg. 2 work accounting
    assert dyn.rows == sorted(dyn.rows, reverse=True)        # the batch only shrinks
    nai = tr.run(X, Wd, bd, pc, f, mode="naive")
    assert sum(nai.rows) == int(f.max()) * S * B             # Alg. 1 decodes every slot
    assert nai.steps == dyn.steps == int(f.max())


@pytest.mark.slow
def test_trace_full_size_sampled():
    """BASELINE cfg 'trace' at full size (1280 sentences x beam 5, V = 90000,
    H = 1024): compaction bit-exact against the oracle at EVERY step; the output
    layer against the oracle on 16 sampled sentences at 4 sampled steps."""
    from paper_1805_09863_b200.trace import DecodeTrace
    w = synth.CONFIGS["trace"]
    S, B, H, V = w.S, w.B, w.H, w.V
    X, W, b, pc = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w), synth.gen_prev_cost(w)
    f = synth.eos_schedule(w.seed, S, B)
    dev = torch.device("cuda", 0)
    tr = DecodeTrace(H, V, S, B, device=dev)
    Wo, bo = O.as_f64(W), O.as_f64(b)
    steps_checked = {0, 5, 20, 40}
    seen = {"compact": 0, "ol": 0}

    def as_bytes(c):
        rb = c.element_size()
        for d in c.shape[1:]:
            rb *= int(d)
        return c.contiguous().view(torch.uint8).reshape(c.shape[0], rb).cpu().numpy()

    def check(t, inp, out):
        if inp[0] == "compact":
            _, src_cols, alive, off = inp
            dst_cols, new_off, src_row, counts = out
            rc, ro, rs, rn, rsa = O.compact([as_bytes(c) for c in src_cols], alive.cpu().numpy(),
                                            off.cpu().numpy())
            assert counts.cpu().tolist() == [rn, rsa]
            assert np.array_equal(new_off.cpu().numpy(), ro)
            assert np.array_equal(src_row.cpu().numpy(), rs)
            for d, r in zip(dst_cols, rc):
                assert np.array_equal(as_bytes(d), r)
            seen["compact"] += 1
            return
        if t not in steps_checked:
            return
        Xs, _, _, prev, off, k_s = inp
        idx, cost = out
        offn, ksn = off.cpu().numpy(), k_s.cpu().numpy()
        live = [s for s in range(S) if offn[s + 1] > offn[s]]
        sent = live[:: max(1, len(live) // 16)][:16]
        rows = np.concatenate([np.arange(offn[s], offn[s + 1]) for s in sent])
        logp = O.log_softmax(O.add_bias(O.gemm(O.as_f64(Xs[torch.from_numpy(rows).to(Xs.device)]), Wo), bo))
        prevd = O.as_f64(prev)[rows]
        sub_off = np.concatenate([[0], np.cumsum([offn[s + 1] - offn[s] for s in sent])])
        _, _, oc64, nxt = O.kbest_sentences(logp, prevd, sub_off, B, ksn[sent])
        pos = {int(r): i for i, r in enumerate(rows)}
        compare_kbest(idx.cpu().numpy()[sent], cost.cpu().numpy()[sent],
                      lambda s, r, v: prevd[pos[r]] + logp[pos[r], v], oc64, ksn[sent], "bf16", V,
                      o_next=nxt)
        seen["ol"] += 1

    dyn = tr.run(X, W.to(dev), b.to(dev), pc, f, mode="dynamic", check=check)
    assert seen["compact"] == dyn.steps and seen["ol"] == 4
    assert sum(dyn.rows) == int(f.sum())


def test_trace_graph_mode_same_rows_as_dynamic():
    """Alg. 2 with N on the device, all steps in one CUDA graph (run_graph):
    the schedule alone decides the live rows, so every step must decode
    exactly the rows the eager dynamic mode decodes."""
    from paper_1805_09863_b200.trace import DecodeTrace
    S, B, H, V = 40, 5, 128, 3000
    w = synth.Workload("trace-graph", H=H, V=V, S=S, B=B, k=B, seed=synth.BASE_SEED + 45)
    X, W, b, pc = synth.gen_X(w), synth.gen_W(w), synth.gen_b(w), synth.gen_prev_cost(w)
    f = synth.eos_schedule(w.seed, S, B, p=1 / 4, cap=9)
    dev = torch.device("cuda", 0)
    tr = DecodeTrace(H, V, S, B, device=dev)
    Wd, bd = W.to(dev), b.to(dev)
    dyn = tr.run(X, Wd, bd, pc, f, mode="dynamic")
    gr = tr.run_graph(X, Wd, bd, pc, f, log_steps=(0, 2, 4, 6))
    assert gr.rows[:len(dyn.rows)] == dyn.rows
    # the graph-mode winners against the oracle on the step's own inputs
    Wo, bo = O.as_f64(W), O.as_f64(b)
    for t, lg in gr.logs.items():
        n = int(lg["N"][0])
        assert n == gr.rows[t]
        logp = O.log_softmax(O.add_bias(O.gemm(O.as_f64(lg["X"][:n]), Wo), bo))
        prevd = O.as_f64(lg["prev"][:n])
        offn, ksn = lg["off"].numpy(), lg["k_s"].numpy()
        _, _, oc64, nxt = O.kbest_sentences(logp, prevd, offn, B, ksn)
        compare_kbest(lg["idx"].numpy(), lg["cost"].numpy(), lambda s, r, v: prevd[r] + logp[r, v],
                      oc64, ksn, "bf16", V, o_next=nxt)
    assert all(n == 0 for n in gr.rows[len(dyn.rows):])
    assert sum(gr.rows) == int(f.sum())
    # the surviving ids after the last step: none (everything finished)
    final = tr._graph_state["cnt"][gr.steps % 2]
    assert int(final[0].item()) == 0
