"""Vocab-sharded path across real NCCL ranks (north_star: "a small NCCL
all-gather over NVLink feeds an exact cross-shard merge"; Alg. 6's shard +
reduce). Spawns torch.cuda.device_count() processes, one per GPU,
with the NCCL backend: every rank runs the library's partial kernel on its
vocab shard, the records travel through NCCL (all_gather_into_tensor — it
runs even at world 1, force_sharded=True), and every rank merges. Rank 0's
output is compared with the oracle on the full vocabulary; all ranks must
hold bit-identical outputs. The one-shot exchange (f3) runs through real IPC
buffers at the same world size and must be bit-identical to the NCCL path
(reading G18)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from tests.compare import compare_kbest

W_CFG = synth.Workload("mr", H=256, V=20011, S=12, B=3, k=4, seed=synth.BASE_SEED + 31)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        from paper_1805_09863_b200.sharded import ShardedOutputLayer, shard_range
        w = W_CFG
        v0, v1 = shard_range(w.V, world, rank)
        X, pc, off = (synth.gen_X(w).to(dev), synth.gen_prev_cost(w).to(dev),
                      synth.gen_offsets(w).to(dev))
        W, b = synth.gen_W(w, v0, v1 - v0).to(dev), synth.gen_b(w, v0, v1 - v0).to(dev)
        outs = {}
        for ex in ("nccl", "oneshot"):
            lay = ShardedOutputLayer(w.H, w.V, world, rank, k_max=w.k, max_rows=w.N,
                                     max_sentences=w.S, device=dev, exchange=ex,
                                     force_sharded=True)
            for _ in range(3):        # repeated calls (epochs / generations advance)
                idx, cost = lay(X, W, b, pc, off, w.k)
            torch.cuda.synchronize()
            outs[ex] = (idx.clone(), cost.clone())
            # every rank holds the same merged output
            a = torch.cat([idx.view(-1).double(), cost.view(-1).double()])
            lo, hi = a.clone(), a.clone()
            dist.all_reduce(lo, op=dist.ReduceOp.MIN)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX)
            outs[ex + "_identical"] = bool(torch.equal(lo, hi))
            if lay.oneshot is not None:
                lay.oneshot.close()
            del lay
        if rank == 0:
            q.put({"world": world,
                   "nccl": [t.cpu().numpy() for t in outs["nccl"]],
                   "oneshot": [t.cpu().numpy() for t in outs["oneshot"]],
                   "identical": (outs["nccl_identical"], outs["oneshot_identical"])})
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:   # noqa: BLE001 (reported to the parent)
        q.put({"error": f"rank {rank}: {type(e).__name__}: {e}"})
        raise


@pytest.mark.gpu
def test_nccl_ranks_match_oracle_and_oneshot():
    world = torch.cuda.device_count()
    assert world >= 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
    assert "error" not in res, res
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert res["world"] == world and res["identical"] == (True, True)
    gi, gc = res["nccl"]
    oi, oc = res["oneshot"]
    assert np.array_equal(gi, oi) and np.array_equal(gc, oc), "one-shot != NCCL path"
    w = W_CFG
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))),
                   O.as_f64(synth.gen_b(w)))
    logp = O.log_softmax(L)
    pcs = O.as_f64(synth.gen_prev_cost(w))
    off = np.arange(w.S + 1) * w.B
    _, _, oc64, nxt = O.kbest_sentences(logp, pcs, off, w.k)
    compare_kbest(gi, gc, lambda s, r, v: pcs[r] + logp[r, v], oc64, np.full(w.S, w.k), "bf16",
                  w.V, o_next=nxt)
