"""Vocab-sharded path, host logic, world_size 2 over gloo on CPU: each rank
owns shard_range(V, 2, rank) of the vocabulary, builds its per-row partial
records in the ABI layout {m, s, l[k], v[k]} (here from the oracle's
shard_partial, since there is no GPU), exchanges them with the SAME
sharded.exchange() the GPU path uses (all_gather_into_tensor), and merges in
rank order. The result must equal the oracle on the full vocabulary."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pack(m, s, l, v, k):
    N = len(m)
    rec = np.zeros((N, 2 + 2 * k), np.float32)
    rec[:, 0] = m
    rec[:, 1] = s
    rec[:, 2:2 + k] = l
    rec[:, 2 + k:] = v.astype(np.int32).view(np.float32)
    return torch.from_numpy(rec)


def _unpack(rec, k):
    rec = rec.numpy()
    return (rec[:, 0].astype(np.float64), rec[:, 1].astype(np.float64),
            rec[:, 2:2 + k].astype(np.float64), rec[:, 2 + k:].copy().view(np.int32).astype(np.int64))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_09863_b200.sharded import exchange, shard_range
    w = synth.Workload("sh", H=32, V=1001, S=6, B=3, k=4, dist="flat", seed=synth.BASE_SEED + 7)
    v0, v1 = shard_range(w.V, world, rank)
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w, v0, v1 - v0))),
                   O.as_f64(synth.gen_b(w, v0, v1 - v0)))
    part = _pack(*O.shard_partial(L, w.k, v_offset=v0), w.k)
    allp = exchange(part, world)                     # [world, N, 2+2k]
    if rank == 0:
        parts = [_unpack(allp[g], w.k) for g in range(world)]
        M, S, l, v = O.combine_partials(parts, w.k)
        q.put((M, S, v, [shard_range(w.V, world, g) for g in range(world)]))
    dist.destroy_process_group()


def test_two_rank_exchange_and_merge():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    M, S, v, ranges = q.get(timeout=10)
    w = synth.Workload("sh", H=32, V=1001, S=6, B=3, k=4, dist="flat", seed=synth.BASE_SEED + 7)
    assert ranges[0][0] == 0 and ranges[-1][1] == w.V and ranges[0][1] == ranges[1][0]
    L = O.add_bias(O.gemm(O.as_f64(synth.gen_X(w)), O.as_f64(synth.gen_W(w))), O.as_f64(synth.gen_b(w)))
    fm, fs, fl, fv = O.shard_partial(L, w.k)
    # records travel as fp32: m exact to fp32, s to fp32 rounding
    assert np.allclose(M, fm, rtol=1e-6) and np.allclose(S, fs, rtol=1e-5)
    assert np.array_equal(v, fv)


@pytest.mark.parametrize("V,world", [(90000, 8), (90000, 3), (1000, 4), (17, 8)])
def test_shard_range_partition(V, world):
    from paper_1805_09863_b200.sharded import shard_range
    r = [shard_range(V, world, g) for g in range(world)]
    covered = [x for a, b in r for x in range(a, b)]
    assert covered == list(range(V))
    assert all(a % 16 == 0 for a, b in r if b > a)


class _FakeBuffers:
    """Stands in for the library's one-shot buffer calls (no GPU here): the
    'pointer' of rank r's buffer is 0x1000 * (r + 1), its 64-byte handle
    encodes r, opening a handle yields 0x100000 + that pointer."""

    def __init__(self, rank):
        self.rank, self.log = rank, []

    def alloc(self, plan, world):
        self.log.append(("alloc", world))
        return 0x1000 * (self.rank + 1), bytes([self.rank]) * 64

    def open(self, handle, device):
        assert len(handle) == 64 and len(set(handle)) == 1
        self.log.append(("open", handle[0]))
        return 0x100000 + 0x1000 * (handle[0] + 1)

    def close(self, ptr):
        self.log.append(("close", ptr))

    def free(self, ptr):
        self.log.append(("free", ptr))


def _oneshot_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_09863_b200.sharded import OneShotExchange
    fake = _FakeBuffers(rank)
    ex = OneShotExchange(None, world, rank, 0, lib=fake)
    ptrs = list(ex.ptrs)
    ex.close()
    q.put((rank, ptrs, fake.log))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_oneshot_handle_exchange(world):
    """OneShotExchange (NEXT f3 host logic) over gloo: every rank ends with
    the rank-ordered buffer list, its own allocation at its own index and
    every peer's buffer opened from that peer's handle; close() unmaps the
    peers and frees the own buffer."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oneshot_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = dict((r, (ptrs, log)) for r, ptrs, log in (q.get(timeout=10) for _ in range(world)))
    for r in range(world):
        ptrs, log = got[r]
        assert ptrs == [0x1000 * (p + 1) if p == r else 0x100000 + 0x1000 * (p + 1)
                        for p in range(world)]
        assert log[0] == ("alloc", world)
        assert sorted(e[1] for e in log if e[0] == "open") == [p for p in range(world) if p != r]
        assert log[-1] == ("free", 0x1000 * (r + 1))
        assert len([e for e in log if e[0] == "close"]) == world - 1
