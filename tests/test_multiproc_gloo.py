"""The N>1 path on CPU: world_size-2 gloo processes shard a workload by
interleaving, compute their records (oracle stand-in for the kernel: this tests
the sharding and the exchange, not the simulation), gather them with
paper_2510_15330_b200.parallel and reduce segment histograms; the gathered
result must equal the single-process result byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _records(cols, ids):
    import oracle

    b = oracle.Bound(cols)
    recs = np.zeros((len(ids), 34), dtype=np.uint64)  # 272 B = 34 u64 words
    seg = np.zeros((int(cols["n_segments"]), 3), dtype=np.int64)
    for i, sid in enumerate(ids):
        r = oracle.run_scenario(b, int(sid))
        recs[i, 0] = sid
        recs[i, 1] = r["ticks"]
        recs[i, 2] = r["served"]
        recs[i, 3] = r["words_out"]
        recs[i, 4] = np.float64(r["energy_j"]).view(np.uint64)
        s = cols["sc_segment"][sid]
        seg[s] += [r["served"], r["ticks"], r["rewritten"]]
    return recs, seg


def _worker(rank, world, port, cols, q):
    from paper_2510_15330_b200 import parallel as P

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = len(cols["sc_seed"])
    ids = W.shard(n, rank, world)
    recs, seg = _records(cols, ids)
    local = torch.from_numpy(recs.view(np.uint8).reshape(len(ids), 272).copy())
    full = P.gather_summaries(local, n, rank, world)
    segt = P.reduce_segments(torch.from_numpy(seg))
    if rank == 0:
        q.put((full.numpy().copy(), segt.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_matches_single_process(world):
    cols = W.config_c2(n_seeds=3, rates=[1.0, 4.0], horizon_s=60).columns()  # 12 scenarios, not divisible by 8
    n = len(cols["sc_seed"])
    want, want_seg = _records(cols, np.arange(n))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, seg = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(full.view(np.uint64).reshape(n, 34), want)
    assert np.array_equal(seg, want_seg)


def test_gather_reorder_uneven():
    """Reordering logic for n not divisible by world (no process group needed)."""
    for n, world in ((7, 2), (10, 3), (5, 8)):
        m = (n + world - 1) // world
        gathered = np.full((world * m,), -1)
        for r in range(world):
            ids = list(range(r, n, world))
            gathered[r * m: r * m + len(ids)] = ids
        full = gathered.reshape(world, m).T.reshape(-1)[:n]
        assert list(full) == list(range(n))


def _peer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_15330_b200 import parallel as PAR

    opened = []

    def export(ptr):  # a fake IPC handle naming the exporting rank and its base
        return (f"rank{rank}".encode(), ptr - 0x1000 * (rank + 1))

    def open_(hb, off):
        g = int(hb.decode()[4:])
        base = 0x7000_0000 + g
        opened.append((g, off))
        return base, base + off

    local = 0x1000 * (rank + 1) + 0x40  # "device pointer" of this rank's array
    ptrs, bases = PAR.exchange_peer_pointers(local, rank, world, export, open_)
    q.put((rank, ptrs, bases, opened))
    dist.destroy_process_group()


def test_peer_pointer_exchange_gloo():
    """Host side of the fused exchange at world size 3 over gloo (fake IPC):
    every rank gets one pointer per rank in rank order, its own array at its
    own index, and maps each other rank's export exactly once at its offset."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        r, ptrs, bases, opened = q.get(timeout=120)
        got[r] = (ptrs, bases, opened)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (ptrs, bases, opened) in got.items():
        assert len(ptrs) == world and len(bases) == world - 1
        assert ptrs[r] == 0x1000 * (r + 1) + 0x40
        assert sorted(g for g, _ in opened) == [g for g in range(world) if g != r]
        for g in range(world):
            if g != r:
                assert ptrs[g] == 0x7000_0000 + g + 0x40  # base + the exporter's offset


def _peer_fail_worker(rank, world, port, q, fail_export, fail_open):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_15330_b200 import parallel as PAR

    opened, closed = [], []

    def export(ptr):
        if rank == fail_export:
            raise RuntimeError("no IPC here")
        return (f"rank{rank}".encode(), 0x40)

    def open_(hb, off):
        g = int(hb.decode()[4:])
        if rank == fail_open and len(opened) == 1:  # the second mapping fails
            raise RuntimeError("peer access refused")
        opened.append(0x7000_0000 + g)
        return 0x7000_0000 + g, 0x7000_0000 + g + off

    try:
        PAR.exchange_peer_pointers(0x1040, rank, world, export, open_, closed.append)
        outcome = "ok"
    except PAR.PeerExchangeError:
        outcome = "raised"
    dist.barrier()  # every rank reached the same point: no collective left unmatched
    q.put((rank, outcome, opened, closed))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_export,fail_open", [(1, -1), (-1, 2), (0, 2)])
def test_peer_pointer_exchange_failure_is_collective(fail_export, fail_open):
    """a failed export or a failed mapping on ONE rank makes EVERY
    rank raise PeerExchangeError after the same collectives (no hang, no
    mismatched all_gather), and every mapping already opened is unmapped."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_fail_worker, args=(r, world, port, q, fail_export, fail_open))
          for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    for _ in range(world):
        r, outcome, opened, closed = q.get(timeout=120)
        got[r] = (outcome, opened, closed)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (outcome, opened, closed) in got.items():
        assert outcome == "raised", (r, outcome)
        assert sorted(closed) == sorted(opened), (r, opened, closed)
