"""Fused summary exchange (include/bellman_sim.h bellman_sim_set_peers, SURVEY
§8(e)): two ranks — two processes sharing cuda:0, a gloo group for the handle
exchange — each simulate their interleaved shard while the tick kernel stores
every finished record into both ranks' full-size arrays through CUDA IPC
mappings.  After the runs every rank's array must equal, byte for byte, a
single whole-set run; the workspace copy (bellman_sim_stats) stays the shard's.
On the 8-GPU box the same mapping goes over NVLink / NVSwitch."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _workload():
    import workloads as W

    return W.config_c2(n_seeds=4, rates=[0.5, 2.0, 4.0, 8.0])


def _rank_main(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2510_15330_b200 import Simulator, _abi
    from paper_2510_15330_b200 import parallel as PAR

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = _workload()
    n = w.n_scenarios
    sim = Simulator(w.columns(), device=0)
    full = torch.zeros((n, _abi.STATS.itemsize), dtype=torch.uint8, device="cuda:0")
    peers = PAR.PeerRecords(full, rank, world, 0)
    sim.set_peers(peers.ptrs)
    for _ in range(2):  # the second run rewrites every record: idempotent
        dist.barrier()
        sim.run(first=rank, count=PAR.shard_count(n, rank, world), stride=world)
        torch.cuda.synchronize()
        dist.barrier()
    np.save(os.path.join(outdir, f"full{rank}.npy"), full.cpu().numpy())
    np.save(os.path.join(outdir, f"own{rank}.npy"), sim.stats().view(np.uint8).reshape(n, -1))
    dist.barrier()
    peers.close()
    sim.set_peers([])
    dist.destroy_process_group()


@pytest.mark.parametrize("engine", ["warp", "lane"])
def test_fused_exchange_two_ranks_one_gpu(tmp_path, monkeypatch, engine):
    """Both engines store the records to the peers: the warp kernels (the default
    at this size) and K2L (BELLMAN_LANE=2, inherited by the spawned ranks)."""
    import torch
    import torch.multiprocessing as mp

    from paper_2510_15330_b200 import Simulator

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    monkeypatch.setenv("BELLMAN_LANE", "2" if engine == "lane" else "0")
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    w = _workload()
    ref = Simulator(w.columns(), device=0)
    ref.run()
    torch.cuda.synchronize()
    assert (ref.last_engines & 0x18) != 0 if engine == "lane" else ref.last_engines == 1
    want = ref.stats().view(np.uint8).reshape(w.n_scenarios, -1)
    for r in range(2):
        got = np.load(tmp_path / f"full{r}.npy")
        assert np.array_equal(got, want), f"rank {r}: fused exchange differs from a single run"
        own = np.load(tmp_path / f"own{r}.npy")
        mine = np.arange(r, w.n_scenarios, 2)
        assert np.array_equal(own[mine], want[mine])
        others = np.setdiff1d(np.arange(w.n_scenarios), mine)
        assert not own[others].any()  # the workspace copy holds the shard only


def test_set_peers_local_arrays_and_validation():
    """One process, two local record arrays as 'peers': both receive every
    record of the run, equal to bellman_sim_stats; argument validation."""
    import torch

    from paper_2510_15330_b200 import BellmanError, Simulator, _abi

    w = _workload()
    n = w.n_scenarios
    sim = Simulator(w.columns(), device=0)
    a = torch.zeros((n, _abi.STATS.itemsize), dtype=torch.uint8, device="cuda:0")
    b = torch.zeros_like(a)
    sim.set_peers([a.data_ptr(), b.data_ptr()])
    sim.run()
    torch.cuda.synchronize()
    want = sim.stats().view(np.uint8).reshape(n, -1)
    assert np.array_equal(a.cpu().numpy(), want) and np.array_equal(b.cpu().numpy(), want)
    sim.set_peers([])  # off: later runs leave the arrays alone
    a.zero_()
    sim.run()
    torch.cuda.synchronize()
    assert not a.any()
    with pytest.raises(BellmanError, match="n_peers"):
        sim.set_peers([a.data_ptr()] * 9)
    with pytest.raises(BellmanError, match="aligned"):
        sim.set_peers([a.data_ptr() + 4])
