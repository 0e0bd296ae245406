"""Scenario sharding and the single exchange step.

Scenarios are independent units: rank r of W simulates ids r, r+W, r+2W, ...
(interleaving puts every (rate, controller) cell on every rank, which balances
per-tick cost).  The only collective is at the end of a step: all_gather of
the 272-byte summary records (NCCL over NVLink on GPUs, gloo in CPU tests)
and an all_reduce(SUM) of the integer segment histograms.  Integer sums are
order-independent, so results are bit-identical for any world size.

On GPUs the record all-gather can instead be fused into the simulation
kernel (`PeerRecords` + `Simulator.set_peers`): every rank maps every other
rank's full-size record array into its process (CUDA IPC over NVLink /
NVSwitch, through the library's bellman_ipc_* calls) and the tick kernel
stores each record into all of them as it finishes the scenario, so the
exchange overlaps the simulation; only the segment-histogram sum stays a
collective.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

REC = 272  # bytes per bellman_scenario_stats


def shard_count(n: int, rank: int, world: int) -> int:
    return len(range(rank, n, world))


def shard_rows(full_rows: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's records (ids rank, rank+world, ...) as a contiguous block."""
    return full_rows[rank::world].contiguous()


def gather_summaries(local: torch.Tensor, n: int, rank: int, world: int, out: torch.Tensor | None = None):
    """All-gather every rank's (count_r, REC) uint8 record block and return the
    (n, REC) records in scenario-id order (on every rank)."""
    if world == 1:
        return local[:n]
    m = (n + world - 1) // world
    buf = torch.zeros((m, REC), dtype=torch.uint8, device=local.device)
    buf[: local.shape[0]] = local
    gathered = torch.empty((world * m, REC), dtype=torch.uint8, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(gathered, buf)
    else:
        parts = list(gathered.chunk(world))
        dist.all_gather(parts, buf)
        gathered = torch.cat(parts)
    full = gathered.view(world, m, REC).transpose(0, 1).reshape(world * m, REC)[:n]
    if out is not None:
        out.copy_(full)
        return out
    return full


def reduce_segments(seg: torch.Tensor) -> torch.Tensor:
    """Sum the int64 segment histograms over ranks (in place)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(seg, op=dist.ReduceOp.SUM)
    return seg


class PeerExchangeError(RuntimeError):
    """The fused exchange could not be set up on some rank (raised on every rank)."""


def _agree(ok: bool, world: int) -> list:
    """Every rank's flag, on every rank (one all_gather_object)."""
    flags = [None] * world
    if world > 1:
        dist.all_gather_object(flags, ok)
    else:
        flags = [ok]
    return flags


def exchange_peer_pointers(local_ptr: int, rank: int, world: int, export, open_, close=None) -> tuple:
    """Host side of the fused exchange: export this rank's array (export(ptr)
    -> (handle bytes, offset)), all-gather the (handle, offset) pairs over the
    process group, and map every other rank's (open_(handle, offset) -> (base,
    ptr)).  Returns (ptrs, bases): ptrs[g] is rank g's array as seen here
    (ptrs[rank] = local_ptr), bases the mappings to unmap later.

    Collective-safe: every rank joins the same two all_gather_object calls
    whatever fails locally (a failed export sends None), and if the export or
    any mapping failed on ANY rank, every rank unmaps what it opened (close(base))
    and raises PeerExchangeError — all ranks take the same path.  Pure host
    logic, so it is tested with fake export/open callables over gloo."""
    err = None
    try:
        mine = export(local_ptr)
    except Exception as e:  # noqa: BLE001 — reported collectively below
        mine, err = None, f"rank {rank} export: {type(e).__name__}: {e}"
    allh = [None] * world
    if world > 1:
        dist.all_gather_object(allh, mine)
    else:
        allh = [mine]
    ptrs, bases = [], []
    if all(h is not None for h in allh):
        try:
            for g, (hb, o) in enumerate(allh):
                if g == rank:
                    ptrs.append(local_ptr)
                    continue
                base, ptr = open_(hb, o)
                bases.append(base)
                ptrs.append(ptr)
        except Exception as e:  # noqa: BLE001
            err = f"rank {rank} open: {type(e).__name__}: {e}"
    else:
        err = err or "export failed on rank(s) " + ",".join(str(g) for g, h in enumerate(allh) if h is None)
    flags = _agree(err is None, world)
    if not all(flags):
        if close is not None:
            for b in bases:
                try:
                    close(b)
                except Exception:  # noqa: BLE001 — best effort unmapping on the failure path
                    pass
        bad = [g for g, f in enumerate(flags) if not f]
        raise PeerExchangeError(err or f"peer exchange failed on rank(s) {bad}")
    return ptrs, bases


class PeerRecords:
    """Every rank's full-size (n, REC) record array, mapped into this process.

    `local` is this rank's array (a CUDA tensor, 16-byte aligned); the IPC
    handle of its allocation is exchanged over the process group and each
    other rank's array is opened on `device` (`exchange_peer_pointers` with the
    library's bellman_ipc_export / bellman_ipc_open).  `ptrs[g]` is rank g's
    array as a device pointer valid here (rank == g: local itself).  Raises
    PeerExchangeError on every rank if any rank fails."""

    def __init__(self, local: torch.Tensor, rank: int, world: int, device: int):
        from . import _abi as A

        assert local.is_cuda and local.is_contiguous() and local.data_ptr() % 16 == 0
        self.local = local
        L = A.lib()

        def export(ptr):
            h = (C.c_uint8 * 64)()
            off = C.c_uint64()
            A.check(L.bellman_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
            return bytes(h), int(off.value)

        def open_(hb, o):
            base, ptr = C.c_void_p(), C.c_void_p()
            hh = (C.c_uint8 * 64).from_buffer_copy(hb)
            A.check(L.bellman_ipc_open(hh, o, device, C.byref(base), C.byref(ptr)))
            return base.value, ptr.value

        def close(b):
            L.bellman_ipc_close(C.c_void_p(b))

        self.ptrs, self.bases = exchange_peer_pointers(local.data_ptr(), rank, world, export, open_, close)

    def close(self):
        from . import _abi as A

        for b in self.bases:
            A.lib().bellman_ipc_close(C.c_void_p(b))
        self.bases, self.ptrs = [], []


def open_peer_records(local: torch.Tensor, rank: int, world: int, device: int):
    """(PeerRecords, None) if every rank mapped every peer array, else
    (None, reason) on every rank (the caller falls back to the NCCL all-gather)."""
    try:
        return PeerRecords(local, rank, world, device), None
    except PeerExchangeError as e:
        return None, str(e)[:200]
