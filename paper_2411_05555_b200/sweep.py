"""Multi-GPU sweep orchestration (host side).

Sweep points are independent (reference SPEC.md:267,446-448), so a sweep is
sharded over ranks with no data-path collective: rank r takes points
r, r+W, r+2W, ... (strided, so the rate-sorted grid spreads its cost evenly),
runs them on its own GPU through the C-ABI, and the per-point summaries
(~300 B each) are gathered to rank 0 and placed by point index. The merged
result is therefore bit-identical for any world size.

One process per GPU; torch.distributed is only the control plane: the
summaries are gathered in host memory over a gloo group (a gloo subgroup is
created when the default group is NCCL), never through NCCL or device
memory. The single-process alternative is kvsim_gpu_run_multi (one host
thread per GPU, csrc/kvsim_shard.hpp), which bench.py and the kvsim CLI use.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

from .abi import PointDesc, PointSummary

SUMMARY_BYTES = C.sizeof(PointSummary)


def shard_indices(n: int, rank: int, world: int) -> list[int]:
    return list(range(rank, n, world))


def pack(summaries: Sequence[PointSummary]) -> bytes:
    return b"".join(bytes(s) for s in summaries)


def unpack(buf: bytes) -> list[PointSummary]:
    n = len(buf) // SUMMARY_BYTES
    arr = (PointSummary * n).from_buffer_copy(buf[:n * SUMMARY_BYTES])
    return list(arr)


_GLOO = None


def _host_group(dist):
    """The group the gather runs on: the default group if it is gloo, else a
    gloo subgroup over all ranks (host memory, no NCCL)."""
    global _GLOO
    if dist.get_backend() == "gloo":
        return None
    if _GLOO is None:
        _GLOO = dist.new_group(backend="gloo")
    return _GLOO


def run_sharded(points: Sequence[PointDesc], run_fn: Callable[[list], list], dist=None):
    """Run `points` sharded over the process group; returns the merged list of
    summaries on rank 0 (None on other ranks). run_fn(points) -> summaries."""
    import torch
    if dist is None or not dist.is_initialized():
        return list(run_fn(list(points)))
    rank, world = dist.get_rank(), dist.get_world_size()
    group = _host_group(dist)
    idx = shard_indices(len(points), rank, world)
    local = run_fn([points[i] for i in idx]) if idx else []
    payload = torch.frombuffer(bytearray(pack(local) or b"\0"), dtype=torch.uint8)
    n_max = (len(points) + world - 1) // world
    buf = torch.zeros(n_max * SUMMARY_BYTES, dtype=torch.uint8)
    buf[:len(local) * SUMMARY_BYTES] = payload[:len(local) * SUMMARY_BYTES]
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    if rank != 0:
        return None
    out: list = [None] * len(points)
    for r in range(world):
        ridx = shard_indices(len(points), r, world)
        got = unpack(bufs[r].numpy().tobytes()[:len(ridx) * SUMMARY_BYTES])
        for i, s in zip(ridx, got):
            out[i] = s
    return out
