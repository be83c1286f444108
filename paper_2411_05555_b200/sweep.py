"""Multi-GPU sweep orchestration (host side).

Sweep points are independent (reference SPEC.md:267,446-448), so a sweep is
sharded over ranks with no data-path collective: rank r takes points
r, r+W, r+2W, ... (strided, so the rate-sorted grid spreads its cost evenly),
runs them on its own GPU through the C-ABI, and the per-point summaries
(~300 B each) are gathered to rank 0 and placed by point index. The merged
result is therefore bit-identical for any world size.

One process per GPU; torch.distributed is only the control plane (gather of
summaries). With the NCCL backend the gather goes through a device tensor;
with gloo (CPU tests) through a host tensor.
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


def run_sharded(points: Sequence[PointDesc], run_fn: Callable[[list], list], dist=None, device=None):
    """Run `points` sharded over the process group; returns the merged list of
    summaries on rank 0 (None on other ranks). run_fn(points) -> summaries."""
    import torch
    if dist is None or not dist.is_initialized():
        return list(run_fn(list(points)))
    rank, world = dist.get_rank(), dist.get_world_size()
    idx = shard_indices(len(points), rank, world)
    local = run_fn([points[i] for i in idx]) if idx else []
    payload = torch.frombuffer(bytearray(pack(local) or b"\0"), dtype=torch.uint8)
    n_max = (len(points) + world - 1) // world
    buf = torch.zeros(n_max * SUMMARY_BYTES, dtype=torch.uint8)
    buf[:len(local) * SUMMARY_BYTES] = payload[:len(local) * SUMMARY_BYTES]
    if device is not None:
        buf = buf.to(device)
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    if rank != 0:
        return None
    out: list = [None] * len(points)
    for r in range(world):
        ridx = shard_indices(len(points), r, world)
        got = unpack(bufs[r].cpu().numpy().tobytes()[:len(ridx) * SUMMARY_BYTES])
        for i, s in zip(ridx, got):
            out[i] = s
    return out
