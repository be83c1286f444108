"""The N>1 sweep path on CPU: world_size-2 gloo processes shard
the points, run them (kernel core under the SIMT emulator) and gather the
summaries to rank 0; the merge must be byte-identical to a single-process
run (results independent of the GPU count)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _points():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from configs import random_small
    return [random_small(3000 + i, max_req=40) for i in range(12)]


def _run_emu(points):
    from harness import run_points_emu
    return [r.summary for r in run_points_emu(points, ev_cap=0, recs=False, warps=2)]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from paper_2411_05555_b200.sweep import pack, run_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    merged = run_sharded(_points(), _run_emu, dist)
    if rank == 0:
        with open(out_path, "wb") as f:
            f.write(pack(merged))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_merge_matches_single(tmp_path):
    from paper_2411_05555_b200.sweep import pack, shard_indices
    assert shard_indices(5, 0, 2) == [0, 2, 4] and shard_indices(5, 1, 2) == [1, 3]
    out = str(tmp_path / "merged.bin")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    single = pack(_run_emu(_points()))
    assert open(out, "rb").read() == single
