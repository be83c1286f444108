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


def test_sharder_worker_count_invariance():
    """The multi-device sharder (kvsim_shard.hpp: guided chunks over the
    cost-sorted points, results scattered by index) with 1-4 emulated
    devices: byte-identical summaries, every worker used."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from harness import emu
    from paper_2411_05555_b200.abi import PointDesc, PointSummary
    L = emu()
    L.kvemu_run_multi.argtypes = [C.POINTER(PointDesc), C.c_int64, C.c_int, C.c_int64, C.POINTER(PointSummary),
                                  C.POINTER(C.c_int64)]
    pts = _points() + [p for p in _points()]
    P = (PointDesc * len(pts))(*pts)
    outs = []
    for w in (1, 2, 3, 4):
        S = (PointSummary * len(pts))()
        per = (C.c_int64 * w)()
        assert L.kvemu_run_multi(P, len(pts), w, 1, S, per) == 0
        assert sum(per) == len(pts) and min(per) > 0
        outs.append(b"".join(bytes(s) for s in S))
    assert all(o == outs[0] for o in outs)


def test_sharder_static_lpt_mode():
    """Few points per device: one launch per worker, points dealt by greedy
    LPT (kvsim_shard.hpp make_static); results identical to one worker."""
    import ctypes as C
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from harness import emu
    from paper_2411_05555_b200.abi import PointDesc, PointSummary
    L = emu()
    L.kvemu_run_multi.argtypes = [C.POINTER(PointDesc), C.c_int64, C.c_int, C.c_int64, C.POINTER(PointSummary),
                                  C.POINTER(C.c_int64)]
    pts = _points()
    P = (PointDesc * len(pts))(*pts)
    outs = []
    for w in (1, 3):
        S = (PointSummary * len(pts))()
        per = (C.c_int64 * w)()
        assert L.kvemu_run_multi(P, len(pts), w, 0, S, per) == 0  # min_chunk 0: static LPT deal
        assert sum(per) == len(pts)
        outs.append(b"".join(bytes(s) for s in S))
    assert outs[0] == outs[1]
