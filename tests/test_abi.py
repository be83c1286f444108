"""The product library loads without a GPU, exports every symbol declared in
include/kvsim_gpu.h, validates points on the host, and refuses to run (no CPU
fallback) when no device is visible."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

import paper_2411_05555_b200 as pkg
from paper_2411_05555_b200.abi import make_point

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kvsim_gpu.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|int64_t)\s+(kvsim_[a-z0-9_]+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_05555_b200 import build
    build.build_cuda()
    return pkg.load_library()


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s


def test_struct_sizes_match_header(lib):
    src = r'''
#include <stdio.h>
#include "kvsim_gpu.h"
int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(kvsim_point_desc), sizeof(kvsim_point_summary),
  sizeof(kvsim_request_record), sizeof(kvsim_event_record), sizeof(kvsim_trace_view),
  sizeof(kvsim_instance_record), sizeof(kvsim_run_opts), sizeof(kvsim_multi_stats));}
'''
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "s.c"), "w").write(src)
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), os.path.join(d, "s.c"), "-o",
                        os.path.join(d, "s")], check=True)
        out = subprocess.run([os.path.join(d, "s")], capture_output=True, text=True).stdout.split()
    want = [C.sizeof(pkg.PointDesc), C.sizeof(pkg.PointSummary), C.sizeof(pkg.RequestRecord),
            C.sizeof(pkg.EventRecord), C.sizeof(pkg.TraceView), C.sizeof(pkg.InstanceRecord),
            C.sizeof(pkg.RunOpts), C.sizeof(pkg.MultiStats)]
    assert [int(x) for x in out] == want


def test_host_validation(lib):
    err = C.create_string_buffer(256)
    assert lib.kvsim_point_validate(C.byref(make_point()), err, 256) == 0
    assert lib.kvsim_point_validate(C.byref(make_point(policy="accellm", instances=5)), err, 256) == -3
    assert b"even instance count required" in err.value
    p = make_point(device=(1e12, 10e9, 1e12, 1e9))
    assert lib.kvsim_point_validate(C.byref(p), err, 256) == -2
    assert b"model does not fit in instance memory" in err.value
    d = make_point()
    lib.kvsim_point_defaults(C.byref(d))
    assert d.num_layers == 80 and d.compute_eff == 0.5 and d.prefill_token_budget == 8192


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU visible")
    assert lib.kvsim_gpu_device_count() == 0
    with pytest.raises(pkg.KvSimError):
        pkg.KvSim(0)


def test_pinned_host_buffers(lib):
    # kvsim_gpu_host_alloc: page-locked memory for bulk trace ingestion, NULL
    # without a device (callers then use ordinary memory); free(NULL) is a no-op
    import ctypes as C
    import torch
    lib.kvsim_gpu_host_alloc.restype = C.c_void_p
    lib.kvsim_gpu_host_alloc.argtypes = [C.c_size_t]
    lib.kvsim_gpu_host_free.argtypes = [C.c_void_p]
    lib.kvsim_gpu_host_free(None)
    assert lib.kvsim_gpu_host_alloc(0) is None
    p = lib.kvsim_gpu_host_alloc(1 << 20)
    if not torch.cuda.is_available():
        assert p is None
    else:
        assert p is not None
        C.memset(p, 7, 1 << 20)
        lib.kvsim_gpu_host_free(p)
