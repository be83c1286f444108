"""The reference's C++ perfmodel API (include/kvsim/perfmodel.hpp, signature-
identical to reference proj/include/kvsim/perfmodel.hpp:23-123) called from
a C++ program linked against the product library: SPEC worked examples and
the declared exceptions through the kvsim:: span signatures. Host code only
(no GPU needed)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_perfmodel_cpp_client(tmp_path):
    from paper_2411_05555_b200 import build
    lib = build.build_cuda()
    exe = tmp_path / "perfmodel_api"
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "perfmodel_api.cpp"), "-o", str(exe),
                    "-L" + os.path.dirname(lib), "-lkvsim_gpu", "-Wl,-rpath," + os.path.dirname(lib)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "perfmodel_api: ok" in r.stdout
