"""Event mix of the kernel core on the SIMT emulator (exploratory): builds a
profiling emulator (KVSIM_EMU_PROFILE) into /tmp, runs a config-4 subsample
(every k-th rate, N requests) and prints the EMU_COUNT call counters per
simulated request; also checks the summaries against the oracle.
usage: python tools/emu_mix.py POLICY [RATE_STRIDE] [REQUESTS] [extra g++ flags...]"""
import ctypes as C, os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import harness
from bench import config4_points
pol = sys.argv[1] if len(sys.argv) > 1 else "accellm"
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 83
nreq = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
so = "/tmp/libkvsim_emu_prof.so"
subprocess.run(["g++", "-DKVSIM_EMU", "-DKVSIM_EMU_PROFILE", "-O2", "-std=gnu++20", "-ffp-contract=off", "-fPIC",
                "-shared", "-I" + os.path.join(R, "include"), *sys.argv[4:], "-o", so,
                os.path.join(R, "tests", "emu", "kvsim_emu.cpp"), "-lpthread"], check=True)
harness.EMU_SO = so
harness.build_emu = lambda: None
pts = [p for i, p in enumerate(config4_points(0, 833, nreq, policies=(pol,))) if i % stride == 0]
got = harness.run_points_emu(pts, ev_cap=0, recs=False, warps=8)
bad = 0
for p, g in zip(pts, got):
    ref = harness.run_oracle(p, ev_cap=0, recs=False)
    if harness.diff_results(ref, g):
        bad += 1
L = harness.emu()
prof = (C.c_longlong * 32)()
L.kvemu_prof(prof)
reqs = sum(g.summary.n_requests for g in got)
print(f"{pol}: {len(pts)} points, {reqs} requests, oracle mismatches {bad}")
for i in range(32):
    if prof[i]:
        print(f"  counter {i:2d}: {prof[i]:12d}  {prof[i] / reqs:9.3f} per request")
