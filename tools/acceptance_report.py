"""Print the SPEC acceptance table (docs/SEMANTICS.md §9) from the CPU oracle
at the SPEC setups (tests/acceptance.py). Test infrastructure: the numbers are
the oracle's; tests/test_gpu_acceptance.py shows the B200 kernels produce the
same summaries bit for bit."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import acceptance as A  # noqa: E402
from harness import oracle_sweep, run_oracle  # noqa: E402


def main():
    out = {}
    pts = A.a3_points(); s, _ = oracle_sweep(pts, detail=True, instances=False); out["3"] = A.a3_eval(pts, s)
    pts = A.a5_points(); s, _ = oracle_sweep(pts, instances=False); out["5"] = A.a5_eval(pts, s)
    pts = A.a7_points(); s, i = oracle_sweep(pts); out["7"] = A.a7_eval(pts, s, i)
    pts = A.a8_points()
    out["8"] = A.a8_eval(pts, [run_oracle(p, ev_cap=1 << 22, recs=False, inst=False).events for p in pts])
    pts = A.a9_points(); s, _ = oracle_sweep(pts, instances=False); out["9"] = A.a9_eval(pts, s)
    pts = A.a10_points(); s, _ = oracle_sweep(pts, instances=False); out["10"] = A.a10_eval(pts, s)
    json.dump(out, sys.stdout, indent=1, default=float)


if __name__ == "__main__":
    main()
