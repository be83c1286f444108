"""Bulk trace ingestion (reference SPEC.md:164-172,185):
`kvsim` parses `#kvsim-trace v1` files with all host threads into page-locked
buffers (kvsim_gpu_host_alloc). Checked on CPU through `validate-config`'s
trace_summary: every value must equal what a sequential, correctly rounded
parse (Python float()) gives, and errors must name the first bad line in file
order wherever the parallel chunk seams fall."""
import json
import random
import struct

import pytest

from test_cli import kvsim, run, write  # noqa: F401  (fixture)


def fnv1a(values):
    h = 1469598103934665603
    for v in values:
        for byte in struct.pack("<d", v):
            h = ((h ^ byte) * 1099511628211) & (2**64 - 1)
    return f"{h:016x}"


def make_trace(n, seed, crlf_every=7, comment_every=1000):
    r = random.Random(seed)
    t = 0.0
    rows, arr, pl, dl = ["#kvsim-trace v1", "id,arrival_s,prompt_len,decode_len"], [], [], []
    for i in range(n):
        t += r.expovariate(3.0)
        # mixed spellings: shortest repr, fixed 9 digits, 17 significant digits
        s = [repr(t), f"{t:.9f}", f"{t:.17g}"][i % 3]
        a = float(s)
        arr.append(a)
        p, d = r.randint(1, 8000), r.randint(1, 2000)
        pl.append(p)
        dl.append(d)
        rows.append(f"{i},{s},{p},{d}" + ("\r" if i % crlf_every == 0 else ""))
        if comment_every and i % comment_every == comment_every - 1:
            rows.append("# comment")
            rows.append("")
    return rows, arr, pl, dl


def summary(kvsim, tmp_path, rows):
    tr = tmp_path / "t.csv"
    tr.write_text("\n".join(rows) + "\n")
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "c.json", {"trace": str(tr), "instances": 2}))
    return r


def test_bulk_values_match_sequential_parse(kvsim, tmp_path):
    rows, arr, pl, dl = make_trace(250_000, 1)  # ~8 MB: several parser threads
    r = summary(kvsim, tmp_path, rows)
    assert r.returncode == 0, r.stderr
    ts = json.loads(r.stdout)["trace_summary"]
    assert ts["rows"] == len(arr)
    assert ts["prompt_tokens"] == sum(pl) and ts["decode_tokens"] == sum(dl)
    assert ts["arrival_fnv1a"] == fnv1a(arr)


def test_small_trace_and_no_trailing_newline(kvsim, tmp_path):
    tr = tmp_path / "t.csv"
    tr.write_text("#kvsim-trace v1\n0,0.1,5,3\n1, 0.25,+7,4")
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "c.json", {"trace": str(tr), "instances": 2}))
    assert r.returncode == 0, r.stderr
    ts = json.loads(r.stdout)["trace_summary"]
    assert ts["rows"] == 2 and ts["prompt_tokens"] == 12 and ts["arrival_fnv1a"] == fnv1a([0.1, 0.25])


@pytest.mark.parametrize("frac", [0.0, 0.13, 0.37, 0.5, 0.71, 0.999])
def test_first_error_in_file_order(kvsim, tmp_path, frac):
    rows, arr, _, _ = make_trace(200_000, 2, comment_every=0)
    k = 2 + int(frac * 199_999)  # index into rows (line number k + 1)
    i = k - 2
    # arrival decreases at row i (line k + 1); a later parse error must not win
    prev = arr[i - 1] if i > 0 else 0.0
    rows[k] = f"{i},{prev / 2 if i > 0 else -1.0},10,10"
    if i == 0:
        rows[k + 1] = "garbage"  # row 0 cannot decrease: check the parse error instead
        want = f"t.csv:{k + 2}: parse error"
    else:
        want = f"t.csv:{k + 1}: arrival_s decreases"
    rows[-5] = "1,2,3"
    r = summary(kvsim, tmp_path, rows)
    assert r.returncode == 2 and want in r.stderr, (r.returncode, r.stderr[:300])


def test_errors_name_the_line(kvsim, tmp_path):
    base = ["#kvsim-trace v1", "0,0.5,10,5", "1,0.6,10,5"]
    for bad, msg in [("2,0.7,0,5", "lengths out of range"), ("3,0.7,10,5", "ids must be 0..n-1 in order"),
                     ("2,nan,10,5", "arrival_s must be finite"), ("2,0.7,10,5,9", "parse error"),
                     ("2,0.7,10,5 ", "parse error")]:
        r = summary(kvsim, tmp_path, base + [bad, "3,0.8,10,5"])
        assert r.returncode == 2 and f"t.csv:4: {msg}" in r.stderr, (bad, r.stderr)
    r = summary(kvsim, tmp_path, ["#kvsim-trace v2", "0,0.5,10,5"])
    assert r.returncode == 2 and "t.csv:1: missing '#kvsim-trace v1' header" in r.stderr
