"""Attribute an ncu source-page capture of kvsim_sweep_kernel<MINB[, FULL]> to kvsim_sim.cuh
functions (instructions executed, warp-stall samples, no_instruction stalls).

  ncu -i REPORT --page source --csv --print-source sass > sass.csv
  cuobjdump -xelf all paper_2411_05555_b200/_build/libkvsim_gpu.so
  nvdisasm -g -c kvsim_sweep.sm_100a.cubin > dis.txt
  python tools/ncu_attribute.py sass.csv dis.txt paper_2411_05555_b200/csrc/kvsim_sim.cuh

The SASS offsets in sass.csv are matched to the line table of the same build.
"""
import collections, csv, re, sys


def main(sass_csv, dis_txt, sim_cuh):
    rows = list(csv.reader(open(sass_csv)))
    m = re.search(r"kvsim_sweep_kernel<\(int\)(\d+)(?:, \(bool\)(\d))?>", rows[0][1])
    minb, full = m.group(1), m.group(2)
    tag = f"ILi{minb}EE" if full is None else f"ILi{minb}ELb{full}EE"
    dis = open(dis_txt).read().split("\n")
    start = [i for i, l in enumerate(dis) if l.startswith(".text._Z18kvsim_sweep_kernel" + tag)][0]
    off2src, cur = {}, None
    for l in dis[start:]:
        if l.startswith("//----") and tag not in l:
            break
        m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s", l)
        if m:
            off2src[int(m.group(1), 16)] = cur
    funcs = []
    for i, l in enumerate(open(sim_cuh), 1):
        m = re.match(r"\s+KV_DEV\w* [\w:<>,\* &]+?\b(\w+)\(", l)
        if m:
            funcs.append((i, m.group(1)))

    def fn(src):
        if src is None:
            return "?"
        f, ln = src
        if f != "kvsim_sim.cuh":
            return f
        name = "hdr"
        for s, n in funcs:
            if s <= ln:
                name = n
            else:
                break
        return name

    hdr = rows[1]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    iss, ino = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("stall_no_inst")
    base = int(rows[2][ia], 16)
    inst, samp, noi = collections.Counter(), collections.Counter(), collections.Counter()
    execd = []
    per = []  # (executed count, function) per SASS instruction
    for r in rows[2:]:
        if len(r) <= ino:
            continue
        o = int(r[ia], 16) - base
        k = fn(off2src.get(o))
        n = int(r[ie] or 0)
        inst[k] += n
        samp[k] += int(r[iss] or 0)
        noi[k] += int(r[ino] or 0)
        execd.append(n)
        per.append((n, k))
    ti, ts, tn = sum(inst.values()), sum(samp.values()), sum(noi.values())
    print(f"instructions executed {ti:.3e}; stall samples {ts}; no_instruction share {tn / ts:.3f}")
    print(f"{'function':28s} {'samples':>8s} {'inst':>7s} {'no_inst':>8s}")
    for k, v in samp.most_common(25):
        print(f"{k:28s} {100 * v / ts:7.1f}% {100 * inst[k] / ti:6.1f}% {100 * noi[k] / tn:7.1f}%")
    execd.sort(reverse=True)
    acc = 0
    marks = [0.5, 0.8, 0.9, 0.95, 0.99]
    for i, n in enumerate(execd):
        acc += n
        while marks and acc >= marks[0] * ti:
            print(f"{marks[0]:.2f} of executed instructions in the {i + 1} hottest SASS instructions "
                  f"({(i + 1) * 16 / 1024:.0f} KB)")
            marks.pop(0)
    # hot footprint by function: SASS bytes among the instructions that make
    # up 90% of all executed instructions
    per.sort(key=lambda t: -t[0])
    acc, foot = 0, collections.Counter()
    for n, k in per:
        if acc >= 0.9 * ti:
            break
        acc += n
        foot[k] += 16
    print("hot footprint (90% of executed instructions) by function, bytes:")
    for k, v in foot.most_common(25):
        print(f"  {k:28s} {v:7d}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
