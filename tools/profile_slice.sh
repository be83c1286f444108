#!/bin/bash
# ncu --set full of the sweep kernel on a config-4 slice (tools/ncu_slice.py),
# reduced ON THE GPU BOX to small summaries under gpurun_out/ (the .ncu-rep and
# the SASS source page are far above gpurun's 64 MiB copy-back limit):
#   <tag>_metrics.csv   selected raw metrics (time, issue, stalls, caches, DRAM, L2)
#   <tag>_attr.txt      per-function executed instructions / stall samples
#   <tag>_sass_cols.txt column names of the source page (for reference)
# usage: tools/profile_slice.sh TAG [RATES] [REQUESTS] [POLICY]
set -u
TAG=${1:-slice}; RATES=${2:-84}; REQ=${3:-10000}; POL=${4:-}
O=gpurun_out
python tools/ncu_slice.py $RATES $REQ $POL > $O/${TAG}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kvsim_sweep -s 0 -c 1 -o /tmp/$TAG \
    python tools/ncu_slice.py $RATES $REQ $POL > $O/${TAG}_ncu.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > /tmp/${TAG}_raw.csv 2>/dev/null
python - /tmp/${TAG}_raw.csv > $O/${TAG}_metrics.csv <<'PY'
import csv, sys, re
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
keep = re.compile(r"gpu__time_duration.sum|smsp__issue_active|smsp__inst_executed.sum$|sm__warps_active|"
                  r"stall|dram__bytes_(read|write).sum$|lts__t_bytes.sum$|l1tex__t_bytes.sum$|icc|"
                  r"launch__registers|launch__occupancy|smsp__average_warp_latency|l1tex__data_pipe_lsu_wavefronts_mem_shared|"
                  r"smsp__sass_inst_executed_op_(local|shared|global)|sm__sass_inst_executed_op_(local|shared|global)|"
                  r"l1tex__t_sectors_pipe_lsu_mem_local|l1tex__t_sector_hit_rate|lts__t_sector_hit_rate")
w = csv.writer(sys.stdout)
w.writerow(["metric", "unit", "value"])
for h, u, v in zip(hdr, units, vals):
    if keep.search(h):
        w.writerow([h, u, v])
PY
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_sass.csv 2>/dev/null
head -1 /tmp/${TAG}_sass.csv | tr ',' '\n' > $O/${TAG}_sass_cols.txt
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all ${KVSIM_LIB:-$GRAFT_REPO_ROOT/paper_2411_05555_b200/_build/libkvsim_gpu.so} > /dev/null)
nvdisasm -g -c /tmp/cub/kvsim_sweep.sm_100a.cubin > /tmp/${TAG}_dis.txt 2>/dev/null
python tools/ncu_attribute.py /tmp/${TAG}_sass.csv /tmp/${TAG}_dis.txt paper_2411_05555_b200/csrc/kvsim_sim.cuh > $O/${TAG}_attr.txt 2>&1
ls -la $O
