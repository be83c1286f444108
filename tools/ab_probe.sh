# A/B of variants/*.so on one box: config-4 sweep wall time, alternating, $1 rounds (default 3)
R=${1:-3}
for r in $(seq 1 $R); do for f in variants/*.so; do KVSIM_LIB=$f python tools/occupancy_probe.py 2>&1 | sed "s#^#$(basename $f) #" >> gpurun_out/ab.log; done; done
