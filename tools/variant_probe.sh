# Config-4 sweep wall time for the in-tree build and each variants/*.so (KVSIM_LIB)
python tools/occupancy_probe.py > gpurun_out/var_base.log 2>&1
for f in variants/*.so; do KVSIM_LIB=$f python tools/occupancy_probe.py > gpurun_out/var_$(basename $f .so).log 2>&1; done
