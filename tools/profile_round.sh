#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Writes gpurun_out/prof_*.
set -x
R=${1:-r01}
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare SHARES, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_launches_bench.log 2>&1
# 2. full capture of the interaction kernels (traffic = dram bytes per launch)
ncu --set full --clock-control none --import-source on -k regex:k_interact -s 2 -c 2 \
    -o gpurun_out/${R}_interact python tools/prof_one.py c1 xpencil 3 > gpurun_out/${R}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_interact_global -s 1 -c 1 \
    -o gpurun_out/${R}_global python tools/prof_one.py c1 global 2 > gpurun_out/${R}_ncu2.log 2>&1
# 3. binning kernels at 2^24 particles (configs[2] ppc 8: larger than L2)
ncu --set full --clock-control none --import-source on -k regex:"k_count|k_scan|k_scatter" -s 3 -c 3 \
    -o gpurun_out/${R}_bin python tools/prof_one.py c2_ppc8 global 2 > gpurun_out/${R}_ncu3.log 2>&1
ls -la gpurun_out
