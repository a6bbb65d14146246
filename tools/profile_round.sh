#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Writes gpurun_out/${R}_*.
set -x
R=${1:-r01}
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare SHARES, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-binning-2e24 > gpurun_out/${R}_launches_bench.log 2>&1
# 2. full captures of the three interaction kernels on configs[1] (traffic = dram bytes per launch)
for A in xpencil global fullload; do
  ncu --set full --clock-control none --import-source on -k regex:k_interact_$A -s 2 -c 1 \
      -o gpurun_out/${R}_$A python tools/prof_one.py c1 $A 3 > gpurun_out/${R}_ncu_$A.log 2>&1
done
# 3. binning kernels at 2^24 (configs[2] ppc 8): pi_step re-binning (AoS path) and pi_bin (random order)
ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_scatter" -s 4 -c 2 \
    -o gpurun_out/${R}_rebin python tools/prof_rebin.py c2_ppc8 > gpurun_out/${R}_ncu_rebin.log 2>&1
ncu --set full --clock-control none -k regex:"k_count|k_scan|k_partition|k_scatter" -s 4 -c 4 \
    -o gpurun_out/${R}_bin python tools/prof_bin.py c2_ppc8 > gpurun_out/${R}_ncu_bin.log 2>&1
ls -la gpurun_out
