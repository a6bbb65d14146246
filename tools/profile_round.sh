#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Writes gpurun_out/${R}_*.
# The bench workload is configs[4] (2^27 particles, 256^3 cells).
set -x
R=${1:-r02}
mkdir -p gpurun_out
# 1. launch list of the bench command (cold-cache, serialised: compare SHARES, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-binning-2e24 --no-c1 > gpurun_out/${R}_launches_bench.log 2>&1
# 2. full capture of the bench's interaction kernel on configs[4] (traffic = dram bytes per launch)
ncu --set full --clock-control none --import-source on -k regex:k_interact_xpencil -s 1 -c 1 \
    -o gpurun_out/${R}_xpencil_c4 python tools/prof_one.py c4 xpencil 2 > gpurun_out/${R}_ncu_xpencil_c4.log 2>&1
# 3. the strategies on configs[1]
for A in xpencil global fullload xpreg; do
  ncu --set full --clock-control none --import-source on -k regex:k_interact_$A -s 2 -c 1 \
      -o gpurun_out/${R}_$A python tools/prof_one.py c1 $A 3 > gpurun_out/${R}_ncu_$A.log 2>&1
done
# 4. binning: pi_step re-binning on configs[4] (the bench step's binning) and pi_bin at 2^24
ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_scatter" -s 4 -c 2 \
    -o gpurun_out/${R}_rebin python tools/prof_rebin.py c4 > gpurun_out/${R}_ncu_rebin.log 2>&1
ncu --set full --clock-control none -k regex:"k_count|k_scan|k_partition|k_scatter" -s 4 -c 4 \
    -o gpurun_out/${R}_bin python tools/prof_bin.py c2_ppc8 > gpurun_out/${R}_ncu_bin.log 2>&1
ls -la gpurun_out
