#!/bin/bash
# One gpurun pass at the end of a work session (1 GPU): the GPU test suite, the default bench
# line, then the round's ncu captures (tools/profile_round.sh) summarised by
# tools/round_summary.py; the summaries land in gpurun_out/profiles/ and the large .ncu-rep
# files are deleted so gpurun_out/ stays under the copy-back limit.  usage: round_final.sh TAG
R=${1:-r02b}
mkdir -p gpurun_out/profiles
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputests.log 2>&1
tail -3 gpurun_out/${R}_gputests.log
timeout 900 python bench.py > gpurun_out/${R}_bench.log 2>&1
tail -1 gpurun_out/${R}_bench.log > gpurun_out/profiles/${R}_bench.json
bash tools/profile_round.sh $R > gpurun_out/${R}_profile.log 2>&1
python tools/round_summary.py $R > gpurun_out/${R}_summary.log 2>&1
cp profiles/${R}_ncu_summary.md profiles/ncu_traffic.json profiles/ncu_smem.json gpurun_out/profiles/
cp gpurun_out/${R}_launches.csv gpurun_out/profiles/ 2>/dev/null
for f in gpurun_out/*.ncu-rep; do [ -f "$f" ] && tools/ncu_export.sh "$f"; done
ls -la gpurun_out gpurun_out/profiles
