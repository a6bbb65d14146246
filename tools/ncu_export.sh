#!/bin/bash
# On the GPU box: export an ncu report's details/raw/source pages as gzipped CSV next to it and
# delete the (large) report, so gpurun_out/ stays under the copy-back limit.  usage: ncu_export.sh REP.ncu-rep
r=${1%.ncu-rep}
ncu -i $1 --page details --csv > $r.details.csv
ncu -i $1 --page raw --csv | gzip > $r.raw.csv.gz
ncu -i $1 --page source --csv --print-source sass | gzip > $r.source.csv.gz
rm -f $1
