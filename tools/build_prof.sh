#!/bin/bash
# Builds tools/libpi_prof.so: libpi with the X-pencil phase counters (-DXP_PROFILE).
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/piprof
for f in paper_2406_16091_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
       -DXP_PROFILE -I include -c "$f" -o /tmp/piprof/$(basename "$f" .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libpi_prof.so /tmp/piprof/*.o -ldl -lpthread
echo built tools/libpi_prof.so
