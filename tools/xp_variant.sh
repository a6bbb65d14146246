#!/bin/bash
# libpi variant with interact_xpencil.cu compiled with extra flags, linked against the tree's
# other objects (development aid):  tools/xp_variant.sh OUT.so -DFLAG ...
set -e
cd "$(dirname "$0")/.."
out=$(realpath -m "$1"); shift
B=paper_2406_16091_b200/build
d=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
     --expt-relaxed-constexpr -Xptxas -v -I include "$@" -c paper_2406_16091_b200/csrc/interact_xpencil.cu -o $d/xp.o > $d/log 2>&1 || { cat $d/log; exit 1; }
objs=$(ls $B/*.o | grep -v interact_xpencil.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs $d/xp.o -Xlinker --version-script=$B/exports.map -ldl -lpthread
grep -A3 "k_interact_xpencilILi0ELi20ELb0ELi1E" $d/log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | head -2
rm -rf $d
echo "$out"
