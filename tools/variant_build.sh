#!/bin/bash
# Build a variant of libpi.so from a copy of the tree with one file replaced (development aid):
#   tools/variant_build.sh OUT.so REL_PATH REPLACEMENT [REL_PATH REPLACEMENT ...]
set -e
out=$(realpath -m "$1"); shift
d=$(mktemp -d)
cp -r "$(dirname "$0")/../paper_2406_16091_b200" "$(dirname "$0")/../include" "$d/"
rm -rf "$d/paper_2406_16091_b200/build" "$d/paper_2406_16091_b200/libpi.so"
while [ $# -gt 0 ]; do cp "$2" "$d/$1"; shift 2; done
(cd "$d" && python -c "import sys; sys.path.insert(0,'.'); from paper_2406_16091_b200 import build as b; b.build(force=True)" >/dev/null)
cp "$d/paper_2406_16091_b200/libpi.so" "$out"
rm -rf "$d"
echo "$out"
