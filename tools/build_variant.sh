#!/bin/bash
# Build libps_b200.so from a git revision into build_ab/<name>/ (A/B runs select it with PS_B200_LIB).
# usage: tools/build_variant.sh <name> <rev>
set -e
name=$1; rev=${2:-HEAD}
cd "$(dirname "$0")/.."
rm -rf build_ab/$name; mkdir -p build_ab/$name
git archive "$rev" paper_2507_23480_b200/csrc include | tar -x -C build_ab/$name
make -C build_ab/$name/paper_2507_23480_b200/csrc -j8 -s
echo build_ab/$name/paper_2507_23480_b200/libps_b200.so
