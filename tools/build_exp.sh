#!/bin/bash
# Build an experimental variant of the product library for A/B timing:
#   tools/build_exp.sh NAME "-DFLAG ..."   ->  paper_1808_10481_b200/lib/exp_NAME.so
set -e
name=$1; flags=$2
here=$(cd "$(dirname "$0")/.." && pwd)
bld=$here/paper_1808_10481_b200/build/exp_$name
mkdir -p "$bld"
make -s -C "$here/paper_1808_10481_b200/csrc" -j8 OBJ="$bld" LIB="$here/paper_1808_10481_b200/lib/exp_$name.so" \
  EXTRA_NVFLAGS="$flags" >/dev/null
echo "built exp_$name.so ($flags)"
