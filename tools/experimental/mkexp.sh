#!/bin/bash
# Build an experimental variant of the product library from a patched copy of
# one source: tools/experimental/mkexp.sh NAME FILE.cu PATCHED.cu
# -> paper_1808_10481_b200/lib/exp_NAME.so (git-ignored; tools/ab.sh times it)
set -e
name=$1; file=$2; patched=$3
root=$(cd "$(dirname "$0")/../.." && pwd)
tmp=/tmp/hlf_exp_$name
rm -rf $tmp; mkdir -p $tmp/paper_1808_10481_b200
cp -r $root/include $tmp/
cp -rp $root/paper_1808_10481_b200/csrc $tmp/paper_1808_10481_b200/
[ -d $root/paper_1808_10481_b200/build ] && cp -rp $root/paper_1808_10481_b200/build $tmp/paper_1808_10481_b200/
cp $patched $tmp/paper_1808_10481_b200/csrc/$file
make -s -C $tmp/paper_1808_10481_b200/csrc -j8 >/dev/null 2>&1
cp $tmp/paper_1808_10481_b200/lib/libhlf_b200.so $root/paper_1808_10481_b200/lib/exp_$name.so
