#!/bin/bash
# Build libqsg.so of git revision REV into abl/NAME.so (A/B timing baseline;
# abl/*.so travels to the GPU box, git ignores *.so).  Dev tool.
# Usage: tools/build_rev.sh REV NAME
set -eu
cd "$(dirname "$0")/.."
REV=$1; NAME=$2
W=cache/rev_$NAME
rm -rf $W; mkdir -p $W
git archive "$REV" paper_2605_10433_b200/csrc include | tar -x -C $W
make -s -C $W/paper_2605_10433_b200/csrc -j"$(nproc)" > /dev/null
mkdir -p abl
cp $W/paper_2605_10433_b200/libqsg.so abl/$NAME.so
rm -rf $W
echo abl/$NAME.so
