#!/bin/bash
# Build the working tree's libqsg.so with extra nvcc flags into abl/NAME.so
# (A/B timing of compile-time variants; dev tool).
# Usage: tools/build_variant.sh NAME "-DQSG_FOO -DQSG_BAR"
set -eu
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=${2:-}
W=cache/var_$NAME
rm -rf $W; mkdir -p $W/paper_2605_10433_b200 $W/include
cp -r paper_2605_10433_b200/csrc $W/paper_2605_10433_b200/
cp include/qsg.h $W/include/
make -s -C $W/paper_2605_10433_b200/csrc -j"$(nproc)" NVCC="nvcc $FLAGS" > /dev/null
mkdir -p abl
cp $W/paper_2605_10433_b200/libqsg.so abl/$NAME.so
rm -rf $W
echo abl/$NAME.so
