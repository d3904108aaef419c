#!/bin/bash
# A/B of library builds in abl/ against the in-tree build (dev tool).
# Usage: LIBS="abl/a.so ..." CASES="254:sagms,bp4:0.02,0.1 1022:sagms:0.03" tools/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/${ABTAG:-ab}.log
: > $OUT
for c in $CASES; do
  IFS=: read code dec ps <<< "$c"
  LIBS="$LIBS paper_2605_10433_b200/libqsg.so" bash tools/ab3.sh $code $dec $ps >> $OUT 2>&1
done
python tools/ab_table.py $OUT
