#!/bin/bash
# One full ncu capture of the dominant decode kernel (plain run first).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O; TAG=${TAG:-r01}
CODE=${CODE:-254}; VAR=${VAR:-sagms}; P=${P:-0.08}
PCMD="python tools/perf_probe.py $CODE $VAR $P"
FRAMES=131072 timeout 300 $PCMD > $O/plain_probe_$TAG.log 2>&1 && \
  FRAMES=131072 timeout 1200 ncu --set full --clock-control none --import-source on \
     -k regex:decode_kernel -s 1 -c 1 -o $O/prof_$TAG -f $PCMD > $O/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
