#!/bin/bash
# One GPU session: bench (ours + reference arm), launch list and one full ncu
# capture of the dominant decode kernel.  Outputs land in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
TAG=${TAG:-r01}
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 600 $CMD > $O/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file $O/launches_$TAG.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch-list rc=$?"
PCMD="python tools/perf_probe.py 254 sagms 0.08"
FRAMES=131072 timeout 300 $PCMD > $O/plain_probe.log 2>&1 && \
  FRAMES=131072 timeout 1200 ncu --set full --clock-control none --import-source on \
     -k regex:decode_kernel -s 1 -c 1 -o $O/prof_$TAG -f $PCMD > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"
ls -la $O
