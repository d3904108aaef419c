#!/bin/bash
# One GPU session (dev tool): gpu tests, bench, FER-match GPU leg, launch list.
# TAG names the outputs; STEPS selects parts (tests,bench,fer,launch,ncu).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
TAG=${TAG:-r02}; STEPS=${STEPS:-tests,bench,fer,launch}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi_$TAG.txt 2>&1
has() { [[ ",$STEPS," == *",$1,"* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 $O/gputest_$TAG.log
fi
if has bench; then
  timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; echo "bench rc=$?"; cat $O/bench_$TAG.json | head -c 3000; echo
fi
if has fer; then
  timeout 1200 python tools/fer_match_configs.py gpu --gpu-dir $O/fer_cfg > $O/fer_gpu_$TAG.log 2>&1; echo "fer rc=$?"
fi
if has launch; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
  timeout 600 $CMD > $O/plain_launch.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
       --log-file $O/launches_$TAG.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch-list rc=$?"
fi
if has ncu; then
  CODE=${CODE:-254}; VAR=${VAR:-sagms}; P=${P:-0.08}
  python -c "import sys; sys.path.insert(0, '.'); from paper_2605_10433_b200 import _native; print(_native.lib().qsg_build_id().decode())" > $O/build_id_$TAG.txt
  PCMD="python tools/perf_probe.py $CODE $VAR $P"
  FRAMES=131072 timeout 300 $PCMD > $O/plain_probe_$TAG.log 2>&1 && \
    FRAMES=131072 timeout 1200 ncu --set full --clock-control none --import-source on \
       -k regex:decode_kernel -s 1 -c 1 -o $O/prof_$TAG -f $PCMD > $O/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi
