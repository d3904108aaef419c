#!/bin/bash
# GPU correctness session (dev tool): the -m gpu suite, stress parity, the FER-match GPU leg.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gputest_$TAG.log
for s in ${STRESS_SEEDS:-}; do timeout 900 python tools/stress_parity.py $s 150 > gpurun_out/stress_${TAG}_$s.log 2>&1; echo "stress $s rc=$?"; tail -1 gpurun_out/stress_${TAG}_$s.log; done
if [ -n "${FER:-}" ]; then timeout 1200 python tools/fer_match_configs.py gpu --only $FER --gpu-dir gpurun_out/fer_cfg > gpurun_out/fer_gpu_$TAG.log 2>&1; echo "fer rc=$?"; fi
