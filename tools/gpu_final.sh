#!/bin/bash
# End-of-round GPU session (dev tool): smoke, the -m gpu suite, bench, launch
# list, ncu captures of the min-sum and BP4 kernels, every BASELINE config.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
TAG=${TAG:-r02z}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_$TAG.log
TAG=$TAG STEPS=tests,bench,launch bash tools/gpu_session.sh
TAG=ms008_$TAG VAR=sagms P=0.08 STEPS=ncu bash tools/gpu_session.sh
TAG=bp4_$TAG VAR=bp4 P=0.1 STEPS=ncu bash tools/gpu_session.sh
timeout 1200 python tools/configs_bench.py --out $O/configs_$TAG.json > $O/configs_$TAG.log 2>&1; echo "configs rc=$?"
