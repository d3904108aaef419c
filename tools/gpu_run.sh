#!/bin/bash
# Round GPU session (dev tool): tests, bench, launch list, ncu captures of the
# min-sum and BP4 kernels on this build.
cd "$(dirname "$0")/.."
TAG=${TAG:-r02d}
TAG=$TAG STEPS=tests,bench,launch bash tools/gpu_session.sh
TAG=ms008_$TAG VAR=sagms P=0.08 STEPS=ncu bash tools/gpu_session.sh
TAG=bp4_$TAG VAR=bp4 P=0.1 STEPS=ncu bash tools/gpu_session.sh
