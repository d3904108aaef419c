#!/bin/bash
# A/B throughput of the in-tree build against ${AB_BASE:-ab/libqsg_base.so} (dev tool).
# Usage: tools/ab_probe.sh CODES DECODERS PS  (perf_probe.py arguments)
set -u
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in ${AB_BASE:-ab/libqsg_base.so} paper_2605_10433_b200/libqsg.so; do
    echo "== $lib (rep $rep)"
    QSG_LIB=$PWD/$lib timeout 600 python tools/perf_probe.py "$@" 2>&1 | sed 's/^/  /'
  done
done
