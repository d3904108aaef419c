#!/bin/bash
# A/B/C throughput of several library builds (dev tool).
# Usage: LIBS="ab/a.so ab/b.so paper_2605_10433_b200/libqsg.so" tools/ab3.sh CODES DECODERS PS
set -u
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib (rep $rep)"
    QSG_LIB=$PWD/$lib timeout 600 python tools/perf_probe.py "$@" 2>&1 | sed 's/^/  /'
  done
done
