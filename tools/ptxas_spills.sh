#!/bin/bash
# Kernels whose ptxas log reports spills (dev tool): tools/ptxas_spills.sh [W...]
cd "$(dirname "$0")/.."
for w in ${@:-0 2 3 4 5 6 8}; do
  grep -E "Compiling entry|registers|spill" build/csrc/qsg_inst_w$w.ptxas.log \
    | grep -o "decode_kernel[_a-z]*ILi[0-9]ELi[0-9]*ELb[01]ELb[01]ELi[0-9]*\|Used [0-9]* registers\|[0-9]* bytes spill stores, [0-9]* bytes spill loads" \
    | paste - - - | grep -v "\b0 bytes spill stores, 0 bytes spill loads" | sed "s/^/W$w  /"
done
