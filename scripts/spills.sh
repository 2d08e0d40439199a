#!/bin/bash
# ptxas spill report of the stage-kernel instantiations (compiles k_umma.cu alone)
R="$(cd "$(dirname "$0")/.." && pwd)"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I"$R/include" -Xptxas -v \
  -c "$R/paper_2106_06445_b200/csrc/k_umma.cu" -o /tmp/k_umma_spills.o 2>&1 |
  grep -A2 "Compiling entry.*k_stage" | grep -o "SCfgIL[^']*'\|[0-9]* bytes spill stores, [0-9]* bytes spill loads" |
  paste - - | sed 's/SCfgIL//; s/EEEEEvNS_9StageArgsE.//; s/ELi/,/g; s/^i//'
