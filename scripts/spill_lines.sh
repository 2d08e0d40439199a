#!/bin/bash
# source lines of local-memory loads/stores (spills) in one stage-kernel instantiation
# usage: spill_lines.sh '9,32,32,32,7,0,16384,8,24,0,0'
R="$(cd "$(dirname "$0")/.." && pwd)"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo -I"$R/include" \
  -cubin -o /tmp/k_sl.cubin "$R/paper_2106_06445_b200/csrc/k_umma.cu" 2>/dev/null
F=".text._ZN2ci7k_stageINS_4SCfgILi$(echo "$1" | sed 's/,/ELi/g')EEEEEvNS_9StageArgsE:"
nvdisasm --print-line-info /tmp/k_sl.cubin 2>/dev/null | awk -v f="$F" '$0==f{on=1;next} on && /^\.text\./{on=0} on' |
  awk '/line [0-9]+/{match($0,/line [0-9]+/); ln=substr($0,RSTART+5,RLENGTH-5)} /STL/{print "STL", ln} /LDL/{print "LDL", ln}' |
  sort -k2n | uniq -c | while read c op l; do echo "$c $op $l: $(sed -n ${l}p "$R/paper_2106_06445_b200/csrc/k_umma.cu" | cut -c1-90)"; done
