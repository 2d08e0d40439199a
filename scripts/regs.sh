#!/bin/bash
# register / stack usage of the stage kernel instantiations in the built library
cuobjdump --dump-resource-usage "$(dirname "$0")/../paper_2106_06445_b200/libcodedinv.so" 2>/dev/null | grep -A1 "k_stage" |
  grep -o "Function [^:]*\|REG:[0-9]*\|STACK:[0-9]*" | paste - - - | awk '{print $2, $3, $4}' |
  sed 's/_ZN2ci7k_stageINS_4SCfgIL//; s/EEEEEvNS_9StageArgsE//; s/ELi/,/g; s/^i//'
