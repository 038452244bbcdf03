#!/bin/bash
# V-scaling study (the paper's Fig 8 axis) at 4096^3: gathered form (FORM=vnm) and the planner's form
for V in 32 64 128 256; do for M in 8 16 32; do
  w=sweep_4096x4096x4096_${V}:2:${M}
  FORM=vnm timeout 120 python tools/time_spmm_ab.py $w 20 "" 2>&1 | sed "s|^|gathered |"
  timeout 120 python tools/time_spmm_ab.py $w 20 "" 2>&1 | sed "s|^|planner  |"
done; done
