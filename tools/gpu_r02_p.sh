#!/bin/bash
for W in sweep_4096x4096x4096_128:2:32 sweep_4096x4096x4096_128:2:16 sweep_4096x4160x4096_128:2:40 fig6_1024x4160x4096_128:2:20 sweep_4096x4096x4096_256:2:32; do
  REPS=20 timeout 60 python tools/time_spmm.py $W "" "tile_t=128" "tile_t=192" 2>&1 | grep -v Warn
done
