#!/bin/bash
for w in sweep_4096x4096x4096_128:2:32 sweep_4096x4160x4096_128:2:40 sweep_4096x4096x4096_128:2:16 fig6_1024x4160x4096_128:2:10 fig6_1024x4160x4096_128:2:40 fig6_1024x4800x4096_128:2:100 sweep_4096x4096x4096_256:2:32; do
  timeout 120 python tools/time_spmm_ab.py $w 20 "" "tile_t=192" "tile_t=128" "tile_t=64"
done
