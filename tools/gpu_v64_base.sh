#!/bin/bash
# baseline V = 64 gathered SpMM timings (before the M = 64 MMA rework)
set -x
for w in sweep_4096x4096x4096_64:2:16 sweep_4096x4096x4096_64:2:32 sweep_4096x4096x4096_128:2:16 \
         enc_qkv_3072x1040x16384_64:2:10 enc_o_1024x1040x16384_64:2:10 enc_ffn1_4096x1040x16384_64:2:10 \
         enc_ffn2_1024x4160x16384_64:2:10; do
  timeout 120 python tools/time_spmm.py $w '' 'tile_t=64' 'tile_t=256'
done
timeout 300 python tools/bench_encoder.py --layers 24 --steps 5
