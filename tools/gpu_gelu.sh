#!/bin/bash
for w in enc_ffn1_4096x1040x16384_64:2:10 sweep_4096x4096x4096_128:2:16; do
  timeout 120 python tools/time_spmm.py $w '' 'gelu=1'
done
timeout 300 python -m pytest tests -m gpu -x -q -k gelu 2>&1 | tail -2
