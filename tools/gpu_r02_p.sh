#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests -q -m gpu -x -k "spmm or smoke or graph" 2>&1 | tail -2
for W in gpt3_ffn_12288x49152x8192_128:2:16 bert_large_ffn2_1024x4096x4096_64:2:8 bert_large_ffn1_4096x1024x4096_64:2:8 sweep_4096x4096x4096_128:2:32 sweep_4096x4096x4096_128:2:4; do
for lib in libvenom_prev.so libvenom.so; do
  VENOM_LIB=paper_2310_02065_b200/$lib REPS=20 timeout 60 python tools/time_spmm.py $W "" 2>&1 | grep -v Warn | tail -1
done; done
