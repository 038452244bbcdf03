#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v64_tests.txt 2>&1
echo "tests rc=$?"
for w in sweep_4096x4096x4096_64:2:16 sweep_4096x4096x4096_64:2:32 \
         enc_qkv_3072x1040x16384_64:2:10 enc_o_1024x1040x16384_64:2:10 enc_ffn1_4096x1040x16384_64:2:10 \
         enc_ffn2_1024x4160x16384_64:2:10; do
  timeout 120 python tools/time_spmm.py $w '' 'transposed_out=1' 'gelu=1'
done > gpurun_out/v64_times.txt 2>&1
timeout 200 python tools/encoder_breakdown.py > gpurun_out/enc_breakdown_m64.txt 2>&1
timeout 300 python tools/bench_encoder.py --layers 24 --steps 5 > gpurun_out/enc_m64.json 2>&1
REPS=1 timeout 600 ncu --set full --clock-control none -k regex:vnm_spmm -c 2 -o gpurun_out/ncu_qkv \
  python tools/time_spmm.py enc_qkv_3072x1040x16384_64:2:10 '' 'transposed_out=1' > gpurun_out/ncu_qkv.log 2>&1
ncu -i gpurun_out/ncu_qkv.ncu-rep --page details --csv > gpurun_out/ncu_qkv_details.csv 2>&1
rm -f gpurun_out/ncu_qkv.ncu-rep
