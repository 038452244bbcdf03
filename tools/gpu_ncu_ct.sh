#!/bin/bash
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:vnm_spmm -c 1 -o gpurun_out/ncu_ct \
  python tools/time_spmm.py enc_qkv_3072x1040x16384_64:2:10 'transposed_out=1' > gpurun_out/ncu_ct.log 2>&1
ncu -i gpurun_out/ncu_ct.ncu-rep --page details --csv > gpurun_out/ncu_ct_details.csv 2>&1
ncu -i gpurun_out/ncu_ct.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_ct_source.csv 2>&1
ncu -i gpurun_out/ncu_ct.ncu-rep --page raw --csv > gpurun_out/ncu_ct_raw.csv 2>&1
rm -f gpurun_out/ncu_ct.ncu-rep
