#!/bin/bash
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vnm_compress_tma -c 1 -o gpurun_out/ncu_cmp \
  python tools/time_format.py 12288 49152 128 16 > gpurun_out/ncu_cmp.log 2>&1
ncu -i gpurun_out/ncu_cmp.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_cmp_cuda.csv 2>&1
ncu -i gpurun_out/ncu_cmp.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_cmp_sass.csv 2>&1
ncu -i gpurun_out/ncu_cmp.ncu-rep --page details --csv > gpurun_out/ncu_cmp_details.csv 2>&1
rm -f gpurun_out/ncu_cmp.ncu-rep
