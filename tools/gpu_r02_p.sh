#!/bin/bash
mkdir -p gpurun_out
W=gpt3_ffn_12288x49152x8192_128:2:16
for lib in libvenom_r1.so libvenom_p8.so libvenom.so libvenom_r1.so; do
  VENOM_LIB=paper_2310_02065_b200/$lib timeout 300 python tools/time_spmm.py $W group_n=1 group_n=3
done 2>&1 | grep -v Warn
