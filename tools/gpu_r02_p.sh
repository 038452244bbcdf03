#!/bin/bash
mkdir -p gpurun_out
W=gpt3_ffn_12288x49152x8192_128:2:16
for lib in libvenom.so libvenom_p11.so libvenom.so; do
  VENOM_LIB=paper_2310_02065_b200/$lib timeout 60 python tools/time_spmm.py $W "" 2>&1 | grep -v Warn | tail -1
done
VENOM_LIB=paper_2310_02065_b200/libvenom.so timeout 300 python -m pytest tests -q -m gpu -x -k "spmm" 2>&1 | tail -2
