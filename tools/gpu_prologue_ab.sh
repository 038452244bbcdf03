#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for lib in build_ab/libvenom_before.so paper_2310_02065_b200/libvenom.so build_ab/libvenom_before.so paper_2310_02065_b200/libvenom.so; do
  for w in bert_large_ffn2_1024x4096x4096_64:2:8 bert_large_ffn1_4096x1024x4096_64:2:8 sweep_4096x4096x4096_128:2:32 sweep_4096x4096x4096_64:2:16 enc_qkv_3072x1040x16384_64:2:10; do
    VENOM_LIB=$PWD/$lib timeout 120 python tools/time_spmm_ab.py $w 20 "" 2>&1 | sed "s|^|$(basename $lib) |"
  done
done
