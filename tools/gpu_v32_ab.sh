#!/bin/bash
true
for lib in build_ab/libvenom_before.so paper_2310_02065_b200/libvenom.so; do
  for w in sweep_4096x4096x4096_32:2:8 sweep_4096x4096x4096_32:2:16 sweep_4096x4096x4096_32:2:32; do
    FORM=vnm VENOM_LIB=$PWD/$lib timeout 120 python tools/time_spmm_ab.py $w 20 "" "transposed_out=1" 2>&1 | sed "s|^|$(basename $lib) |"
  done
done
