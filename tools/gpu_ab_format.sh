#!/bin/bash
# A/B of the format kernels between build_ab/libvenom_before.so and the in-tree build
for rep in 1 2; do for lib in build_ab/libvenom_before.so paper_2310_02065_b200/libvenom.so; do
  VENOM_LIB=$PWD/$lib timeout 200 python tools/time_format.py 12288 49152 128 16 2>&1 | grep "^compress " | sed "s|^|$(basename $lib) gpt3 |"
  VENOM_LIB=$PWD/$lib timeout 200 python tools/time_format.py 1024 4096 64 8 2>&1 | grep "^compress" | sed "s|^|$(basename $lib) bert |"
done; done
