#!/bin/bash
# A/B of two builds (build_ab/libvenom_before.so vs the in-tree libvenom.so), alternating processes
for rep in 1 2; do
for lib in build_ab/libvenom_before.so paper_2310_02065_b200/libvenom.so; do
  for w in $WORKLOADS; do
    VENOM_LIB=$PWD/$lib timeout 200 python tools/time_spmm_ab.py $w ${ROUNDS:-20} "" 2>&1 | grep median | sed "s|^|$(basename $lib) |"
  done
done; done
