#!/bin/bash
for lib in libvenom.so libvenom_t16.so; do
VENOM_LIB=paper_2310_02065_b200/$lib timeout 300 python tools/time_format.py 12288 49152 128 16 2>&1 | grep -v Warn | grep "cold" | head -2
done
VENOM_LIB=paper_2310_02065_b200/libvenom_t16.so timeout 600 python -m pytest tests -q -m gpu -x -k "compress" 2>&1 | tail -2
