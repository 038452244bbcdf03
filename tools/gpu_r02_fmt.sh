#!/bin/bash
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or decompress or expand or graph or smoke" > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python tools/time_format.py 12288 49152 128 16 2>&1 | grep -v Warn
timeout 300 python tools/time_format.py 1024 4096 64 8 2>&1 | grep -v Warn
timeout 300 python tools/time_format.py 4096 1024 64 8 2>&1 | grep -v Warn
