#!/bin/bash
timeout 300 python -m pytest tests -m gpu -x -q -k "decompress" > gpurun_out/bg_tests.txt 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/bg_tests.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-secondary --no-e2e --cpu-budget 2 > gpurun_out/bench_bg.json 2> gpurun_out/bench_bg.err; echo "bench rc=$?"
