#!/bin/bash
# round 2: independent feed microbenchmark, the new bench line (GPT-3 default), GPU tests
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 300 ./tools/microbench_feed > gpurun_out/microbench_feed.txt 2>&1; tail -40 gpurun_out/microbench_feed.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
