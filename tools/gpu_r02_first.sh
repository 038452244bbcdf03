#!/bin/bash
# round 2 first contact: tests on the restored build, current bench lines (BERT and GPT-3)
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/bench_bert.json 2> gpurun_out/bench_bert.err; cat gpurun_out/bench_bert.json
timeout 600 python bench.py --workload gpt3_ffn_12288x49152x8192_128:2:16 --steps 10 --no-cpu-baseline > gpurun_out/bench_gpt3.json 2> gpurun_out/bench_gpt3.err; cat gpurun_out/bench_gpt3.json; tail -3 gpurun_out/bench_gpt3.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
