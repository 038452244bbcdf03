#!/bin/bash
# One gpurun session: default bench line, larger workloads, ncu launch list + full capture of the SpMM.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --workload gpt3_ffn_12288x49152x8192_128:2:16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_gpt3.json 2> gpurun_out/bench_gpt3.err
for m in 4 8 16 32; do
  timeout 200 python bench.py --workload sweep_4096x4096x4096_128:2:$m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --step spmm > gpurun_out/bench_sweep_m$m.json 2>> gpurun_out/bench_sweep.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 4 -c 2 -o gpurun_out/prof_spmm_bert python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_bert.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 2 -c 1 -o gpurun_out/prof_spmm_gpt3 python bench.py --workload gpt3_ffn_12288x49152x8192_128:2:16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_gpt3.txt 2>&1
ls -la gpurun_out
