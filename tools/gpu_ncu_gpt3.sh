#!/bin/bash
# ncu --set full capture of the GPT-3 FFN SpMM (configs[3]) — its own gpurun call (64 MiB limit).
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 ncu --set full --clock-control none -k regex:vnm_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_gpt3 python bench.py --workload gpt3_ffn_12288x49152x8192_128:2:16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_full_gpt3.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python tools/ncu_summary.py full gpurun_out/prof_spmm_gpt3.ncu-rep gpurun_out/r01_ncu_full_spmm_gpt3.md gpt3_ffn_12288x49152x8192_128:2:16 > /dev/null
ncu -i gpurun_out/prof_spmm_gpt3.ncu-rep --page details --csv > gpurun_out/prof_spmm_gpt3_details.csv 2>/dev/null
rm -f gpurun_out/prof_spmm_gpt3.ncu-rep
ls -la gpurun_out
