#!/bin/bash
# Round evidence: tests, bench line, reference arm, ncu launch list + full capture of venom_spmm.
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 6 -c 2 -o gpurun_out/prof_spmm_bert python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_full.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:vnm_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_gpt3 python bench.py --workload gpt3_ffn_12288x49152x8192_128:2:16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_full_gpt3.txt 2>&1
ls gpurun_out
