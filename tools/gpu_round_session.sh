#!/bin/bash
# Round evidence: tests, bench line, reference arm, ncu launch list + full capture of venom_spmm
# (BERT; the GPT-3 capture is a second call: gpurun_out/ is limited to 64 MiB per call), encoder.
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:vnm_spmm -s 6 -c 2 -o gpurun_out/prof_spmm_bert python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_full.txt 2>&1
# summaries on the box (the report itself exceeds gpurun's 64 MiB copy-back)
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python tools/ncu_summary.py full gpurun_out/prof_spmm_bert.ncu-rep gpurun_out/r01_ncu_full_spmm_bert.md bert_large_ffn_4096tok_64:2:8 > /dev/null
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/r01_ncu_launches_bert.md > /dev/null
ncu -i gpurun_out/prof_spmm_bert.ncu-rep --page details --csv > gpurun_out/prof_spmm_bert_details.csv 2>/dev/null
rm -f gpurun_out/prof_spmm_bert.ncu-rep
timeout 400 python tools/bench_encoder.py > gpurun_out/encoder.json 2> gpurun_out/encoder.err
timeout 200 python tools/encoder_breakdown.py > gpurun_out/encoder_breakdown.txt 2>&1
ls -la gpurun_out
