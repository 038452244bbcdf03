#!/bin/bash
# Round-2 (second half) evidence: the default bench line first (no profiler), then ncu launch list of the default bench step (GPT-3 FFN), --set full captures of
# the GPT-3 SpMM, compressor and decompressor, and of the BERT FFN SpMMs; summaries on the box
# (the reports exceed gpurun's copy-back limit).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02b_bench_line.json 2> gpurun_out/r02b_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_bench_reference_line.json 2>/dev/null
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-secondary > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r02b_launches.csv gpurun_out/r02b_ncu_launches_gpt3.md > /dev/null
W=gpt3_ffn_12288x49152x8192_128:2:16
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vnm_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_gpt3 \
  env REPS=1 python tools/time_spmm.py $W "" > gpurun_out/ncu_gpt3.txt 2>&1
python tools/ncu_summary.py full gpurun_out/prof_spmm_gpt3.ncu-rep gpurun_out/r02b_ncu_full_spmm_gpt3.md $W > /dev/null
python tools/ncu_brief.py gpurun_out/prof_spmm_gpt3.ncu-rep vnm_spmm 12 > gpurun_out/r02b_ncu_brief_spmm_gpt3.txt
ncu -i gpurun_out/prof_spmm_gpt3.ncu-rep --page details --csv > gpurun_out/r02b_ncu_details_spmm_gpt3.csv 2>/dev/null
rm -f gpurun_out/prof_spmm_gpt3.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vnm_compress_tma|vnm_decompress_m8|order_metadata" -c 3 \
  -o gpurun_out/prof_fmt_gpt3 python tools/time_format.py 12288 49152 128 16 > gpurun_out/ncu_fmt.txt 2>&1
python tools/ncu_summary.py full gpurun_out/prof_fmt_gpt3.ncu-rep gpurun_out/r02b_ncu_full_format_gpt3.md > /dev/null
python tools/ncu_brief.py gpurun_out/prof_fmt_gpt3.ncu-rep "compress_tma|decompress" 8 > gpurun_out/r02b_ncu_brief_format_gpt3.txt
rm -f gpurun_out/prof_fmt_gpt3.ncu-rep
timeout 600 ncu --set full --clock-control none -k regex:vnm_spmm -s 6 -c 2 -o gpurun_out/prof_spmm_bert \
  python bench.py --workload bert_large_ffn_4096tok_64:2:8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
python tools/ncu_summary.py full gpurun_out/prof_spmm_bert.ncu-rep gpurun_out/r02b_ncu_full_spmm_bert.md bert_large_ffn_4096tok_64:2:8 > /dev/null
rm -f gpurun_out/prof_spmm_bert.ncu-rep
W2=enc_qkv_3072x1040x16384_64:2:10
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vnm_spmm -s 3 -c 1 -o gpurun_out/prof_spmm_encqkv \
  env REPS=1 python tools/time_spmm.py $W2 "transposed_out=1" > gpurun_out/ncu_encqkv.txt 2>&1
python tools/ncu_summary.py full gpurun_out/prof_spmm_encqkv.ncu-rep gpurun_out/r02b_ncu_full_spmm_enc_qkv.md > /dev/null
python tools/ncu_brief.py gpurun_out/prof_spmm_encqkv.ncu-rep vnm_spmm 8 > gpurun_out/r02b_ncu_brief_spmm_enc_qkv.txt
rm -f gpurun_out/prof_spmm_encqkv.ncu-rep
ls -la gpurun_out
