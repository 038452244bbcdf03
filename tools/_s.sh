python -m paper_2310_02065_b200.build >/dev/null
NOTEST=1 FORMS="auto" WLS="bert_large_ffn_4096tok_64:2:8 sweep_4096x4096x4096_64:2:4 sweep_4096x4096x4096_64:2:8 sweep_4096x4096x4096_64:2:16 sweep_4096x4096x4096_64:2:32 sweep_4096x4160x4096_64:2:40 sweep_4096x4096x4096_128:2:4 sweep_4096x4096x4096_128:2:8 sweep_4096x4096x4096_128:2:16 sweep_4096x4096x4096_128:2:32 sweep_4096x4160x4096_128:2:40 gpt3_ffn_12288x49152x8192_128:2:16" bash tools/quick_perf.sh > gpurun_out/sweep.txt 2>&1
NOTEST=1 FORMS="vnm 2to4" WLS="sweep_4096x4096x4096_64:2:16 sweep_4096x4096x4096_64:2:32 sweep_4096x4096x4096_128:2:8 sweep_4096x4096x4096_128:2:16" bash tools/quick_perf.sh >> gpurun_out/sweep.txt 2>&1
cat gpurun_out/sweep.txt
