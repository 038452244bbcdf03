python -m paper_2310_02065_b200.build >/dev/null
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
NOTEST=1 FORMS="auto" WLS="bert_large_ffn_4096tok_64:2:8 sweep_4096x4096x4096_64:2:4 sweep_4096x4096x4096_64:2:8 sweep_4096x4096x4096_64:2:16 sweep_4096x4096x4096_128:2:4 sweep_4096x4096x4096_128:2:8" bash tools/quick_perf.sh
