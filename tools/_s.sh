python -m paper_2310_02065_b200.build >/dev/null
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
VENOM_DEBUG_FLAGS=4 timeout 300 python bench.py --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], d['spmm_only'])"
timeout 120 python tools/ablate.py 4096 1024 4096 64 4 1 2 0 4 | grep -v host
