python -m paper_2310_02065_b200.build >/dev/null
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 60 python tools/ablate.py 1024 4096 4096 64 4 1 2 0 4 | grep -v host
timeout 60 python tools/ablate.py 4096 1024 4096 64 4 1 2 0 4 | grep -v host
timeout 60 python tools/ablate.py 4096 4096 4096 128 4 1 2 0 4 | grep -v host
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
