python -m paper_2310_02065_b200.build >/dev/null
timeout 900 python -m pytest tests -q -m gpu -x -k "compress or encoder or graph" > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
bash tools/ncu_times.sh gpurun_out/t1.csv python tools/time_format.py | grep venom
