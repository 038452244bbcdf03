python -m paper_2310_02065_b200.build >/dev/null
timeout 600 python -m pytest tests -q -m gpu -x -k "two_row" > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for t in 256 240; do
TILE=$t timeout 60 python tools/ablate.py 1024 4096 4096 64 4 1 2 0 4 | grep -v host
TILE=$t timeout 60 python tools/ablate.py 4096 1024 4096 64 4 1 2 0 4 | grep -v host
TILE=$t timeout 60 python tools/ablate.py 4096 4096 4096 128 4 1 2 0 4 | grep -v host
TILE=$t timeout 60 python tools/ablate.py 4096 8192 8192 128 4 1 2 0 | grep -v host
done
