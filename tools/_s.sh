python -m paper_2310_02065_b200.build >/dev/null
timeout 900 python -m pytest tests -q -m gpu -x -k "compress" > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python -m paper_2310_02065_b200.build --ablation >/dev/null
for fl in 0 2; do echo "flags $fl: $(VENOM_DEBUG_FLAGS=$fl bash tools/ncu_times.sh gpurun_out/t2.csv python tools/time_format.py 2>&1 | grep 'compress_tile_kernel')"; done
