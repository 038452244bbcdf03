python -m paper_2310_02065_b200.build >/dev/null
for fl in 0 15 31 64 79 8; do echo "flags $fl: $(VENOM_DEBUG_FLAGS=$fl bash tools/ncu_times.sh gpurun_out/t2.csv python tools/time_format.py 2>&1 | grep 'compress_tile_kernel<0, 1>')"; done
