python -m paper_2310_02065_b200.build >/dev/null
timeout 60 python tools/ablate.py 4096 2048 4096 128 4 1 2 0 | grep -v host
timeout 60 python tools/ablate.py 4096 4096 4096 128 8 1 1 0 | grep -v host
timeout 60 python tools/ablate.py 4096 1024 4096 128 4 1 2 0 | grep -v host
timeout 60 python tools/ablate.py 4096 4096 4096 128 16 1 1 0 | grep -v host
