python -m paper_2310_02065_b200.build >/dev/null
timeout 60 python tools/ablate.py 4096 4096 4096 128 4 1 1 127 383 639 895 0 256 | grep -v host
timeout 60 python tools/ablate.py 4096 8192 4096 128 4 1 1 127 383 639 895 | grep -v host
timeout 60 python tools/ablate.py 4096 4096 4096 128 4 1 2 127 383 0 256 | grep -v host
