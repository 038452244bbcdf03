python -m paper_2310_02065_b200.build >/dev/null
NOTEST=1 FORMS="auto" WLS="fig6_1024x4160x4096_128:2:10 fig6_1024x4160x4096_128:2:20 fig6_1024x4160x4096_128:2:40 fig6_1024x4800x4096_128:2:100" bash tools/quick_perf.sh > gpurun_out/fig6.txt 2>&1; cat gpurun_out/fig6.txt
