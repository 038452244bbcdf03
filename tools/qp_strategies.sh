mkdir -p gpurun_out
for wl in bert_large_ffn_4096tok_64:2:8 sweep_4096x4096x4096_128:2:8 sweep_4096x4096x4096_128:2:16; do
 for st in gather densek; do
  timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --step spmm --strategy $st 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$wl', '$st', 'spmm TF/s', d['spmm_only']['tflops'], 'ms', d['spmm_only']['ms_per_launch'], 'speedup', d['speedup_vs_cublas'], 'frac', d['roofline']['frac'])
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"
 done
done
