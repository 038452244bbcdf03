#!/bin/bash
# quick perf iteration: parity tests + spmm-only timings on the main workloads
# env: WLS (workload list), STRATS (auto|gather|densek), TILES, FORMS (auto|vnm|2to4), NOTEST=1
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
fi
for wl in ${WLS:-bert_large_ffn_4096tok_64:2:8 gpt3_ffn_12288x49152x8192_128:2:16 sweep_4096x4096x4096_128:2:8 sweep_4096x4096x4096_128:2:16 sweep_4096x4096x4096_128:2:32}; do
  for st in ${STRATS:-auto}; do
  for tt in ${TILES:-0}; do
  for fm in ${FORMS:-auto}; do
    SA=""; [ "$st" != "auto" ] && SA="--strategy $st"
    timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --step spmm --tile-t $tt --form $fm $SA 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$wl', '$st', 'tile', $tt, '$fm', 'spmm TF/s', d['spmm_only']['tflops'], 'ms', d['spmm_only']['ms_per_launch'], 'speedup', d['speedup_vs_cublas'], 'frac', d['roofline']['frac'])
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"
  done
  done
  done
done
