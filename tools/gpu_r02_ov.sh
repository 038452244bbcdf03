#!/bin/bash
mkdir -p gpurun_out
for a in "" "--no-overlap"; do
timeout 300 python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-secondary $a > gpurun_out/b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$a', d['value'], d['step_ms'], d['step_breakdown_ms']['compress_all_layers'], d['step_breakdown_ms']['spmm_all_layers'], d['step_breakdown_ms']['decompress_all_layers'], d['clocks'])"
done
