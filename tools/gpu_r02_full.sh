#!/bin/bash
# full GPU test suite + the default bench line
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
for k in ("value", "ms_per_step", "step_ms", "spmm_only", "step_breakdown_ms", "speedup_vs_cublas", "roofline", "e2e", "secondary", "clocks", "cpu_baseline"):
    print(k, json.dumps(d.get(k))[:600])
PY
