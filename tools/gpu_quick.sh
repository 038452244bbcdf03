#!/bin/bash
# quick GPU check: build, GPU tests (optionally filtered by $1), GPT-3 bench line without the slow legs
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu -x ${1:+-k "$1"} > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --no-secondary ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench_quick.json"))
except Exception as e:
    print("bench failed", e); print(open("gpurun_out/bench_quick.err").read()[-2000:]); raise SystemExit
print("value", d["value"], "ms/step", d["step_ms"], "spmm", d["spmm_only"], "breakdown", d["step_breakdown_ms"], "speedup", d["speedup_vs_cublas"], d["clocks"])
PY
