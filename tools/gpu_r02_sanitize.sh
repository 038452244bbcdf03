#!/bin/bash
mkdir -p gpurun_out
python -m paper_2310_02065_b200.build > /dev/null
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all calls ok|Error|error" gpurun_out/sanitize_$tool.txt | head -8
done
