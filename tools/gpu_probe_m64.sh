#!/bin/bash
# M = 64 sparse MMA TMEM layout probes (tools/probe_m64.cu); each call its own process so a
# rejected address form cannot take the others down
for args in "0 0 0" "0 16 0" "1 0 0" "1 16 0" "1 0 16" "1 0 64" "1 16 16"; do
  timeout 30 ./tools/probe_m64 $args > gpurun_out/probe_m64_${args// /_}.txt 2>&1
  echo "args=$args rc=$?"
done
