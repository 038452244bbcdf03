#!/bin/bash
# the multi-rank bench path (strong scaling, all-gather legs) with 2 ranks on the one GPU over gloo
mkdir -p gpurun_out
VENOM_BENCH_DEVICE=0 VENOM_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo rc=$?; tail -3 gpurun_out/bench_2rank.err
python -c "
import json; d=json.load(open('gpurun_out/bench_2rank.json')); print({k: d[k] for k in ('value','n_gpus','scaling','ms_per_step','config','allgather_C','gpu_launches')})"
