#!/bin/bash
# One GPU iteration: gpu tests, bench, ncu of K2.  Usage: scripts/gpu_cycle.sh TAG [pytest-args]
TAG=$1; shift
(timeout 900 python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -4)
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value', d['value'], 'step_ms', d['ms_per_step'], 'k2_ms', d['roofline']['kernel_ms'], 'e2e_ms', d['e2e']['ms_per_step'])"
ncu --set full --clock-control none --import-source on -k regex:"k2_(relay|hotset)" -s 1 -c 1 -o gpurun_out/k2_$TAG python scripts/profile_k2.py --launches 2 ${K2_VARIANT:+--variant $K2_VARIANT} > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
