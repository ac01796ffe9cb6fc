#!/bin/bash
# C3 fused multi-layer iteration: parity tests, C3 timing (1M trials), ncu of k2_layers.  Usage: scripts/gpu_c3.sh TAG
TAG=$1
(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3)
timeout 900 python scripts/sweep.py --only c3 --out gpurun_out/c3_$TAG.json 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('step_ms','fused_step_ms','fused_bitwise_equal_unfused')})"
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:"k2_layers" -s 1 -c 1 -o gpurun_out/k2l_$TAG python scripts/profile_layers.py > gpurun_out/ncu_k2l_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k2l_$TAG.log
fi
