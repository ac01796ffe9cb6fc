#!/bin/bash
# A/B of K2 builds: gpu tests (default build), bench for each variant, optional ncu.
# Usage: scripts/gpu_ab.sh TAG "name=ENV ..." ...   e.g. legacy=ARE_K2_LEGACY=1 t512=ARE_LIB=build/lib_t512.so
# NCU=1 captures the default build's K2 with ncu --set full.
TAG=$1; shift
(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4)
run() {
  name=$1; shift
  env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_$name.json 2> gpurun_out/bench_${TAG}_$name.err
  tail -1 gpurun_out/bench_${TAG}_$name.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$name.json')); print('$name', 'value %.4g' % d['value'], 'k2_ms %.4f' % d['roofline']['kernel_ms'], 'pre_ms %.4f' % d['precombined_k2']['kernel_ms'])"
}
run default X=1
for spec in "$@"; do name=${spec%%=*}; envs=${spec#*=}; run $name $envs; done
if [ -n "$NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"k2_(stream|hotset)" -s 1 -c 1 -o gpurun_out/k2_$TAG python scripts/profile_k2.py --launches 2 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
