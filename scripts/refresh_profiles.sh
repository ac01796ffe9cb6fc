#!/bin/bash
# GPU-box half of the profile refresh: gpu tests, one ncu --set full capture
# each of K2 (C2 hot-set) and K3 (C2 YLT), and the bench launch list.
# Usage: scripts/refresh_profiles.sh TAG ; then, locally,
#   python scripts/summarize_profile.py gpurun_out/k2_TAG.ncu-rep profiles/TAG_k2_hotset.md \
#       --traffic-json profiles/k2_traffic.json --launches gpurun_out/launches_TAG.csv
TAG=$1
(timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3)
ncu --set full --clock-control none --import-source on -k regex:k2_hotset -s 1 -c 1 -o gpurun_out/k2_$TAG \
    python scripts/profile_k2.py --launches 2 > gpurun_out/ncu_k2_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_select -s 2 -c 1 -o gpurun_out/k3_$TAG \
    python scripts/profile_k2.py --launches 3 --k3 > gpurun_out/ncu_k3_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1
ls gpurun_out | grep $TAG
