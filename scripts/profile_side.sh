#!/bin/bash
# ncu --set full captures of the side K2 kernels: k2_pair (C5 short trials,
# E=100, 1M trials) and k2_dense (event-major dense kernel, C2 data, 200k trials).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k2_pair" -s 1 -c 1 -o gpurun_out/k2pair_r01 \
    python scripts/profile_k2.py --events 100 --launches 2 > gpurun_out/ncu_k2pair.log 2>&1; tail -1 gpurun_out/ncu_k2pair.log
ncu --set full --clock-control none --import-source on -k regex:"k2_dense" -s 1 -c 1 -o gpurun_out/k2dense_r01 \
    python scripts/profile_k2.py --variant dense --trials 200000 --launches 2 > gpurun_out/ncu_k2dense.log 2>&1; tail -1 gpurun_out/ncu_k2dense.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dense.csv \
    python scripts/profile_k2.py --variant dense --trials 200000 --launches 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
