#!/bin/bash
# Full GPU-side refresh of the committed evidence (one box, ~15 min):
# gpu tests + smoke, the bench line (with the CPU baseline), the reference arm,
# a torchrun world-1 bench, ncu captures of K2/K3 + the launch list, sweeps.
# Usage: scripts/round_refresh.sh TAG      (outputs in gpurun_out/*_TAG*)
TAG=$1
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; tail -c 600 gpurun_out/bench_full_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun_$TAG.json 2> gpurun_out/bench_torchrun_$TAG.err
tail -c 300 gpurun_out/bench_torchrun_$TAG.json
ncu --set full --clock-control none --import-source on -k regex:"k2_(relay|hotset)" -s 1 -c 1 -o gpurun_out/k2_$TAG \
    python scripts/profile_k2.py --launches 2 > gpurun_out/ncu_k2_$TAG.log 2>&1
ARE_PACKED_IDS=1 ncu --set full --clock-control none --import-source on -k regex:"k2_relay" -s 1 -c 1 -o gpurun_out/k2pk_$TAG \
    python scripts/profile_k2.py --launches 2 > gpurun_out/ncu_k2pk_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_select -s 2 -c 1 -o gpurun_out/k3_$TAG \
    python scripts/profile_k2.py --launches 3 --k3 > gpurun_out/ncu_k3_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k2_layers$" -s 1 -c 1 -o gpurun_out/k2l_$TAG \
    python scripts/profile_layers.py > gpurun_out/ncu_k2l_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k2_layers_pre$" -s 1 -c 1 -o gpurun_out/k2lp_$TAG \
    python scripts/time_layers.py --trials 200000 --reps 1 > gpurun_out/ncu_k2lp_$TAG.log 2>&1
timeout 600 python scripts/entry_e2e.py > gpurun_out/entry_e2e_$TAG.json 2> gpurun_out/entry_e2e_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1
timeout 1500 python scripts/sweep.py --only c3,c4,c5,refsweeps --out gpurun_out/sweep_$TAG.json > gpurun_out/sweep_$TAG.log 2>&1; tail -2 gpurun_out/sweep_$TAG.log
python scripts/host_path.py > gpurun_out/host_path_$TAG.log 2>&1
python scripts/time_density.py > gpurun_out/density_$TAG.log 2>&1
ls gpurun_out | grep $TAG
