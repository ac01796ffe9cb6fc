# Dense-kernel evidence: density sweep (hot set vs dense vs pre-combined), C2 dense timing, ncu --set full of k2_dense_coop.
python scripts/time_density.py > gpurun_out/density_final.jsonl 2>&1; cat gpurun_out/density_final.jsonl
python scripts/time_dense.py
ncu --set full --clock-control none --import-source on -k regex:"k2_dense" -s 1 -c 1 -o gpurun_out/k2coopfull_r01 python scripts/profile_k2.py --variant dense --trials 200000 --launches 2 > gpurun_out/ncu_coopfull.log 2>&1; tail -1 gpurun_out/ncu_coopfull.log
