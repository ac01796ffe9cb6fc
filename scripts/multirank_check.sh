# Multi-rank control flow of bench.py on a one-GPU box: two ranks share cuda:0 over gloo
# (NCCL refuses duplicate GPUs), then the reference arm under torchrun (rank 1 exits).
set -x
mkdir -p gpurun_out
ARE_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/mr_bench2.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/mr_bench2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/mr_ref2.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/mr_ref2.log
