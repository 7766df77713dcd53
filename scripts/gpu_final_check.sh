mkdir -p gpurun_out
bash scripts/gpu_round_check.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_torchrun.log 2>&1; echo "torchrun rc=$?"; tail -1 gpurun_out/bench_torchrun.log | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --mode splitkv --steps 3 --warmup 3 > gpurun_out/bench_splitkv.log 2>&1; echo "splitkv rc=$?"; tail -1 gpurun_out/bench_splitkv.log | cut -c1-300
