timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu --batch 16 > gpurun_out/bench_b16.log 2>&1; echo "bench16 rc=$?"
timeout 600 python bench.py --mode splitkv --steps 3 --warmup 3 --batch 1 --layers 8 > gpurun_out/bench_splitkv.log 2>&1; echo "splitkv rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --mode splitkv --gpus 1 --steps 3 --warmup 3 --batch 1 --layers 8 > gpurun_out/bench_splitkv_trun.log 2>&1; echo "splitkv-torchrun rc=$?"
tail -2 gpurun_out/bench_splitkv.log; tail -2 gpurun_out/bench_splitkv_trun.log
