mkdir -p gpurun_out
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs_r01f.jsonl > gpurun_out/configs_r01f.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/configs_r01f.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
