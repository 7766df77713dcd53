mkdir -p gpurun_out
P=paper_2602_05305_b200
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_graph_replay.py tests/test_counters.py -x -q > gpurun_out/k2v2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/k2v2_tests.log
cp $P/libfb200.so /tmp/libA.so; cp $P/libfb200.so /tmp/libB.so
for b in 16 4 32; do timeout 300 python scripts/ab_k2.py /tmp/libA.so /tmp/libB.so $b FB_K2_V2=0 FB_K2_V2=1 2>&1 | tail -2; done
timeout 300 python bench.py --no-cpu > gpurun_out/bench_k2v2.log 2>&1; tail -1 gpurun_out/bench_k2v2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_ms'], d['k2_cached_step'], d['clocks'])"
FB_K2_V2=0 timeout 300 python bench.py --no-cpu > gpurun_out/bench_k2v1.log 2>&1; tail -1 gpurun_out/bench_k2v1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench v1', d['value'], d['roofline']['avg_launch_ms'], d['k2_cached_step'], d['clocks'])"
