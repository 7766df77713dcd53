mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python scripts/bench_configs.py --only c4 --out gpurun_out/c4_fused.jsonl > /dev/null 2>&1; echo "c4 rc=$?"
python -c "
import json
for l in open('gpurun_out/c4_fused.jsonl'):
    d=json.loads(l); print(d['density'], 'mask %.3f k7 %.4f k8 %.4f frac %.3f block %.3f speedup %.2f l1 %.4f %.4f' % (d['mask_ms'], d['k7_first_step_ms'], d['k8_cached_step_ms'], d['k8_frac_hbm'], d['block_ms_per_layer_32_steps'], d['speedup_vs_dense_recompute'], d['l1_sparse_only'], d['l1_with_residual']))
"
