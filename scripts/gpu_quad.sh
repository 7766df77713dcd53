mkdir -p gpurun_out
timeout 600 python scripts/bench_configs.py --only f4 --out gpurun_out/f4_quad.jsonl > /dev/null 2>&1; cut -c1-220 gpurun_out/f4_quad.jsonl
for e in 2 0; do FB_K1_QUAD=$e timeout 300 python scripts/ab_diag.py | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d.pop('pair_poly_env')
    print('FB_K1_QUAD=$e', ' '.join('%s: C5 %.3f prefill %.3f' % (k, v['c5_ms'], v['prefill_ms']) for k,v in d.items()))
"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_kernel -c 1 -o gpurun_out/quad_prefill_r01f -f python scripts/prof_pair.py single prefill > gpurun_out/ncu_quadpf.log 2>&1; echo "ncu rc=$?"
