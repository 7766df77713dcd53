mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_pair.py -x -q > gpurun_out/pair_tests.log 2>&1; echo "pair rc=$?"; tail -2 gpurun_out/pair_tests.log
for kk in 1 0; do
FB_KV_KEEP=$kk timeout 300 python scripts/ab_pair.py > gpurun_out/ab_pair_kk$kk.log 2>&1; echo "ab kv_keep=$kk rc=$?"; python -c "
import json,sys
for l in open('gpurun_out/ab_pair_kk$kk.log'):
    if l.startswith('{'):
        d=json.loads(l); print('%-34s %-7s %8.3f ms %7.1f TF %.3f' % (d['case'], d['variant'], d['ms'], d['tflops'], d['frac_tensor']))
"
done
for v in pair single; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"pair_kernel|refresh_kernel" -s 1 -c 1 -o gpurun_out/c5kk_$v -f python scripts/prof_pair.py $v c5 > gpurun_out/ncu_c5kk_$v.log 2>&1; echo "ncu $v rc=$?"
done
