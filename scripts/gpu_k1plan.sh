mkdir -p gpurun_out
timeout 600 python scripts/ab_k1_plan.py > gpurun_out/ab_k1_plan.log 2>&1; echo "rc=$?"; python -c "
import json
for l in open('gpurun_out/ab_k1_plan.log'):
    if l.startswith('{'):
        d=json.loads(l); print('%-12s %-15s %8.4f ms %.3f' % (d['case'], d['variant'], d['ms'], d['frac_hbm']))
    else: print(l.rstrip())
"
