mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 120 python scripts/debug_rr.py
timeout 300 python scripts/ab_pair.py > gpurun_out/ab_pair_rr.log 2>&1; echo "ab rc=$?"; python -c "
import json,sys
for l in open('gpurun_out/ab_pair_rr.log'):
    if l.startswith('{'):
        d=json.loads(l); print('%-34s %-7s %8.3f ms %7.1f TF %.3f' % (d['case'], d['variant'], d['ms'], d['tflops'], d['frac_tensor']))
" | grep F4
