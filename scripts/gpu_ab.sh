#!/bin/bash
# A/B of the in-tree library against scripts/micro/libfb200_old.so on one box.
for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export FB_LIB_PATH=$PWD/scripts/micro/libfb200_old.so; else unset FB_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/ab_$v$i.log 2>&1
    tail -1 gpurun_out/ab_$v$i.log | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['value']), round(d['ms_per_step'],2), 'k1', round(d['roofline']['avg_launch_ms']*1000,1), 'k2', round(d['k2_cached_step']['avg_launch_ms']*1000,2), d['clocks']['sm_mhz'])"
  done
done
