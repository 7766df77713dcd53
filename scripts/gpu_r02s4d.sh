#!/bin/bash
# session-4: bench-context A/B of the K2 v2 changes (old: per-thread stores, one
# Q/K/V barrier; new: TMA store + V barrier), interleaved on one box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
  FB_K2_STORE=0 FB_K2_VSPLIT=0 timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/s4d_old$i.json 2>/dev/null; echo "old$i rc=$?"
  timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/s4d_new$i.json 2>/dev/null; echo "new$i rc=$?"
done
python - <<'PY'
import json
for n in ["old1","new1","old2","new2"]:
    d=json.loads(open(f"gpurun_out/s4d_{n}.json").read().strip().splitlines()[-1])
    print(n, round(d["value"]), "K1", round(d["roofline"]["avg_launch_ms"]*1000,1), "us K2", round(d["k2_cached_step"]["avg_launch_ms"]*1000,2), "us clk", d["clocks"]["sm_mhz"])
PY
