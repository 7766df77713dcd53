#!/bin/bash
# evidence for the fused K5 and the host-buffer cached step: sanitizer + ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "== memcheck: fused K5 (score_fused_kernel, score_mass_kernel), host-buffer cached step"
timeout 1200 $S --tool memcheck python -m pytest tests/test_k5_fused.py tests/test_dropin_host.py -m gpu -q -x 2>&1 | tail -3
echo "== racecheck: fused K5 (ragged tails, split items)"
timeout 1200 $S --tool racecheck python -m pytest tests/test_k5_fused.py -m gpu -q -x -k "1000 or 16384" 2>&1 | tail -3
echo "== synccheck: fused K5"
timeout 1200 $S --tool synccheck python -m pytest tests/test_k5_fused.py -m gpu -q -x -k "1000" 2>&1 | tail -3
} > gpurun_out/sanitize_k5.txt 2>&1
cat gpurun_out/sanitize_k5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -c 2 -o gpurun_out/k5_fused_final -f python scripts/ab_k5_fused.py > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score|topk" --csv python scripts/ab_k5_fused.py > gpurun_out/k5_fused_launches.csv 2>&1; echo "launches rc=$?"
