mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "== memcheck pair + K2 variants"
timeout 900 $S --tool memcheck python -m pytest tests/test_pair.py -q -x -k "not full_size" 2>&1 | tail -3
echo "== racecheck pair (one case)"
timeout 900 $S --tool racecheck python -m pytest tests/test_pair.py -q -x -k "refresh_vs_oracle_and_single_cta and 3-256" 2>&1 | tail -3
echo "== racecheck K2 v1/v2"
timeout 900 $S --tool racecheck python -m pytest tests/test_pair.py -q -x -k "v1_v2 and 2-32" 2>&1 | tail -3
echo "== synccheck pair + K2 v2"
timeout 900 $S --tool synccheck python -m pytest tests/test_pair.py -q -x -k "(refresh_vs_oracle_and_single_cta and 3-256) or (v1_v2 and 20-32)" 2>&1 | tail -3
} > gpurun_out/sanitize_r01f.txt 2>&1
cat gpurun_out/sanitize_r01f.txt
timeout 300 python -m pytest tests/test_pair.py -q -x 2>&1 | tail -2
