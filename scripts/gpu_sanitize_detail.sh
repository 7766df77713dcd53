mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool racecheck --racecheck-report hazard python -m pytest tests/test_pair.py -q -x -k "refresh_vs_oracle_and_single_cta and 3-256" > gpurun_out/race_pair.txt 2>&1
grep -v "Host Frame" gpurun_out/race_pair.txt | grep -v "^\s*$" | head -12
timeout 900 $S --tool racecheck python -m pytest tests/test_pair.py -q -x -k "block_causal and 4-512" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_pair.py tests/test_prefill.py -q -x 2>&1 | tail -2
