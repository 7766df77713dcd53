"""C1 drop-in replay: cProfile of the reference run_sequence with the device
functions patched in (token-threshold), to see the per-call host overhead."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import numpy as np
import flashblock as fbref
from paper_2602_05305_b200.replay import patch_reference_simulator
model = fbref.SyntheticModel(fbref.ModelConfig(num_layers=2, num_heads=4, head_dim=64, seed=0, dtype=np.float32))
args = dict(prompt_len=4096, num_blocks=1, block_size=32, steps_per_block=32,
            policy=fbref.ReuseConfig(tau=2, mode="token-threshold"), seed=0, unmask_per_step=1)
base = fbref.run_sequence(model, **args)
print("cpu tok/s", 32 / (sum(t.wall_ns for t in base.traces) / 1e9))
with patch_reference_simulator(fbref.simulator):
    fbref.run_sequence(model, **args)
    gpu = fbref.run_sequence(model, **args)
    print("gpu tok/s", 32 / (sum(t.wall_ns for t in gpu.traces) / 1e9))
    pr = cProfile.Profile(); pr.enable(); fbref.run_sequence(model, **args); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
# the same on the CPU reference
pr = cProfile.Profile(); pr.enable(); fbref.run_sequence(model, **args); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
