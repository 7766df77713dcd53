"""bench.py's reference arm runs on the host CPU only, so its JSON contract is
checked here without a GPU: one line, the C2 metric / unit / direction, the
reference-arm extras (impl, cpu_baseline with kind / cores / sample, an e2e
block with zero copy bytes)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "flashblock")),
                    reason="reference not installed at baseline/_ref")
def test_reference_arm_line_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("block-diffusion tokens/s") and d["unit"] == "tokens/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] == 1 and d["warmup"] >= 3
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0 \
        and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "flashblock")),
                    reason="reference not installed at baseline/_ref")
def test_reference_arm_under_torchrun_prints_one_line_with_all_blas_threads():
    """The driver launches the reference arm like ours (torchrun for N > 1):
    rank 0 alone runs and prints, the other rank exits 0 without work, and the
    BLAS pool gets every core although torchrun sets OMP_NUM_THREADS=1."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517",
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] == os.cpu_count()
