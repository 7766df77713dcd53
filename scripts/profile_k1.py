"""Small driver for ncu captures of the hot kernels at the C2 shapes.

    python scripts/profile_k1.py [--batch 8] [--layers 4] [--reps 2]

Runs, per layer (distinct KV buffers, so no L2 reuse across launches), one
refresh (K1: refresh_kernel + split combine) and one cached step (K2).
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_05305_b200 import FlashBlockAttention  # noqa: E402
from paper_2602_05305_b200 import kernels as K  # noqa: E402

HQ, HKV, D, BLK, CTX = 32, 8, 128, 32, 32768


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--ctx", type=int, default=CTX)
    a = ap.parse_args()
    b, dev = a.batch, torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    rnd = lambda *s: torch.randn(s, device=dev, generator=g).to(torch.bfloat16)
    kc = [rnd(b, HKV, a.ctx, D) for _ in range(a.layers)]
    vc = [rnd(b, HKV, a.ctx, D) for _ in range(a.layers)]
    q = rnd(b, HQ, BLK, D)
    ki, vi = rnd(b, HKV, BLK, D), rnd(b, HKV, BLK, D)
    eng = FlashBlockAttention(a.layers, b, HQ, HKV, BLK, D, device=dev)
    out = torch.empty(b, HQ, BLK, D, device=dev, dtype=torch.bfloat16)
    for _ in range(a.reps):
        for l in range(a.layers):
            eng.refresh(l, q, kc[l], vc[l], a.ctx, ki, vi, out=out)
            eng.cached(l, q, ki, vi, out=out)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
