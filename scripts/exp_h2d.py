"""Pinned H2D bandwidth: one copy stream vs two vs four, chunk sizes as in the
e2e path (Q 4 MiB, K/V 1 MiB per layer at C2 b=16)."""
import time, torch
dev = torch.device("cuda")
L = 36
hq = torch.randn((L, 16, 32, 32, 128)).to(torch.bfloat16).pin_memory()
hk = torch.randn((L, 16, 8, 32, 128)).to(torch.bfloat16).pin_memory()
hv = torch.randn((L, 16, 8, 32, 128)).to(torch.bfloat16).pin_memory()
dq, dk, dv = hq.to(dev), hk.to(dev), hv.to(dev)
nbytes = (hq.numel() + hk.numel() + hv.numel()) * 2
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(10):
            for l in range(L):
                for j, (d, h) in enumerate(((dq, hq), (dk, hk), (dv, hv))):
                    with torch.cuda.stream(streams[(l * 3 + j) % ns]):
                        d[l].copy_(h[l], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{ns} copy streams: {nbytes * 10 / dt / 1e9:.1f} GB/s", flush=True)
whole = time.perf_counter()
for it in range(10):
    dq.copy_(hq, non_blocking=True); dk.copy_(hk, non_blocking=True); dv.copy_(hv, non_blocking=True)
torch.cuda.synchronize()
print(f"whole-tensor copies: {nbytes * 10 / (time.perf_counter() - whole) / 1e9:.1f} GB/s")
