"""K1 under sustained load: graph of 36 back-to-back launches (distinct KV,
C2 b=16) replayed for ~3 s per variant, nvidia-smi sampled meanwhile:
product kernel vs diagnostic variants (no softmax math / no S load)."""
import ctypes, os, subprocess, sys, threading, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
lib = _lib.load(); lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
HKV, D, CTX, L, b = 8, 128, 32768, 12, int(os.environ.get("B", "16"))
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((b * HKV, 128, D), device="cuda", generator=g).to(torch.bfloat16)
ks = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
vs = [torch.randn((b * HKV, CTX, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(L)]
o = torch.empty((b * HKV, 128, D), device="cuda", dtype=torch.float32)
l = torch.empty((b * HKV, 128), device="cuda", dtype=torch.float32)
byts = 2 * b * HKV * CTX * D * 2

def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line: out.append(line.strip())
    p.terminate()

for diag, name in ((0, "product"), (2, "no-softmax-no-Sload"), (0, "product")):
    lib.fb_debug_set_k1_diag(diag)
    fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(L)]
    s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s): fn()
    for _ in range(20): gr.replay()
    torch.cuda.synchronize()
    stop, lines = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, lines)); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 60
    e0.record()
    for _ in range(n): gr.replay()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    t = e0.elapsed_time(e1) / (n * L)
    clk = sorted(float(x.split(",")[0]) for x in lines if x)
    pw = sorted(float(x.split(",")[1]) for x in lines if x)
    print(f"{name:22s} {t*1000:.1f} us/launch {byts/t/1e6:.0f} GB/s | sm clock median {clk[len(clk)//2]:.0f} MHz, "
          f"power median {pw[len(pw)//2]:.0f} W (samples {len(lines)})", flush=True)
lib.fb_debug_set_k1_diag(0)
