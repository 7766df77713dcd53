"""K1 at b=32 (C2) under sustained load: graphs of 4 launches on distinct KV
replayed for ~3 s, per-replay time and NVML SM clock / power, for the product
kernel (diag 0) and the one without softmax math (diag 1).  Shows how much of
the bench's K1 shortfall at power-capped clocks is the softmax."""
import ctypes, json, os, sys, threading, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05305_b200 import kernels as K, _lib
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
lib = _lib.load(); lib.fb_debug_set_k1_diag.argtypes = [ctypes.c_int]
HKV, D, CTX, b, nd = 8, 128, 32768, 32, 4
groups = b * HKV
gen = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((groups, 128, D), device="cuda", generator=gen).to(torch.bfloat16)
ks = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
vs = [torch.randn((groups, CTX, D), device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nd)]
o = torch.empty((groups, 128, D), device="cuda", dtype=torch.float32)
l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
byts = 2 * groups * CTX * D * 2
for diag in [int(x) for x in os.environ.get("DIAGS", "0,1,0,1").split(",")]:
    lib.fb_debug_set_k1_diag(diag)
    fn = lambda: [K.attention_partial(q, ks[i], vs[i], 0, CTX, None, o, l) for i in range(nd)]
    s = torch.cuda.Stream(); fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): fn()
    clk, pw = [], []
    stop = False
    def samp():
        while not stop:
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
            time.sleep(0.01)
    th = threading.Thread(target=samp); th.start()
    times = []
    t_end = time.time() + 3.0
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / nd)
    stop = True; th.join()
    times.sort()
    med = times[len(times) // 2]
    print(json.dumps({"diag": diag, "launches": len(times) * nd, "median_us": round(med * 1000, 1),
                      "first_us": round(times[0] * 1000, 1), "gbs_median": round(byts / med / 1e6),
                      "sm_mhz_median": sorted(clk)[len(clk) // 2], "power_w_median": round(sorted(pw)[len(pw) // 2])}), flush=True)
lib.fb_debug_set_k1_diag(0)
