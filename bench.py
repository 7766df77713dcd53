"""Benchmark: FlashBlock attention on B200 (BASELINE.json metric).

N = 1 (default): config C2 (BASELINE.json configs[1]).  One bench *step* =
one block of block-diffusion decoding: L=36 layers of 8B-class GQA attention
(32 q / 8 kv heads, head_dim 128), batch b, block B=32, committed context
N=32768, S=32 diffusion steps with 1 unmask per step and tau=2 -> the refresh
schedule is [Recompute, Reuse x31] (policy.refresh_schedule; the reference
simulator's decisions).  Refresh steps run K1 (tcgen05 refresh over the KV
cache) + K2 (internal + merge); cached steps run K2 only.  The
full-recompute baseline runs K1+K2 on every step.  Synthetic bf16 inputs,
N(0,1), seeded; every layer has its own KV cache (inputs > L2).  The line also
carries the schedule sweep (unmask per step x tau) against full recompute.

N > 1: the same C2 line with N ranks each running its own batch (sequences
are independent: no data-path collective, weak scaling, value = all ranks'
tokens / max-over-ranks time), so the curve over N is one workload; the run
then measures config C3 and attaches it as "c3_split_kv".

--workload c3 (main line) / "c3_split_kv": config C3 (configs[2]) -- 128K
context, the KV cache of each sequence split along the sequence over the N
ranks (strong scaling: the same b sequences whatever N).  Refresh step per layer: K1 on
the local shard -> ONE packed exchange of the (O, LSE) partials (grouped
NCCL send/recv by kv-group chunk) -> K3 merge of this rank's kv-head shard
-> K2 on the shard; the 31 cached steps run K2 on the head shard only (no
KV, no exchange).  Time = max over ranks of CUDA events on each rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--workload c2|c3]

--gpus N without torchrun re-launches itself under torch.distributed.run
with N local ranks (127.0.0.1 rendezvous).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# C2 (BASELINE.json configs[1]) shapes
LAYERS, HQ, HKV, D, BLK, CTX = 36, 32, 8, 128, 32, 32768
STEPS_PER_BLOCK, UNMASK_PER_STEP, TAU = 32, 1, 2
METRIC = "block-diffusion tokens/s (FlashBlock attention, C2: 8B-class GQA, 32K ctx)"
UNIT = "tokens/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region.

    NVML (pynvml) polled from a thread every 5 ms on the device selected by
    UUID, so even a sub-second timed region gets tens of samples; falls back
    to `nvidia-smi -lms 50` when NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu):
        # a UUID ("GPU-...") names the physical device whatever CUDA_VISIBLE_DEVICES says
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, int, float]] = []
        self.t = None
        self._stop = threading.Event()
        self._nvml = None
        self._smax = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = (nv.nvmlDeviceGetHandleByUUID(self.gpu) if str(self.gpu).startswith(("GPU-", "MIG-"))
                 else nv.nvmlDeviceGetHandleByIndex(int(self.gpu)))
            self._smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nvml = (nv, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._pump, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self._nvml
        while not self._stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append((sm, rs, pw))
            except Exception:
                pass
            self._stop.wait(0.005)

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self._nvml is not None:
            nv, _ = self._nvml
            self._stop.set()
            self.t.join(timeout=2)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({nm for _, rs, _ in self.samples for nm, bit in bits.items() if rs & bit})
            sm = [x[0] for x in self.samples]
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self._smax,
                    "reasons": reasons, "samples": len(sm), "sampler": "nvml 5 ms",
                    "power_w_max": max((x[2] for x in self.samples), default=None), "gpu": str(self.gpu)}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": "nvidia-smi 50 ms",
                "gpu": str(self.gpu)}


def gpu_smi_id(device) -> str:
    """nvidia-smi --id for a torch device: its UUID (GPU-xxxxxxxx-...), so the
    sampler watches the device this process really runs on."""
    import torch

    try:
        u = str(torch.cuda.get_device_properties(device).uuid)
        if u:
            return u if u.startswith(("GPU-", "MIG-")) else f"GPU-{u}"
    except Exception:
        pass
    return str(device.index if device.index is not None else 0)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- CPU reference


def _reference_module():
    """The unmodified reference package (baseline/_ref) if installed, else the
    oracle port.  Used only for the cpu_baseline / --impl reference legs.
    Returns (kind, attention_streamed, merge_partials, attention_with_reuse,
    CacheEntry)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "flashblock")):
        sys.path.insert(0, ref_dir)
        try:
            import flashblock.attention as A

            return ("reference", A.attention_streamed, A.merge_partials, A.attention_with_reuse,
                    A.CacheEntry)
        except Exception:
            sys.path.remove(ref_dir)
    from oracle import flashblock_oracle as O

    def reuse(q, entry, k_in, v_in, scale=None, tile_size=64):
        return O.with_reuse(q, entry.partial, True, k_in, v_in, scale, tile_size)

    class Entry:
        def __init__(self, partial, step_created, block_id=-1):
            self.partial = partial

    return "port", O.streamed, O.merge, reuse, Entry


def cpu_layer_block(ctx: int, sched, reps: int = 1):
    """Time the reference CPU path over ONE layer x all Hkv kv-heads x one
    whole block schedule at b=1, routed exactly as the reference step driver
    (simulator.py:412-434): a Recompute step concatenates the committed rows
    with the block's K/V and runs attention_streamed + merge_partials, caching
    the external partial; a Reuse step runs attention_with_reuse against it.
    Per kv-head the G=4 query heads are stacked (128 fp32 rows, d=128; rows
    are independent); tile 512 as simulator.py:87.  Returns the
    best-of-`reps` seconds and the reference kind."""
    import numpy as np

    kind, streamed, merge, reuse, Entry = _reference_module()
    rng = np.random.Generator(np.random.Philox(1234))
    rows = (HQ // HKV) * BLK
    heads = []
    for _ in range(HKV):
        heads.append(tuple(rng.standard_normal(s).astype(np.float32) for s in
                           ((rows, D), (ctx, D), (ctx, D), (BLK, D), (BLK, D))))
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        entries = [None] * HKV
        for dec in sched:
            for h, (q, k, v, ki, vi) in enumerate(heads):
                if dec == "Recompute":
                    keys = np.concatenate([k, ki])
                    values = np.concatenate([v, vi])
                    ext, inn = streamed(q, keys, values, ctx, None, 512)
                    merge(ext, inn)
                    entries[h] = Entry(ext, 0, 0)
                else:
                    reuse(q, entries[h], ki, vi, None, 512)
        best = min(best, time.perf_counter() - t0)
    return kind, best


def cpu_tokens_per_s(t_layer_block: float) -> float:
    """tokens/s of the whole C2 job from one layer's block at b=1: the block
    yields BLK tokens per sequence after LAYERS such layers; batch cancels
    (tokens and work both scale with b).  Extrapolation factor: x LAYERS."""
    return BLK / (LAYERS * t_layer_block)


def _sched_names(per_step: int = UNMASK_PER_STEP, tau: int = TAU):
    from paper_2602_05305_b200.policy import ReuseConfig, refresh_schedule

    return [d.value for d in refresh_schedule(ReuseConfig(tau=tau), BLK, STEPS_PER_BLOCK, per_step)]


_BLAS_LIMITS = None


def _blas_threads() -> int:
    """Give the host BLAS every core (torchrun sets OMP_NUM_THREADS=1 per rank,
    and numpy may already be loaded, so the environment alone is not enough)
    and return the thread count its pool actually uses -- the `cores` the CPU
    legs report."""
    global _BLAS_LIMITS
    import numpy  # noqa: F401  (loads the BLAS whose pool is set below)

    try:
        from threadpoolctl import threadpool_info, threadpool_limits

        _BLAS_LIMITS = threadpool_limits(limits=os.cpu_count(), user_api="blas")
        n = [i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001 (threadpoolctl missing: report what was asked for)
        return os.cpu_count() or 1


def _cpu_sample_text(kind, t, sched, reps, cores=None):
    n_ref = sum(1 for d in sched if d == "Recompute")
    return (f"1 layer x {HKV} kv-heads (G={HQ // HKV} stacked -> {(HQ // HKV) * BLK} fp32 rows, d={D}) "
            f"x one {STEPS_PER_BLOCK}-step block ({n_ref} refresh over {CTX} keys via attention_streamed + "
            f"merge_partials, {STEPS_PER_BLOCK - n_ref} attention_with_reuse), b=1, tile 512, best of {reps}: "
            f"{t:.3f} s; extrapolated x{LAYERS} layers (batch cancels); {kind} on {cores or os.cpu_count()} host "
            f"threads ({cpu_model()})")


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    threads = str(os.cpu_count())
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, threads)
    cores = _blas_threads()
    sched = _sched_names()
    for _ in range(args.warmup):
        cpu_layer_block(CTX, sched, reps=1)
    vals, times = [], []
    kind = None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        kind, t = cpu_layer_block(CTX, sched, reps=1)
        times.append(t)
        vals.append(cpu_tokens_per_s(t))
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        # one bench step = one C2 block for the whole batch: b x the per-sequence block time
        "ms_per_step": 1000.0 * args.batch * BLK / value if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic N(0,1), seeded",
        "config": _config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": _cpu_sample_text(kind, statistics.median(times), sched, 1, cores),
                         "extrapolation": f"x{LAYERS} layers (measured: a whole layer-block at b=1)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "measured_s_per_step": statistics.median(times),
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def _config(args, world: int = 1):
    return {"workload": "C2: 8B-class GQA block-diffusion attention, 32K ctx, FlashBlock tau=2",
            "parallelism": f"dp{world} (independent sequences per rank, no data-path collective)",
            "global_batch": args.batch * world,
            "layers": LAYERS, "batch_per_gpu": args.batch, "q_heads": HQ, "kv_heads": HKV,
            "head_dim": D, "block": BLK, "ctx": CTX, "steps_per_block": STEPS_PER_BLOCK,
            "unmask_per_step": UNMASK_PER_STEP, "tau": TAU,
            "l2": f"inputs larger than L2 (distinct KV cache per layer: "
                  f"{2 * args.batch * HKV * CTX * D * 2 / 1e9:.2f} GB/layer)"}


# ---------------------------------------------------------------- GPU arm


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_2602_05305_b200 import FlashBlockAttention, _lib
    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.policy import Decision, ReuseConfig, refresh_schedule

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    b = args.batch
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)

    def rnd(*shape):
        return torch.randn(shape, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)

    cap = CTX
    kc = [rnd(b, HKV, cap, D) for _ in range(LAYERS)]
    vc = [rnd(b, HKV, cap, D) for _ in range(LAYERS)]
    qs = [rnd(b, HQ, BLK, D) for _ in range(LAYERS)]
    kis = [rnd(b, HKV, BLK, D) for _ in range(LAYERS)]
    vis = [rnd(b, HKV, BLK, D) for _ in range(LAYERS)]
    outs = [torch.empty(b, HQ, BLK, D, device=dev, dtype=torch.bfloat16) for _ in range(LAYERS)]
    eng = FlashBlockAttention(LAYERS, b, HQ, HKV, BLK, D, device=dev, config=ReuseConfig(tau=TAU))
    groups, rows = b * HKV, (HQ // HKV) * BLK
    # the full-recompute baseline and the K1 roofline leg write the partial in
    # the engine's cached-partial layout (bf16 O, fp32 LSE)
    o_scr = torch.empty(groups, rows, D, device=dev, dtype=eng.ext_dtype)
    EXT_B = eng.o_ext.element_size()
    l_scr = torch.empty(groups, rows, device=dev, dtype=torch.float32)
    sched = refresh_schedule(ReuseConfig(tau=TAU), BLK, STEPS_PER_BLOCK, UNMASK_PER_STEP)
    n_ref = sum(1 for d in sched if d is Decision.RECOMPUTE)

    def block_flashblock():
        eng.begin_block(0)
        for s, dec in enumerate(sched):
            for l in range(LAYERS):
                if dec is Decision.RECOMPUTE:
                    eng.refresh(l, qs[l], kc[l], vc[l], CTX, kis[l], vis[l], out=outs[l])
                else:
                    eng.cached(l, qs[l], kis[l], vis[l], out=outs[l])

    def block_full():
        for s in range(STEPS_PER_BLOCK):
            for l in range(LAYERS):
                eng.full_recompute(qs[l], kc[l], vc[l], CTX, kis[l], vis[l], out=outs[l],
                                   o_scratch=o_scr, lse_scratch=l_scr)

    stream = torch.cuda.Stream(device=dev)

    def capture(fn):
        fn()  # eager warm-up sizes the workspace before capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        before = lib.fb_launch_count()
        with torch.cuda.graph(g, stream=stream):
            fn()
        launches = lib.fb_launch_count() - before
        torch.cuda.synchronize()
        return g, launches

    g_fb, launches_fb = capture(block_flashblock)
    g_full, launches_full = capture(block_full)

    def timed(graph, steps, warmup):
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    sampler = ClockSampler(gpu_smi_id(dev))
    sampler.start()
    ms_fb = timed(g_fb, args.steps, args.warmup)
    clocks = sampler.stop()

    tokens = world * b * BLK * args.steps
    value = tokens / (ms_fb / 1000.0)

    # ---- K1 roofline: refresh kernel pair (tcgen05 + split combine) timed alone
    kv_bytes = 2 * b * HKV * CTX * D * 2
    k1_bytes = kv_bytes + b * HQ * BLK * D * 2 + b * HQ * BLK * D * EXT_B + b * HQ * BLK * 4
    k1_flops = 4 * b * HQ * BLK * CTX * D
    qg = [K.gqa_view(qs[l], HKV) for l in range(LAYERS)]
    kg = [kc[l].view(groups, cap, D) for l in range(LAYERS)]
    vg = [vc[l].view(groups, cap, D) for l in range(LAYERS)]
    # K1 and K2 timed alone, each as a CUDA graph of LAYERS back-to-back launches on
    # distinct per-layer buffers (no host gaps, no L2 reuse), CUDA events on the
    # replay stream
    def graph_of(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        torch.cuda.synchronize()
        return g

    def k1_all():
        for l in range(LAYERS):
            K.attention_partial(qg[l], kg[l], vg[l], 0, CTX, None, o_scr, l_scr)

    def k2_all():  # the block's cached steps (31 x 36 launches): a 36-launch graph
        for _ in range(STEPS_PER_BLOCK - 1):  # would mostly time the graph launch
            for l in range(LAYERS):
                eng.cached(l, qs[l], kis[l], vis[l], out=outs[l])

    def time_graph(g, reps=3):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()  # graphs replay on the current stream; events on the same stream
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # timed right after the FlashBlock region (same thermal / power state as the
    # step they explain), before the much heavier full-recompute comparison
    g_k1, g_k2 = graph_of(k1_all), graph_of(k2_all)
    k1_ms = time_graph(g_k1) / LAYERS
    k2_ms = time_graph(g_k2) / (LAYERS * (STEPS_PER_BLOCK - 1))

    ms_full = timed(g_full, max(1, args.steps // 2), max(3, args.warmup // 2))
    steps_full = max(1, args.steps // 2)
    full_value = world * b * BLK * steps_full / (ms_full / 1000.0)
    k2_bytes = (b * HQ * BLK * D * 2 + 2 * b * HKV * BLK * D * 2 + b * HQ * BLK * D * EXT_B
                + b * HQ * BLK * 4 + b * HQ * BLK * D * 2)

    peak, peak_kind = _peaks()
    achieved = k1_bytes / (k1_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                tj = json.load(fh)
            ent = tj.get("by_batch", {}).get(str(b))
            if ent is not None:
                traffic = ent.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e: public API, host buffers, copies in the timed region
    e2e = run_e2e(args, eng, kc, vc, dev, sched, world)

    # ---- schedule sweep: unmask per step x tau, each against the
    # full recompute of the same block; every point is one graph of a whole block
    sweep = []
    if not args.no_sweep:
        ms_full_block = ms_full / steps_full
        for per_step in (1, 2, 3):
            for tau in (2, 3):
                sch = refresh_schedule(ReuseConfig(tau=tau), BLK, STEPS_PER_BLOCK, per_step)
                nr = sum(1 for d in sch if d is Decision.RECOMPUTE)

                def blk(sch=sch):
                    eng.begin_block(0)
                    for dec in sch:
                        for l in range(LAYERS):
                            if dec is Decision.RECOMPUTE:
                                eng.refresh(l, qs[l], kc[l], vc[l], CTX, kis[l], vis[l], out=outs[l])
                            else:
                                eng.cached(l, qs[l], kis[l], vis[l], out=outs[l])

                g_s, _ = capture(blk)
                reps = 3 if nr < STEPS_PER_BLOCK else 2
                ms_s = timed(g_s, reps, 1) / reps
                del g_s
                sweep.append({"unmask_per_step": per_step, "tau": tau,
                              "refresh_steps": f"{nr}/{STEPS_PER_BLOCK}",
                              "tokens_per_s": world * b * BLK / (ms_s / 1000.0), "ms_per_block": ms_s,
                              "speedup_vs_full_recompute": ms_full_block / ms_s,
                              "clears_1p4x": ms_full_block / ms_s >= 1.4})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ.setdefault(var, str(os.cpu_count()))
        cores = _blas_threads()
        names = _sched_names()
        kind, t_lb = cpu_layer_block(CTX, names, reps=2)
        cpu = {"value": cpu_tokens_per_s(t_lb), "unit": UNIT, "cores": cores, "kind": kind,
               "cpu_model": cpu_model(), "sample": _cpu_sample_text(kind, t_lb, names, 2, cores),
               "extrapolation": f"x{LAYERS} layers (measured: a whole layer-block at b=1)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_fb / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) bf16, seeded; random KV cache per layer",
            "config": _config(args, world),
            "attention_ms_per_diffusion_step": ms_fb / args.steps / STEPS_PER_BLOCK,
            "full_recompute": {"value": full_value, "unit": UNIT,
                               "ms_per_step": ms_full / steps_full,
                               "attention_ms_per_diffusion_step": ms_full / steps_full / STEPS_PER_BLOCK},
            "speedup_vs_full_recompute": value / full_value,
            "refresh_schedule": f"{n_ref} refresh / {STEPS_PER_BLOCK} steps",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "K1 refresh (refresh_kernel<128> + split combine)",
                         "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": k1_ms,
                         "peak_kind": peak_kind,
                         "tensor_tflops": k1_flops / (k1_ms * 1e-3) / 1e12},
            "k2_cached_step": {"avg_launch_ms": k2_ms, "algorithmic_bytes": k2_bytes,
                               "achieved_gbs": k2_bytes / (k2_ms * 1e-3) / 1e9},
            "schedule_sweep": sweep,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_fb * args.steps,
            "clocks": clocks,
        }
        return line
    return None


def run_e2e(args, eng, kc, vc, dev, sched, world):
    """Same metric through the public engine API (eager launches, no graph):
    every diffusion step copies its Q / K_in / V_in for all layers from pinned
    host memory and copies the step's attention outputs (all layers, bf16)
    back to pinned host memory.  H2D copies run on one copy stream, D2H on
    another (PCIe is full duplex), into / out of double-buffered device slots,
    so step s+1's inputs and step s-1's outputs move while step s computes.
    Timed on the host wall clock around whole blocks, after a synchronize on
    both sides."""
    import torch

    from paper_2602_05305_b200.policy import Decision

    b = args.batch
    hq_shape, kv_shape = (b, HQ, BLK, D), (b, HKV, BLK, D)
    host_q = torch.randn((LAYERS,) + hq_shape, dtype=torch.float32).to(torch.bfloat16).pin_memory()
    host_k = torch.randn((LAYERS,) + kv_shape, dtype=torch.float32).to(torch.bfloat16).pin_memory()
    host_v = torch.randn((LAYERS,) + kv_shape, dtype=torch.float32).to(torch.bfloat16).pin_memory()
    host_o = [torch.empty((LAYERS,) + hq_shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    dq = [torch.empty_like(host_q, device=dev) for _ in range(2)]
    dk = [torch.empty_like(host_k, device=dev) for _ in range(2)]
    dv = [torch.empty_like(host_v, device=dev) for _ in range(2)]
    outs = [torch.empty((LAYERS,) + hq_shape, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    comp = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]     # inputs of slot landed
    consumed = [torch.cuda.Event() for _ in range(2)]  # attention done with slot inputs / outputs written
    drained = [torch.cuda.Event() for _ in range(2)]   # outputs of slot copied to the host
    for sl in range(2):
        consumed[sl].record(comp)
        drained[sl].record(comp)

    def block():
        eng.begin_block(0)
        for s, dec in enumerate(sched):
            sl = s & 1
            with torch.cuda.stream(h2d):
                h2d.wait_event(consumed[sl])  # slot free: step s-2 has consumed it
                dq[sl].copy_(host_q, non_blocking=True)
                dk[sl].copy_(host_k, non_blocking=True)
                dv[sl].copy_(host_v, non_blocking=True)
                ready[sl].record(h2d)
            comp.wait_event(ready[sl])
            comp.wait_event(drained[sl])  # step s-2's outputs have left this slot
            for l in range(LAYERS):
                if dec is Decision.RECOMPUTE:
                    eng.refresh(l, dq[sl][l], kc[l], vc[l], CTX, dk[sl][l], dv[sl][l], out=outs[sl][l])
                else:
                    eng.cached(l, dq[sl][l], dk[sl][l], dv[sl][l], out=outs[sl][l])
            consumed[sl].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(consumed[sl])
                host_o[sl].copy_(outs[sl], non_blocking=True)
                drained[sl].record(d2h)

    steps = max(1, args.steps // 2)
    block()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        block()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h2d_b = STEPS_PER_BLOCK * (host_q.numel() + host_k.numel() + host_v.numel()) * 2
    d2h_b = STEPS_PER_BLOCK * host_o[0].numel() * 2
    return {"value": world * b * BLK * steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b,
            "h2d_gbs": h2d_b * steps / dt / 1e9, "d2h_gbs": d2h_b * steps / dt / 1e9,
            "note": "public engine API, eager launches; every diffusion step: H2D of Q/K_in/V_in (all "
                    "layers) and D2H of the attention outputs (all layers, bf16) from/to pinned host "
                    "memory on two copy streams overlapping the attention; the *_bytes_per_step count "
                    "one bench step = one 32-step block; host wall clock; PCIe-bound"}


C3_CTX = 131072


def run_splitkv(args, rank: int, world: int, local_rank: int):
    """C3 (BASELINE.json configs[2]): 128K context whose committed KV is split
    along the sequence over the `world` ranks (strong scaling: the same b
    sequences whatever the rank count).  Per layer and block:
      refresh step = K1 on the local shard -> ONE packed exchange of the fp32
                     (O, LSE) partials (grouped NCCL send/recv by kv-group
                     chunk; splitkv.py) -> K3 merge for this rank's kv-head
                     shard -> K2 on the shard;
      31 cached steps = K2 on the head shard only (no KV, no exchange).
    The refresh step runs eagerly (the exchange stays outside CUDA graphs);
    the cached steps of a block replay as one CUDA graph.  All 36 layers have
    their own KV shard (b=4: 77 GB at N=1, 9.7 GB per rank at N=8)."""
    import torch
    import torch.distributed as dist

    from paper_2602_05305_b200 import _lib
    from paper_2602_05305_b200 import kernels as K
    from paper_2602_05305_b200.splitkv import SplitKVRefresh, group_chunks, shard_bounds

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    b, N, L = args.c3_batch, args.ctx, args.layers
    groups, rows = b * HKV, (HQ // HKV) * BLK
    lo, hi = shard_bounds(N, world, rank)
    n_loc = hi - lo
    g0, g1 = group_chunks(groups, world)[rank]
    per = g1 - g0
    gen = torch.Generator(device=dev).manual_seed(99 + rank)

    def rnd(*sh):
        return torch.randn(sh, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)

    kc = [rnd(groups, max(n_loc, 1), D) for _ in range(L)]
    vc = [rnd(groups, max(n_loc, 1), D) for _ in range(L)]
    # queries and the current block are the same on every rank (seeded alike)
    gq = torch.Generator(device=dev).manual_seed(7)
    q = [torch.randn((groups, rows, D), device=dev, generator=gq).to(torch.bfloat16) for _ in range(L)]
    ki = [torch.randn((groups, BLK, D), device=dev, generator=gq).to(torch.bfloat16) for _ in range(L)]
    vi = [torch.randn((groups, BLK, D), device=dev, generator=gq).to(torch.bfloat16) for _ in range(L)]
    # cached external partial: bf16 O (the engine's layout), fp32 LSE; the
    # exchanged shard partials stay fp32 (splitkv.PackedPartial)
    o_ext = [torch.empty((per, rows, D), device=dev, dtype=torch.bfloat16) for _ in range(L)]
    l_ext = [torch.empty((per, rows), device=dev, dtype=torch.float32) for _ in range(L)]
    out = [torch.empty((per, rows, D), device=dev, dtype=torch.bfloat16) for _ in range(L)]
    layouts = {"nccl": "all_to_all", "p2p": "p2p"}
    refresh = SplitKVRefresh(layout=layouts[args.exchange] if world > 1 else "all_to_all")

    def refresh_step(rf=None):
        rf = rf or refresh
        for l in range(L):
            rf(q[l], kc[l], vc[l], n_loc, None, out=o_ext[l], lse=l_ext[l])
            K.internal_merge(q[l][g0:g1], ki[l][g0:g1], vi[l][g0:g1], o_ext[l], l_ext[l],
                             out_dtype=torch.bfloat16, out=out[l])

    def cached_steps():
        for _ in range(STEPS_PER_BLOCK - 1):
            for l in range(L):
                K.internal_merge(q[l][g0:g1], ki[l][g0:g1], vi[l][g0:g1], o_ext[l], l_ext[l],
                                 out_dtype=torch.bfloat16, out=out[l], ext_stable=True)

    stream = torch.cuda.current_stream(dev)
    refresh_step()
    cached_steps()
    torch.cuda.synchronize()
    g_cached = torch.cuda.CUDAGraph()
    c0 = lib.fb_launch_count()
    with torch.cuda.graph(g_cached):
        cached_steps()
    cached_launches = lib.fb_launch_count() - c0
    torch.cuda.synchronize()

    def block():
        refresh_step()
        g_cached.replay()

    def max_over_ranks(ms: float) -> float:
        if world == 1:
            return ms
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1))
        if world > 1:
            dist.barrier()
        return ms

    sampler = ClockSampler(gpu_smi_id(dev))
    sampler.start()
    l0 = lib.fb_launch_count()
    ms = timed(block, args.steps, args.warmup)
    eager_launches = lib.fb_launch_count() - l0  # the graph replays are not counted by the host
    clocks = sampler.stop()
    # the two parts of the block alone: T_refresh(P) (K1 + exchange + K3 + K2 over 36
    # layers) and the cached steps
    ms_ref = timed(refresh_step, max(2, args.steps // 2), 2) / max(2, args.steps // 2)
    ms_cached = timed(g_cached.replay, max(2, args.steps // 2), 2) / max(2, args.steps // 2)
    # K1 on the local shard alone (roofline of the dominant kernel at this P)
    o_dt = torch.bfloat16 if world == 1 else torch.float32  # N=1 writes the cached partial directly
    o_s = torch.empty((groups, rows, D), device=dev, dtype=o_dt)
    l_s = torch.empty((groups, rows), device=dev, dtype=torch.float32)

    def k1_only():
        for l in range(L):
            K.attention_partial(q[l], kc[l], vc[l], 0, n_loc, None, out=o_s, lse=l_s)

    ms_k1 = timed(k1_only, 2, 1) / 2 / L

    # the other exchange for comparison (last: a peer-memory set-up that fails
    # leaves every number above already measured): peer-memory (CUDA IPC mapped partials,
    # device flags, K3 reading in place) vs the NCCL grouped send / recv
    other = {"nccl": "p2p", "p2p": "nccl"}[args.exchange]
    ms_ref_other = None
    if world > 1:
        try:  # a set-up failure of the comparison (e.g. no CUDA IPC) must not cost the line
            alt = SplitKVRefresh(layout=layouts[other])
            ms_ref_other = timed(lambda: refresh_step(alt), max(2, args.steps // 2), 2) / max(2, args.steps // 2)
            alt.close()
        except Exception as e:  # noqa: BLE001
            ms_ref_other = f"unavailable: {type(e).__name__}: {e}"[:200]
    k1_bytes = 2 * groups * n_loc * D * 2 + groups * rows * D * 2 + groups * rows * (D * o_s.element_size() + 4)
    peak, peak_kind = _peaks()
    if rank == 0:
        value = b * BLK * args.steps / (ms / 1000.0)
        exch = groups * rows * (D + 1) * 4 * (world - 1) // world if world > 1 else 0
        return {
            "metric": "block-diffusion tokens/s (FlashBlock attention, C3: 128K ctx split-KV)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) bf16, seeded; distinct KV shard per layer",
            "config": {"workload": "C3: 8B-class GQA, 128K ctx, KV split along the sequence over "
                                   f"{world} GPU(s), FlashBlock tau=2 (1 refresh / 32 steps)",
                       "layers": L, "batch": b, "ctx": N, "shard_rows": n_loc, "q_heads": HQ,
                       "kv_heads": HKV, "head_dim": D, "block": BLK, "steps_per_block": STEPS_PER_BLOCK,
                       "kv_groups_per_rank": per,
                       "exchange": ("packed fp32 (O, LSE) partials, one grouped send/recv per layer "
                                    "per block (all_to_all by kv-group chunk); cached steps exchange nothing"
                                    if args.exchange == "nccl" or world == 1 else
                                    "peer memory: CUDA-IPC-mapped packed fp32 (O, LSE) partials, device "
                                    "flag handshake, K3 merging the rank's kv-group chunk in place; no "
                                    "collective; cached steps exchange nothing"),
                       "parallelism": f"split-KV x{world} (refresh) + kv-head shards (cached steps)",
                       "l2": "inputs larger than L2 (distinct KV shard per layer)"},
            "refresh_step_ms": ms_ref, "refresh_ms_per_layer": ms_ref / L,
            "refresh_step_ms_other_exchange": ({other: ms_ref_other} if ms_ref_other is not None else None),
            "exchange_used": args.exchange if world > 1 else None,
            "cached_steps_ms": ms_cached,
            "exchange_bytes_sent_per_layer_per_rank": exch,
            "roofline": {"bound": "hbm", "kernel": "K1 on the local KV shard",
                         "achieved": k1_bytes / (ms_k1 * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": k1_bytes / (ms_k1 * 1e-3) / 1e9 / peak, "traffic": None,
                         "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": ms_k1,
                         "peak_kind": peak_kind},
            "e2e": None,
            "gpu_launches": eager_launches + cached_launches * args.steps,
            "clocks": clocks,
            "nccl_debug": os.environ.get("NCCL_DEBUG"),
        }
    return None


def _relaunch(args) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run
    with N local ranks and a 127.0.0.1 rendezvous; returns its exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=32, help="C2 sequences per GPU (b=32: 155 GB of KV cache over 36 layers)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-sweep", action="store_true", help="skip the schedule sweep")
    ap.add_argument("--workload", default=None, choices=["c2", "c3"],
                    help="c2: 32K headline (default; at N > 1 also measures C3 into c3_split_kv); "
                         "c3: the 128K split-KV line as the main line")
    ap.add_argument("--ctx", type=int, default=C3_CTX, help="context for C3")
    ap.add_argument("--layers", type=int, default=LAYERS, help="layers for C3")
    ap.add_argument("--c3-batch", type=int, default=4, help="sequences for C3 (whole job)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="C3 split-KV exchange at N > 1: NCCL grouped send/recv (default) or peer memory "
                         "(CUDA IPC, device flags, K3 in place); the other one is timed alongside")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(_relaunch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("FB_BENCH_BACKEND", "nccl") != "nccl":  # diagnostics: ranks may share GPUs
        import torch

        local_rank %= max(1, torch.cuda.device_count())
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    # C2 (the headline, configs[1]) at every N: sequences are independent, so
    # N ranks run N x the batch with no data-path collective (weak scaling) and
    # the curve over N stays one workload.  At N > 1 the same run then measures
    # C3 (configs[2]: 128K context split along the sequence over the N GPUs,
    # one packed NCCL exchange per refresh) and attaches it as "c3_split_kv".
    # --workload c3 makes C3 the main line.
    workload = args.workload or "c2"
    if world > 1:
        import torch
        import torch.distributed as dist

        # communicator ranks / NVLS visible in the log
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("FB_BENCH_BACKEND", "nccl")  # gloo: diagnostics (ranks sharing one GPU)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        if workload == "c3":
            line = run_splitkv(args, rank, world, local_rank)
        else:
            line = run_ours(args, rank, world, local_rank)
            if world > 1 and args.workload is None:
                import gc

                import torch

                gc.collect()
                torch.cuda.empty_cache()  # the C2 caches (155 GB at b=32) go before C3's shards
                c3 = run_splitkv(args, rank, world, local_rank)
                if line is not None and c3 is not None:
                    line["c3_split_kv"] = {k: c3[k] for k in (
                        "metric", "value", "unit", "ms_per_step", "scaling", "config", "refresh_step_ms",
                        "refresh_ms_per_layer", "refresh_step_ms_other_exchange", "exchange_used", "cached_steps_ms",
                        "exchange_bytes_sent_per_layer_per_rank",
                        "roofline", "gpu_launches")}
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
