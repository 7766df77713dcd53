"""Secondary benchmark lines for BASELINE.json configs C1, C3, C4, C5 and the
prefill path (F4) and the head-gated refresh (F3), SURVEY 8f.

    python scripts/bench_configs.py [--only c3,c4,c5,f4,f3,c1,cpu] [--out profiles/rXX_configs.jsonl]

One JSON line per measurement.  All device timings are CUDA events around
CUDA-graph replays of the measured launches (no host gaps), after warm-up,
on distinct per-layer buffers where the working set would otherwise sit in
L2.  Peaks from MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_05305_b200 import kernels as K  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
HBM, TENSOR = float(PEAKS["hbm_gbs"]), float(PEAKS["bf16_tflops"])
DEV = torch.device("cuda")


def rnd(g, *shape):
    return torch.randn(shape, device=DEV, generator=g).to(torch.bfloat16)


def graph_ms(fn, reps=5):
    """Average ms of fn() replayed as a CUDA graph."""
    s = torch.cuda.Stream()
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def emit(out, rec):
    line = json.dumps(rec)
    print(line, flush=True)
    out.write(line + "\n")


# ---------------------------------------------------------------- C2 layer


def c2layer(out):
    """the C2 attention LAYER -- QKV projection (4096 -> 6144),
    FlashBlock attention, O projection (4096 -> 4096) -- with random-init bf16
    weights, b=16, 32K context, tau=2 schedule (1 refresh + 31 cached steps per
    32-step block) vs full recompute every step.  Projections are plain cuBLAS
    GEMMs (torch.matmul), head-major outputs straight from a batched GEMM; no
    RoPE / norms (not part of the reference's attention path).  L distinct
    layers (weights + KV) per graph so nothing stays in L2; per-layer times."""
    from paper_2602_05305_b200 import FlashBlockAttention
    HQ, HKV, D, B, N, DM, b, L = 32, 8, 128, 32, 32768, 4096, 16, 6
    g = torch.Generator(device=DEV).manual_seed(2)
    NQKV = (HQ + 2 * HKV) * D  # 6144
    x = [rnd(g, b * B, DM) for _ in range(L)]
    wqkv = [(rnd(g, DM, NQKV).float() * DM ** -0.5).to(torch.bfloat16) for _ in range(L)]
    wo = [(rnd(g, DM, DM).float() * DM ** -0.5).to(torch.bfloat16) for _ in range(L)]
    qkv = [torch.empty(b * B, NQKV, device=DEV, dtype=torch.bfloat16) for _ in range(L)]
    kc = [rnd(g, b, HKV, N, D) for _ in range(L)]
    vc = [rnd(g, b, HKV, N, D) for _ in range(L)]
    att = [torch.empty(b, HQ, B, D, device=DEV, dtype=torch.bfloat16) for _ in range(L)]
    y = [torch.empty(b * B, DM, device=DEV, dtype=torch.bfloat16) for _ in range(L)]
    eng = FlashBlockAttention(L, b, HQ, HKV, B, D, device=DEV)
    groups, rows = b * HKV, (HQ // HKV) * B
    o_scr = torch.empty(groups, rows, D, device=DEV, dtype=torch.float32)
    l_scr = torch.empty(groups, rows, device=DEV, dtype=torch.float32)

    def proj_in(l):
        torch.matmul(x[l], wqkv[l], out=qkv[l])            # one fused QKV GEMM
        t = qkv[l].view(b, B, HQ + 2 * HKV, D).permute(0, 2, 1, 3)  # head-major views
        return (t[:, :HQ].contiguous(), t[:, HQ:HQ + HKV].contiguous(), t[:, HQ + HKV:].contiguous())

    def layer(l, mode):
        q, ki, vi = proj_in(l)
        if mode == "refresh":
            eng.refresh(l, q, kc[l], vc[l], N, ki, vi, out=att[l])
        elif mode == "cached":
            eng.cached(l, q, ki, vi, out=att[l])
        else:
            eng.full_recompute(q, kc[l], vc[l], N, ki, vi, out=att[l], o_scratch=o_scr, lse_scratch=l_scr)
        torch.matmul(att[l].permute(0, 2, 1, 3).reshape(b * B, DM), wo[l].t(), out=y[l])

    att_tok = [torch.empty(b * B, DM, device=DEV, dtype=torch.bfloat16) for _ in range(L)]

    def layer_tok(l, mode):
        # token-major: attention reads q / k / v straight out of the QKV GEMM's
        # output and writes the O GEMM's input; no head-major copies
        torch.matmul(x[l], wqkv[l], out=qkv[l])
        t = qkv[l].view(b, B, HQ + 2 * HKV, D)
        q, ki, vi, o = t[:, :, :HQ], t[:, :, HQ:HQ + HKV], t[:, :, HQ + HKV:], att_tok[l].view(b, B, HQ, D)
        if mode == "refresh":
            eng.refresh_tokmajor(l, q, kc[l], vc[l], N, ki, vi, o)
        else:
            eng.cached_tokmajor(l, q, ki, vi, o)
        torch.matmul(att_tok[l], wo[l].t(), out=y[l])

    eng.begin_block(0)
    for l in range(L):
        layer(l, "refresh")
    t_ref = graph_ms(lambda: [layer(l, "refresh") for l in range(L)], reps=3) / L
    t_cac = graph_ms(lambda: [layer(l, "cached") for l in range(L)], reps=3) / L
    t_full = graph_ms(lambda: [layer(l, "full") for l in range(L)], reps=3) / L
    t_gemm = graph_ms(lambda: [(proj_in(l), torch.matmul(att[l].permute(0, 2, 1, 3).reshape(b * B, DM),
                                                         wo[l].t(), out=y[l])) for l in range(L)], reps=3) / L
    t_ref_tok = graph_ms(lambda: [layer_tok(l, "refresh") for l in range(L)], reps=3) / L
    t_cac_tok = graph_ms(lambda: [layer_tok(l, "cached") for l in range(L)], reps=3) / L
    fb_block = t_ref + 31 * t_cac
    tok_block = t_ref_tok + 31 * t_cac_tok
    full_block = 32 * t_full
    emit(out, {"config": "C2-layer", "batch": b, "ctx": N, "d_model": DM, "q_heads": HQ, "kv_heads": HKV,
               "layer_refresh_ms": t_ref, "layer_cached_ms": t_cac, "layer_full_recompute_ms": t_full,
               "projections_only_ms": t_gemm,
               "tokens_per_s_36_layers": b * B / (36 * fb_block * 1e-3),
               "full_recompute_tokens_per_s_36_layers": b * B / (36 * full_block * 1e-3),
               "speedup_vs_full_recompute": full_block / fb_block,
               "token_major": {"layer_refresh_ms": t_ref_tok, "layer_cached_ms": t_cac_tok,
                               "tokens_per_s_36_layers": b * B / (36 * tok_block * 1e-3),
                               "speedup_vs_full_recompute": full_block / tok_block},
               "note": "per layer: QKV GEMM + attention + O GEMM (cuBLAS projections, random-init "
                       "weights); block = 1 refresh + 31 cached steps (tau=2 schedule)"})
    del kc, vc
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- C3


def c3(out):
    """128K context, KV split over P shards.  Single-GPU emulation: each shard's
    K1 runs alone on the full GPU (what each of P GPUs does), then the K3 merge
    of the P fp32 partials.  The NCCL exchange is not measured on one GPU; its
    payload is reported."""
    HQ, HKV, D, B, N, L = 32, 8, 128, 32, 131072, 4
    for b in (1, 8):
        g = torch.Generator(device=DEV).manual_seed(3)
        groups, rows = b * HKV, (HQ // HKV) * B
        q = [rnd(g, groups, rows, D) for _ in range(L)]
        k = [rnd(g, groups, N, D) for _ in range(L)]
        v = [rnd(g, groups, N, D) for _ in range(L)]
        res = {}
        for P in (1, 2, 4, 8):
            n = N // P
            parts = [K.attention_partial(q[0], k[0], v[0], 0, n) for _ in range(P)]
            t_k1 = graph_ms(lambda: [K.attention_partial(q[l], k[l], v[l], 0, n) for l in range(L)]) / L
            # after the all_to_all each rank merges the P partials of its own
            # kv-head shard only (splitkv.py): 1/P of the rows.  8 merges per
            # graph: a one-node graph would time the graph launch
            gs = max(1, groups // P)
            mine = [(o[:gs], l_[:gs]) for o, l_ in parts]
            t_m = graph_ms(lambda: [K.combine(mine) for _ in range(8)]) / 8 if P > 1 else 0.0
            res[P] = t_k1 + t_m
            kv_bytes = 2 * groups * n * D * 2
            payload = groups * rows * (D + 1) * 4
            emit(out, {"config": "C3", "batch": b, "ctx": N, "shards": P,
                       "k1_shard_ms": t_k1, "merge_ms": t_m, "t_refresh_ms": t_k1 + t_m,
                       "k1_gbs": kv_bytes / (t_k1 * 1e-3) / 1e9, "k1_frac_hbm": kv_bytes / (t_k1 * 1e-3) / 1e9 / HBM,
                       "exchange_bytes_per_gpu": payload * (P - 1) // max(P, 1),
                       "efficiency_T1_over_P_TP": res[1] / (P * res[P]),
                       "note": "single-GPU emulation: shard K1 on the whole GPU + K3 merge of this "
                               "rank's 1/P kv-head shard; NCCL exchange not measured"})
        del q, k, v
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- C4


def c4(out):
    """64K sparse with residual reuse, densities sweep; per layer at b=4."""
    HQ, HKV, D, B, N, L = 32, 8, 128, 32, 65536, 4
    b = 4
    g = torch.Generator(device=DEV).manual_seed(4)
    groups, rows = b * HKV, (HQ // HKV) * B
    q = [rnd(g, groups, rows, D) for _ in range(L)]
    k = [rnd(g, groups, N, D) for _ in range(L)]
    v = [rnd(g, groups, N, D) for _ in range(L)]
    ki = [rnd(g, groups, B, D) for _ in range(L)]
    vi = [rnd(g, groups, B, D) for _ in range(L)]
    nb = N // 16
    t_dense = graph_ms(lambda: [K.full_attention(q[l], k[l], v[l], N, ki[l], vi[l]) for l in range(L)]) / L
    for dens in (0.1, 0.2, 0.3, 0.4, 0.5, 1.0):
        budget = K.mask_budget(N, dens, 16)
        sel = [K.topk_blocks(K.block_mass(q[l], k[l], ki[l], N, 16), budget) for l in range(L)]
        res = [K.sparse_partitioned(q[l], k[l], v[l], ki[l], vi[l], N, sel[l])[2] for l in range(L)]
        t_mask = graph_ms(lambda: [K.topk_blocks(K.block_mass(q[l], k[l], ki[l], N, 16), budget)
                                   for l in range(L)]) / L
        t_k7 = graph_ms(lambda: [K.sparse_partitioned(q[l], k[l], v[l], ki[l], vi[l], N, sel[l])
                                 for l in range(L)]) / L
        t_k8 = graph_ms(lambda: [K.sparse_attend_merge(q[l], k[l], v[l], ki[l], vi[l], N, sel[l], res[l])
                                 for l in range(L)]) / L
        # accuracy (sparse.py:303-325 measure_sparse_gap): a later step's drifted
        # queries against the dense result; residual cached at the first step
        q2 = (q[0].float() + 0.3 * torch.randn(q[0].shape, device=DEV, generator=g)).to(torch.bfloat16)
        dense = K.full_attention(q2, k[0], v[0], N, ki[0], vi[0])[0].float()
        so = K.sparse_attend_merge(q2, k[0], v[0], ki[0], vi[0], N, sel[0], None).float()
        wr = K.sparse_attend_merge(q2, k[0], v[0], ki[0], vi[0], N, sel[0], res[0]).float()
        l1_so = float((so - dense).abs().mean())
        l1_wr = float((wr - dense).abs().mean())
        sel_keys = budget * 16
        k8_bytes = 2 * groups * sel_keys * D * 2 + groups * rows * (D + 1) * 4 * 2
        k7_bytes = 2 * groups * N * D * 2
        # fused K5: K read once (the per-row block sums and maxima it writes and the
        # reduce kernel reads back are overhead, not algorithmic bytes)
        k5_bytes = groups * N * D * 2
        t_k5 = graph_ms(lambda: [K.block_mass(q[l], k[l], ki[l], N, 16) for l in range(L)]) / L
        step_block = t_mask + t_k7 + 31 * t_k8
        emit(out, {"config": "C4", "batch": b, "ctx": N, "density": dens, "budget_blocks": budget,
                   "mask_ms": t_mask, "k5_ms": t_k5, "k5_gbs": k5_bytes / (t_k5 * 1e-3) / 1e9,
                   "k5_frac_hbm": k5_bytes / (t_k5 * 1e-3) / 1e9 / HBM,
                   "k5_note": "block_mass (fused score pass + mass reduce) over K once; mask_ms adds K6",
                   "k7_first_step_ms": t_k7, "k7_gbs": k7_bytes / (t_k7 * 1e-3) / 1e9,
                   "k8_cached_step_ms": t_k8, "k8_gbs": k8_bytes / (t_k8 * 1e-3) / 1e9,
                   "k8_frac_hbm": k8_bytes / (t_k8 * 1e-3) / 1e9 / HBM,
                   "block_ms_per_layer_32_steps": step_block,
                   "dense_full_recompute_block_ms_per_layer": 32 * t_dense,
                   "speedup_vs_dense_recompute": 32 * t_dense / step_block,
                   "l1_sparse_only": l1_so, "l1_with_residual": l1_wr,
                   "l1_note": "mean |out - dense| on a drifted query (q + 0.3 N(0,1)), random N(0,1) K/V"})
    del q, k, v
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- C5


def c5(out):
    """Video block diffusion (Wan-1.3B-like): 12 heads x 128, chunk B = 4680
    tokens, external context up to 56,160; compute-bound."""
    H, D, B = 12, 128, 4680
    for n_ext in (18720, 56160):
        g = torch.Generator(device=DEV).manual_seed(5)
        q = rnd(g, H, B, D)
        k = rnd(g, H, n_ext, D)
        v = rnd(g, H, n_ext, D)
        ki, vi = rnd(g, H, B, D), rnd(g, H, B, D)
        o_ext, l_ext = K.attention_partial(q, k, v, 0, n_ext)
        t_k1 = graph_ms(lambda: K.attention_partial(q, k, v, 0, n_ext, None, o_ext, l_ext), reps=3)
        t_k2 = graph_ms(lambda: K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.bfloat16), reps=3)
        f1 = 4.0 * H * B * n_ext * D
        f2 = 4.0 * H * B * B * D
        emit(out, {"config": "C5", "heads": H, "block": B, "n_ext": n_ext,
                   "k1_refresh_ms": t_k1, "k1_tflops": f1 / (t_k1 * 1e-3) / 1e12,
                   "k1_frac_tensor": f1 / (t_k1 * 1e-3) / 1e12 / TENSOR,
                   "k2_cached_ms": t_k2, "k2_tflops": f2 / (t_k2 * 1e-3) / 1e12,
                   "k2_frac_tensor": f2 / (t_k2 * 1e-3) / 1e12 / TENSOR,
                   "speedup_cached_vs_refresh_step": (t_k1 + t_k2) / t_k2})
        del q, k, v
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- F4 prefill


def f4(out):
    """Prefill / commit attention at the C2 attention shapes:
    a whole prompt's block-causal attention in one launch (the reference
    commits it block by block, simulator.py:343-354).  Compute-bound."""
    HQ, HKV, D, B = 32, 8, 128, 32
    G = HQ // HKV
    for b, n_q in ((1, 8192), (1, 32768)):
        g = torch.Generator(device=DEV).manual_seed(9)
        groups = b * HKV
        q = rnd(g, groups, G * n_q, D)
        k = rnd(g, groups, n_q, D)
        v = rnd(g, groups, n_q, D)
        o, l = K.block_causal_attention(q, k, v, n_q, 0, B)
        t = graph_ms(lambda: K.block_causal_attention(q, k, v, n_q, 0, B, None, o, l), reps=3)
        lim = sum(min(n_q, (p // B + 1) * B) for p in range(0, n_q, B)) * B  # sum over positions
        flops = 4.0 * groups * G * lim * D
        emit(out, {"config": "F4-prefill", "batch": b, "prompt": n_q, "q_heads": HQ, "kv_heads": HKV,
                   "block": B, "ms": t, "tflops": flops / (t * 1e-3) / 1e12,
                   "frac_tensor": flops / (t * 1e-3) / 1e12 / TENSOR,
                   "tokens_per_s": b * n_q / (t * 1e-3)})
        del q, k, v
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- F3 head-gated refresh


def f3(out):
    """Head-gated refresh at the C5 video shapes (12 heads,
    1:1, chunk 4680, 18,720 external keys): K1 over the heads whose gate is
    off + K2 for all, vs the full refresh; and the calibrator's per-step
    cost (row cosine of the external partials)."""
    from paper_2602_05305_b200.analysis import HeadGateCalibrator

    H, D, B, n_ext = 12, 128, 4680, 18720
    g = torch.Generator(device=DEV).manual_seed(6)
    q, k, v = rnd(g, H, B, D), rnd(g, H, n_ext, D), rnd(g, H, n_ext, D)
    ki, vi = rnd(g, H, B, D), rnd(g, H, B, D)
    o_ext, l_ext = K.attention_partial(q, k, v, 0, n_ext)
    t_full = graph_ms(lambda: (K.attention_partial(q, k, v, 0, n_ext, None, o_ext, l_ext),
                               K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.bfloat16)), reps=3)
    for n_on in (3, 6, 9):
        gl = torch.arange(n_on, dtype=torch.int32, device=DEV)
        t = graph_ms(lambda: (K.attention_partial_groups(q, k, v, gl, 0, n_ext, None, o_ext, l_ext),
                              K.internal_merge(q, ki, vi, o_ext, l_ext, out_dtype=torch.bfloat16)), reps=3)
        emit(out, {"config": "F3-head-gated", "heads": H, "block": B, "n_ext": n_ext,
                   "heads_refreshed": n_on, "step_ms": t, "full_refresh_step_ms": t_full,
                   "speedup_vs_full_refresh": t_full / t})
    cal = HeadGateCalibrator(1, H)
    cal.observe(0, o_ext, B)
    t_cal = graph_ms(lambda: cal.observe(0, o_ext, B), reps=5)
    emit(out, {"config": "F3-calibrator", "heads": H, "rows": B, "observe_ms": t_cal,
               "bytes": 3 * H * B * D * 4, "gbs": 3 * H * B * D * 4 / (t_cal * 1e-3) / 1e9,
               "note": "fb_row_cosine_update: reads this and the previous step's partial, writes the copy; "
                       "+ per-head means and the [b, Hq] sum / min"})


# ---------------------------------------------------------------- C1


def c1(out):
    """Tiny CPU-runnable LM (2 layers, d=256, 4 heads, block 32, 4K context):
    the reference's own run_sequence, CPU vs its attention routed through
    libfb200.so (drop-in replay), FlashBlock tau=2 vs always-recompute."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "flashblock")):
        emit(out, {"config": "C1", "unavailable": "reference not installed at baseline/_ref"})
        return
    sys.path.insert(0, ref_dir)
    import flashblock as fbref

    from paper_2602_05305_b200.replay import patch_reference_simulator

    model = fbref.SyntheticModel(fbref.ModelConfig(num_layers=2, num_heads=4, head_dim=64, seed=0,
                                                   dtype=__import__("numpy").float32))
    for pol in ("token-threshold", "always-recompute"):
        args = dict(prompt_len=4096, num_blocks=1, block_size=32, steps_per_block=32,
                    policy=fbref.ReuseConfig(tau=2, mode=pol), seed=0, unmask_per_step=1)
        t0 = time.perf_counter()
        base = fbref.run_sequence(model, **args)
        t_cpu = sum(t.wall_ns for t in base.traces) / 1e9
        with patch_reference_simulator(fbref.simulator):
            fbref.run_sequence(model, **args)  # warm
            gpu = fbref.run_sequence(model, **args)
        t_gpu = sum(t.wall_ns for t in gpu.traces) / 1e9
        same = [a.decision for a in gpu.traces] == [a.decision for a in base.traces]
        emit(out, {"config": "C1", "policy": pol, "cpu_tokens_per_s": 32 / t_cpu,
                   "gpu_replay_tokens_per_s": 32 / t_gpu, "decisions_equal": same,
                   "final_ids_equal": bool((gpu.final_ids == base.final_ids).all()),
                   "max_checksum_rel_diff": max(abs(a.checksum - b.checksum) / max(1.0, abs(b.checksum))
                                                for a, b in zip(gpu.traces, base.traces)),
                   "note": "steps only (wall_ns of denoise_step); the reference API is synchronous "
                           "numpy, so every (layer, head) call is one host<->device round trip: cached "
                           "steps go through fb_internal_merge_host (pinned staging, one upload, one "
                           "read-back) against the device-resident cached partial"})


# ---------------------------------------------------------------- CPU reference at C3 / C4


def cpu(out):
    """The reference CPU path at the C3 (128K) and C4 (64K sparse, 10 / 50 %)
    shapes: one layer x 8 kv-heads x one 32-step block at b=1
    (G = 4 query heads stacked per kv head), on all host cores, with the GPU
    time of the same layer-block for the ratio."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import bench as BN

    threads = str(os.cpu_count())
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, threads)
    sched = BN._sched_names()
    # C3: dense FlashBlock layer-block over 131,072 committed keys
    kind, t = BN.cpu_layer_block(131072, sched, reps=1)
    emit(out, {"config": "C3-cpu", "ctx": 131072, "kind": kind, "cores": os.cpu_count(),
               "cpu_model": BN.cpu_model(), "layer_block_s_b1": t,
               "tokens_per_s_36_layers": BN.cpu_tokens_per_s(t),
               "sample": "1 layer x 8 kv-heads x one 32-step block (1 refresh + 31 reuse), b=1, tile 512"})
    # C4: sparse + residual reuse at 64K: build_sparse_mask + the exact first
    # step, then 31 later steps against the cached residual (sparse.py:83-183)
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "flashblock")):
        return
    sys.path.insert(0, ref_dir)
    import flashblock.sparse as S
    import flashblock.attention as A

    N, B, G, D = 65536, 32, 4, 128
    rng = np.random.Generator(np.random.Philox(77))
    heads = [tuple(rng.standard_normal(sh).astype(np.float32) for sh in ((G * B, D), (N + B, D), (N + B, D)))
             for _ in range(8)]
    for dens in (0.1, 0.5):
        t0 = time.perf_counter()
        for q, k, v in heads:
            mask = S.build_sparse_mask(q, k, N, dens, 16)
            _, resid = S.sparse_attention_with_residual(q, mask, k, v, None, tile_size=512)
            entry = A.CacheEntry(resid, 0, 0)
            for _ in range(31):
                S.sparse_attention_with_residual(q, mask, k, v, entry, tile_size=512)
        t = time.perf_counter() - t0
        emit(out, {"config": "C4-cpu", "ctx": N, "density": dens, "kind": "reference", "cores": os.cpu_count(),
                   "cpu_model": BN.cpu_model(), "layer_block_s_b1": t,
                   "tokens_per_s_36_layers": B / (36 * t),
                   "sample": "1 layer x 8 kv-heads: build_sparse_mask + the exact first step + 31 cached-residual "
                             "steps, b=1, tile 512"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c2layer,c3,c4,c5,f4,f3,c1,cpu")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as out:
        for name in a.only.split(","):
            globals()[name.strip()](out)


if __name__ == "__main__":
    main()
