"""Generate golden input/output vectors by running the REAL reference package.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py            # golden.npz
    python tests/golden/make_golden.py prefill    # golden_prefill.npz
    python tests/golden/make_golden.py analysis   # golden_analysis.npz

The fixtures it writes (``tests/golden/*.npz``) are committed; the tests read
only the fixtures.  Inputs are seeded (Philox) and, for the cases the bf16
GPU path consumes, rounded to bf16-representable float32 values so the same
numbers can be fed to the device exactly.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)) << np.uint32(16)
    return r.view(np.float32)


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import flashblock as fb  # the real reference
    from flashblock.attention import CacheEntry

    rng = np.random.Generator(np.random.Philox(20261017))
    out: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}

    # -- attention_partial / streamed / merge, fp64 and fp32, ragged sizes --
    cases = [
        ("p0", 4, 20, 8, np.float64, 64),
        ("p1", 3, 50, 8, np.float64, 17),
        ("p2", 5, 0, 8, np.float64, 64),      # empty sentinel
        ("p3", 7, 1, 16, np.float32, 64),     # single key
        ("p4", 33, 257, 64, np.float32, 512),
        ("p5", 128, 384, 128, np.float32, 512),
        ("p6", 16, 129, 128, np.float64, 64),
    ]
    for name, nq, n, d, dt, tile in cases:
        q = rng.standard_normal((nq, d)).astype(dt)
        k = rng.standard_normal((n, d)).astype(dt)
        v = rng.standard_normal((n, d)).astype(dt)
        if dt == np.float32:
            q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
        p = fb.attention_partial(q, k, v, tile_size=tile)
        out.update({f"{name}_q": q, f"{name}_k": k, f"{name}_v": v,
                    f"{name}_out": p.out, f"{name}_lse": p.lognorm})
        meta[name] = {"nq": nq, "n": n, "d": d, "dtype": np.dtype(dt).name, "tile": tile}

    # streamed + merge at several boundaries (incl. 0 and n)
    q = rng.standard_normal((6, 32))
    k = rng.standard_normal((40, 32))
    v = rng.standard_normal((40, 32))
    out.update({"s_q": q, "s_k": k, "s_v": v})
    for b in (0, 1, 17, 39, 40):
        e, i = fb.attention_streamed(q, k, v, b)
        out[f"s_b{b}_ext_out"] = e.out
        out[f"s_b{b}_ext_lse"] = e.lognorm
        out[f"s_b{b}_int_out"] = i.out
        out[f"s_b{b}_int_lse"] = i.lognorm
        out[f"s_b{b}_merged"] = fb.merge_partials(e, i)

    # combine with one side empty / both sides partially empty rows
    a = fb.attention_partial(q, k[:10], v[:10])
    bpart = fb.attention_partial(q, k[10:], v[10:])
    lse_a = a.lognorm.copy()
    lse_a[[1, 4]] = -np.inf
    out_a = a.out.copy()
    out_a[[1, 4]] = 0.0
    lse_b = bpart.lognorm.copy()
    lse_b[[4, 5]] = -np.inf
    out_b = bpart.out.copy()
    out_b[[4, 5]] = 0.0
    c = fb.combine_partials(fb.AttnPartial(out_a, lse_a), fb.AttnPartial(out_b, lse_b))
    out.update({"c_a_out": out_a, "c_a_lse": lse_a, "c_b_out": out_b, "c_b_lse": lse_b,
                "c_out": c.out, "c_lse": c.lognorm})

    # reuse: cached external from q0, drifted q1
    q0 = bf16_round(rng.standard_normal((64, 64)).astype(np.float32))
    kk = bf16_round(rng.standard_normal((300, 64)).astype(np.float32))
    vv = bf16_round(rng.standard_normal((300, 64)).astype(np.float32))
    q1 = bf16_round((q0 + 0.3 * rng.standard_normal(q0.shape)).astype(np.float32))
    ext, _ = fb.attention_streamed(q0, kk, vv, 268)
    entry = CacheEntry(partial=ext, step_created=0, block_id=0)
    ro, ri = fb.attention_with_reuse(q1, entry, kk[268:], vv[268:])
    out.update({"r_q0": q0, "r_q1": q1, "r_k": kk, "r_v": vv, "r_ext_out": ext.out,
                "r_ext_lse": ext.lognorm, "r_out": ro, "r_int_out": ri.out,
                "r_int_lse": ri.lognorm})

    # -- sparse: masks over densities, planted blocks, residual outputs --
    for name, nq, n_ext, n_in, d, kbs, planted in [
        ("m0", 4, 64, 8, 8, 16, None),
        ("m1", 8, 160, 8, 16, 16, None),
        ("m2", 32, 1000, 32, 64, 16, [3, 17, 40]),
        ("m3", 128, 2048, 32, 128, 16, [5, 77, 100, 127]),
    ]:
        qq = bf16_round(rng.standard_normal((nq, d)).astype(np.float32))
        keys = bf16_round(rng.standard_normal((n_ext + n_in, d)).astype(np.float32))
        vals = bf16_round(rng.standard_normal((n_ext + n_in, d)).astype(np.float32))
        if planted:
            for blk in planted:
                keys[blk * kbs:(blk + 1) * kbs] += bf16_round(
                    (qq.mean(axis=0) * 0.6).astype(np.float32))
            keys = bf16_round(keys)
        out.update({f"{name}_q": qq, f"{name}_k": keys, f"{name}_v": vals})
        dens = [0.05, 0.1, 0.2, 0.3, 0.5, 1.0]
        for di, dn in enumerate(dens):
            mask = fb.build_sparse_mask(qq, keys, n_ext, dn, kbs, block_id=3)
            out[f"{name}_d{di}_sel"] = mask.selected
            o1, res = fb.sparse_attention_with_residual(qq, mask, keys, vals, None)
            out[f"{name}_d{di}_out1"] = o1
            out[f"{name}_d{di}_res_out"] = res.out
            out[f"{name}_d{di}_res_lse"] = res.lognorm
            q2 = bf16_round((qq + 0.05 * np.random.Generator(np.random.Philox(di)).standard_normal(qq.shape)).astype(np.float32))
            o2, _ = fb.sparse_attention_with_residual(
                q2, mask, keys, vals, CacheEntry(partial=res, step_created=0, block_id=3))
            out[f"{name}_d{di}_q2"] = q2
            out[f"{name}_d{di}_out2"] = o2
        meta[name] = {"nq": nq, "n_ext": n_ext, "n_in": n_in, "d": d, "kbs": kbs,
                      "densities": dens}

    # -- policy: decisions straight from the reference simulator --
    sched_cases = []
    for (bs, steps, per, tau) in [(32, 32, 1, 2), (32, 16, 2, 2), (8, 8, 1, 1),
                                  (8, 8, 3, 2), (32, 32, 0, 2), (16, 10, 2, 3)]:
        model = fb.SyntheticModel(fb.ModelConfig(num_layers=1, num_heads=2, head_dim=8, seed=1))
        run = fb.run_sequence(model, 16, 1, bs, steps, fb.ReuseConfig(tau=tau),
                              seed=2, unmask_per_step=per)
        sched_cases.append({
            "block_size": bs, "steps": steps, "per_step": per, "tau": tau,
            "schedule": fb.unmask_schedule(bs, steps, per),
            "decisions": [t.decision for t in run.traces],
            "updated": [t.updated_tokens for t in run.traces],
        })
    meta["schedules"] = sched_cases

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays")




def make_prefill() -> None:
    """Block-causal prefill / commit attention from the reference's own commit
    pass: record every attention_dense call that simulator.prefill and
    commit_context_block make (simulator.py:297-354), per (layer, head), and
    store the stacked queries, the final committed K/V and the outputs.
    Writes tests/golden/golden_prefill.npz."""
    sys.path.insert(0, REF_SRC)
    import flashblock.simulator as sim

    out: dict[str, np.ndarray] = {}
    for name, dtype, heads, d, prompt_len, block, extra in [
        ("pf0", np.float64, 2, 64, 100, 32, 1),   # ragged last block, then one more commit
        ("pf1", np.float32, 3, 32, 48, 16, 0),
    ]:
        cfg = sim.ModelConfig(num_layers=2, num_heads=heads, head_dim=d, seed=5, dtype=dtype)
        model = sim.SyntheticModel(cfg)
        calls = []
        orig = sim.attention_dense

        def rec(q, keys, values, scale=None, _orig=orig):
            o = _orig(q, keys, values, scale)
            calls.append((q.copy(), keys.copy(), values.copy(), o))
            return o

        sim.attention_dense = rec
        try:
            prompt = sim.prompt_ids(model, prompt_len, seed=11)
            kv = sim.prefill(model, prompt, block)
            n_prefill_calls = len(calls)
            if extra:
                ids = np.arange(1, block + 1, dtype=np.int64) % (cfg.vocab_size - 1) + 1
                sim.commit_context_block(model, kv, ids, prompt_len)
        finally:
            sim.attention_dense = orig
        # calls are ordered block-major, then layer, then head
        L, H = cfg.num_layers, cfg.num_heads
        nblk = (prompt_len + block - 1) // block
        assert n_prefill_calls == nblk * L * H
        for layer in range(L):
            for head in range(H):
                sel = [calls[(b * L + layer) * H + head] for b in range(nblk)]
                out[f"{name}_l{layer}_h{head}_q"] = np.concatenate([c[0] for c in sel])
                out[f"{name}_l{layer}_h{head}_out"] = np.concatenate([c[3] for c in sel])
                # keys of the last call = the whole prompt's committed K/V
                out[f"{name}_l{layer}_h{head}_k"] = sel[-1][1]
                out[f"{name}_l{layer}_h{head}_v"] = sel[-1][2]
                if extra:
                    c = calls[n_prefill_calls + layer * H + head]
                    out[f"{name}_x_l{layer}_h{head}_q"] = c[0]
                    out[f"{name}_x_l{layer}_h{head}_k"] = c[1]
                    out[f"{name}_x_l{layer}_h{head}_v"] = c[2]
                    out[f"{name}_x_l{layer}_h{head}_out"] = c[3]
        out[f"{name}_meta"] = np.array([L, H, d, prompt_len, block, extra], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_prefill.npz"), **out)


def make_analysis() -> None:
    """Similarity statistics and head-gate calibration from the reference
    (linalg.py:68-80, analysis.py:28-148, policy.py:110-246).  Writes
    tests/golden/golden_analysis.npz."""
    sys.path.insert(0, REF_SRC)
    import flashblock as fb
    from flashblock.analysis import PartialRecorder, pairwise_step_similarity
    from flashblock.linalg import cosine_similarity
    from flashblock.simulator import run_sequence

    rng = np.random.Generator(np.random.Philox(777))
    out: dict[str, np.ndarray] = {}
    heads, rows, d = 3, 20, 16
    a = rng.standard_normal((heads, rows, d))
    b = a + 0.3 * rng.standard_normal((heads, rows, d))
    a[0, 3] = 0.0           # zero-norm rows -> cosine 0
    b[1, 7] = 1e-14
    b[2] = -b[2]            # anti-correlated head
    out["cos_a"], out["cos_b"] = a, b
    out["cos_rows"] = np.array([[cosine_similarity(a[h, r], b[h, r]) for r in range(rows)]
                                for h in range(heads)])
    out["cos_mean"] = np.array([np.mean(out["cos_rows"][h]) for h in range(heads)])
    out["pair"] = np.stack([pairwise_step_similarity(a[h], b[h]) for h in range(heads)])

    # head-gate calibration on a tiny model: the recorded external partials of
    # every (layer, head, step) and the reference's own table
    cfg = fb.ModelConfig(num_layers=2, num_heads=3, head_dim=16, seed=4, query_noise=0.3,
                         noisy_heads=frozenset({(1, 2)}))
    model = fb.SyntheticModel(cfg)
    samples, gamma = 2, 0.995
    kw = dict(prompt_len=24, block_size=8, steps_per_block=6, unmask_per_step=1)
    for i in range(samples):
        rec = PartialRecorder()
        run_sequence(model, kw["prompt_len"], 1, kw["block_size"], kw["steps_per_block"],
                     fb.ReuseConfig(mode="always-recompute"), seed=i,
                     unmask_per_step=kw["unmask_per_step"], recorder=rec)
        for (layer, head, block), outs in rec.external_by_head().items():
            out[f"cal_s{i}_l{layer}_h{head}"] = np.stack(outs)  # [steps, rows, d]
    table = fb.calibrate_head_gates(model, samples, gamma, prompt_len=kw["prompt_len"],
                                    block_size=kw["block_size"],
                                    steps_per_block=kw["steps_per_block"],
                                    unmask_per_step=kw["unmask_per_step"], base_seed=0)
    out["cal_table_json"] = np.frombuffer(table.to_json().encode(), dtype=np.uint8)
    out["cal_meta"] = np.array([cfg.num_layers, cfg.num_heads, samples], dtype=np.int64)
    out["cal_gamma"] = np.array([gamma])
    np.savez_compressed(os.path.join(HERE, "golden_analysis.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "prefill":
        make_prefill()
    elif len(sys.argv) > 1 and sys.argv[1] == "analysis":
        make_analysis()
    else:
        main()
