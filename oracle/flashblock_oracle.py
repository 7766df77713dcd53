"""CPU oracle for the FlashBlock attention hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's hot-path
algorithm (``flashblock`` 0.1.0, ``/root/reference/pkg/src/flashblock``).  It
is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package ``paper_2602_05305_b200`` never imports it and has no CPU
fallback.

Parity pinning: ``tests/test_oracle.py`` checks every function here against
(a) the reference tests' frozen known-answer values and (b) golden
input/output vectors produced by running the real reference in the build
container (``tests/golden/make_golden.py``, fixtures in ``tests/golden/``).

Citations use ``attention.py:L`` for
``/root/reference/pkg/src/flashblock/attention.py`` line L (same for
``sparse.py``, ``policy.py``, ``simulator.py``, ``linalg.py``).

Semantics restated (not copied):

* a *partial* over a key group is ``(out, lognorm)`` with
  ``out = softmax(s) @ V`` over the group and ``lognorm = log sum exp(s)``;
  the empty group is the sentinel ``(0, -inf)`` (attention.py:60-101).
* the streamed partial computes scores ``q @ k.T * scale`` in the tensor
  dtype, and keeps max / normaliser / accumulator in float64, rescaling by
  ``exp(m_old - m_new)`` per key tile (attention.py:156-182).
* log-space merge of two partials (attention.py:207-233).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_TILE = 64          # attention.py:49
DEFAULT_KEY_BLOCK = 16     # sparse.py:40


class OracleShapeError(ValueError):
    pass


class OracleDegenerateError(ValueError):
    pass


class OracleReuseError(RuntimeError):
    pass


class OracleStalenessError(RuntimeError):
    pass


@dataclass
class Partial:
    """(out, lognorm) pair; lognorm is float64 (attention.py:70-71)."""

    out: np.ndarray
    lognorm: np.ndarray

    def empty_rows(self) -> np.ndarray:
        return np.isneginf(self.lognorm)


def _default_scale(d: int, scale):
    return 1.0 / math.sqrt(d) if scale is None else float(scale)


def dense(q, keys, values, scale=None) -> np.ndarray:
    """Float64 single-matrix softmax attention (attention.py:113-133)."""
    if keys.shape[0] == 0:
        raise OracleDegenerateError("no keys")
    sc = _default_scale(q.shape[1], scale)
    s = np.matmul(q.astype(np.float64), keys.astype(np.float64).T) * sc
    w = np.exp(s - np.max(s, axis=1, keepdims=True))
    return np.matmul(w, values.astype(np.float64)) / np.sum(w, axis=1, keepdims=True)


def block_causal(q, keys, values, n_prefix: int, n_q: int, block: int, scale=None) -> np.ndarray:
    """Block-causal prefill / commit attention (simulator.py:297-354).

    The reference commits a prompt block by block (prefill, simulator.py:343-354);
    each block's commit pass runs attention_dense over the committed context
    plus the block's own keys (simulator.py:316-320).  Restated for stacked
    query heads: q holds heads * n_q rows (row r at position p = r % n_q);
    rows of block j = p // block attend keys [0, n_prefix + min(n_q, (j+1)*block)).
    Returns the float64 outputs [rows, d].
    """
    rows = q.shape[0]
    if rows % n_q:
        raise OracleShapeError("q rows must be heads * n_q")
    out = np.empty((rows, values.shape[1]), dtype=np.float64)
    for h in range(rows // n_q):
        for j0 in range(0, n_q, block):
            j1 = min(j0 + block, n_q)
            lim = n_prefix + j1
            out[h * n_q + j0:h * n_q + j1] = dense(q[h * n_q + j0:h * n_q + j1], keys[:lim],
                                                   values[:lim], scale)
    return out


def partial(q, keys, values, scale=None, tile_size=DEFAULT_TILE) -> Partial:
    """Tile-streamed online-softmax partial (attention.py:136-182).

    Score product in the tensor dtype (attention.py:166), running statistics
    in float64 (attention.py:158-174), output cast back to the tensor dtype
    (attention.py:180), lognorm = m + log(l) (attention.py:181).
    """
    if tile_size < 1:
        raise ValueError("tile_size must be >= 1")
    sc = _default_scale(q.shape[1], scale)
    nq, dv = q.shape[0], values.shape[1]
    run_max = np.full(nq, -np.inf)
    run_sum = np.zeros(nq)
    acc = np.zeros((nq, dv))
    n = keys.shape[0]
    start = 0
    while start < n:
        stop = min(n, start + tile_size)
        s = (np.matmul(q, keys[start:stop].T) * sc).astype(np.float64)
        new_max = np.maximum(run_max, s.max(axis=1))
        shrink = np.exp(run_max - new_max)
        w = np.exp(s - new_max[:, None])
        run_sum = run_sum * shrink + w.sum(axis=1)
        acc = acc * shrink[:, None] + np.matmul(w, values[start:stop].astype(np.float64))
        run_max = new_max
        start = stop
    if n == 0:
        return Partial(np.zeros((nq, dv), dtype=q.dtype), np.full(nq, -np.inf))
    return Partial((acc / run_sum[:, None]).astype(q.dtype), run_max + np.log(run_sum))


def streamed(q, keys, values, boundary, scale=None, tile_size=DEFAULT_TILE):
    """External [0,b) / internal [b,n) split of one key stream (attention.py:185-204)."""
    if not 0 <= boundary <= keys.shape[0]:
        raise IndexError("boundary out of range")
    return (partial(q, keys[:boundary], values[:boundary], scale, tile_size),
            partial(q, keys[boundary:], values[boundary:], scale, tile_size))


def combine(a: Partial, b: Partial) -> Partial:
    """Log-space merge of two partials over disjoint key groups (attention.py:207-233).

    Rows empty on exactly one side pass the other side through bit-for-bit;
    rows empty on both sides stay empty.
    """
    if a.out.shape != b.out.shape:
        raise OracleShapeError("partial shapes differ")
    la = np.asarray(a.lognorm, dtype=np.float64)
    lb = np.asarray(b.lognorm, dtype=np.float64)
    top = np.maximum(la, lb)
    live = np.isfinite(top)
    out = np.zeros_like(a.out)
    lse = np.full(top.shape, -np.inf)
    if live.any():
        wa = np.exp(la[live] - top[live])
        wb = np.exp(lb[live] - top[live])
        z = wa + wb
        out[live] = (wa[:, None] * a.out[live] + wb[:, None] * b.out[live]) / z[:, None]
        lse[live] = top[live] + np.log(z)
    return Partial(out, lse)


def merge(external: Partial, internal: Partial) -> np.ndarray:
    """combine(...).out, refusing rows with no keys at all (attention.py:236-245)."""
    c = combine(external, internal)
    if c.empty_rows().any():
        raise OracleDegenerateError("rows with no keys")
    return c.out


def with_reuse(q, cached: Partial | None, valid: bool, k_in, v_in, scale=None,
               tile_size=DEFAULT_TILE):
    """Cached step: fresh internal partial merged with the cached external one
    (attention.py:295-321)."""
    if cached is None or not valid:
        raise OracleReuseError("no valid cached external partial")
    if cached.out.shape[0] != q.shape[0]:
        raise OracleReuseError("row count mismatch")
    inner = partial(q, k_in, v_in, scale, tile_size)
    return merge(cached, inner), inner


# ------------------------------------------------------------------ sparse


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (linalg.py:52-65)."""
    e = np.exp(x - x.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def block_mass(q, keys, boundary, key_block_size=DEFAULT_KEY_BLOCK, scale=None) -> np.ndarray:
    """Per external key block, the float64 softmax mass summed over every
    query row; the softmax runs over ALL keys passed, including the current
    block's (sparse.py:117-125)."""
    sc = _default_scale(q.shape[1], scale)
    probs = softmax_rows(np.matmul(q.astype(np.float64), keys.astype(np.float64).T) * sc)
    nb = -(-boundary // key_block_size)
    mass = np.empty(nb)
    for blk in range(nb):
        lo = blk * key_block_size
        mass[blk] = probs[:, lo:min(lo + key_block_size, boundary)].sum()
    return mass


def mask_budget(num_blocks: int, density: float, boundary: int, key_block_size: int) -> int:
    """min(nb, max(1, ceil(density * boundary / kbs))) in float64 (sparse.py:126)."""
    return min(num_blocks, max(1, math.ceil(density * boundary / key_block_size)))


def select_blocks(q, keys, boundary, density, key_block_size=DEFAULT_KEY_BLOCK,
                  scale=None) -> np.ndarray:
    """Top-mass key blocks, ties to the lower index, returned ascending
    (sparse.py:83-136)."""
    if not 0.0 < density <= 1.0:
        raise ValueError("density")
    if key_block_size < 1:
        raise ValueError("key_block_size")
    if not 0 <= boundary <= keys.shape[0]:
        raise ValueError("boundary")
    if boundary == 0:
        return np.empty(0, dtype=np.int64)
    mass = block_mass(q, keys, boundary, key_block_size, scale)
    k = mask_budget(mass.size, density, boundary, key_block_size)
    ranked = sorted(range(mass.size), key=lambda b: (-mass[b], b))
    return np.array(sorted(ranked[:k]), dtype=np.int64)


def expand_blocks(selected, key_block_size, n_ext) -> np.ndarray:
    """Block ids -> external row ids, tail block clipped (sparse.py:69-80)."""
    rows = [np.arange(b * key_block_size, min((b + 1) * key_block_size, n_ext))
            for b in selected]
    return np.concatenate(rows) if rows else np.empty(0, dtype=np.int64)


def sparse_with_residual(q, selected, key_block_size, n_ext, keys, values,
                         residual: Partial | None = None, scale=None, tile_size=64):
    """First step: exact partition into (selected ext + all internal) and
    residual (unselected ext) partials; later steps: selected partial merged
    with the cached residual (sparse.py:139-183).  Returns (out, residual,
    selected_partial)."""
    if keys.shape[0] < n_ext:
        raise OracleShapeError("fewer keys than the mask covers")
    sel_ext = expand_blocks(selected, key_block_size, n_ext)
    sel_rows = np.concatenate([sel_ext, np.arange(n_ext, keys.shape[0])]).astype(np.int64)
    sel_p = partial(q, keys[sel_rows], values[sel_rows], scale, tile_size)
    if residual is None:
        keep = np.ones(n_ext, dtype=bool)
        keep[sel_ext] = False
        res_rows = np.flatnonzero(keep)
        residual = partial(q, keys[res_rows], values[res_rows], scale, tile_size)
    return merge(sel_p, residual), residual, sel_p


# ------------------------------------------------------------------ policy


MODES = ("token-threshold", "head-gated", "always-recompute", "always-reuse")


def decide(mode: str, tau: int, cache_valid: bool, first_visit: bool,
           updated_tokens: int, head_gate: bool = True) -> str:
    """Refresh rule (policy.py:71-94): returns "Recompute" or "Reuse"."""
    if first_visit or not cache_valid or mode == "always-recompute":
        return "Recompute"
    if mode == "always-reuse":
        return "Reuse"
    if updated_tokens >= tau or (mode == "head-gated" and not head_gate):
        return "Recompute"
    return "Reuse"


def count_updated(prev_ids, curr_ids) -> int:
    """Hamming distance of token-id vectors (policy.py:97-107)."""
    a, b = np.asarray(prev_ids), np.asarray(curr_ids)
    if a.shape != b.shape or a.ndim != 1:
        raise OracleShapeError("shape")
    return int((a != b).sum())


def unmask_schedule(block_size: int, steps: int, per_step: int) -> list[int]:
    """Unmask counts per step, remainder forced on the last step
    (simulator.py:258-286)."""
    if steps < 1 or block_size < 1:
        raise ValueError("steps and block_size must be >= 1")
    out = [0] * steps
    if per_step <= 0:
        out[-1] = block_size
        return out
    events = min(steps, -(-block_size // per_step))
    revealed = fired = 0
    for s in range(steps):
        due = (s + 1) * events // steps
        if due > fired:
            n = min(per_step * (due - fired), block_size - revealed)
            out[s] = n
            revealed += n
            fired = due
    out[-1] += block_size - revealed
    return out


def refresh_schedule(block_size: int, steps: int, per_step: int, tau: int,
                     mode: str = "token-threshold") -> list[str]:
    """Per-step decision of one block in token-threshold mode.

    The simulator counts M as the Hamming distance between consecutive
    steps' ids (simulator.py:388-392), which under greedy unmasking equals
    the previous step's unmask count; the cache is valid after step 0
    (simulator.py:412-434).  Hence decision(s) = decide(first_visit=s==0,
    cache_valid=s>0, M=schedule[s-1]).
    """
    sched = unmask_schedule(block_size, steps, per_step)
    return [decide(mode, tau, s > 0, s == 0, sched[s - 1] if s else 0)
            for s in range(steps)]


# ---------------------------------------------------------------- similarity

ZERO_NORM_EPS = 1e-12  # linalg.py:25


def cosine_similarity(u, v) -> float:
    """Cosine of two 1-D vectors, 0.0 if either norm < 1e-12 (linalg.py:68-80)."""
    nu = float(np.linalg.norm(u))
    nv = float(np.linalg.norm(v))
    if nu < ZERO_NORM_EPS or nv < ZERO_NORM_EPS:
        return 0.0
    return float(np.dot(u, v) / (nu * nv))


def pairwise_step_similarity(out_s, out_s1) -> np.ndarray:
    """All-pairs cosine, entry (i, j) = cos(out_s1[i], out_s[j]) in float64;
    rows with near-zero norm map to 0 (analysis.py:28-51)."""
    a = np.asarray(out_s1, dtype=np.float64)
    b = np.asarray(out_s, dtype=np.float64)
    na = np.linalg.norm(a, axis=1)
    nb = np.linalg.norm(b, axis=1)
    den = np.outer(na, nb)
    sim = np.zeros_like(den)
    ok = den >= ZERO_NORM_EPS * ZERO_NORM_EPS
    np.divide(a @ b.T, den, out=sim, where=ok)
    sim[na < ZERO_NORM_EPS, :] = 0.0
    sim[:, nb < ZERO_NORM_EPS] = 0.0
    return sim


def gate_stats(runs) -> dict:
    """Head-gate statistics (policy.py:222-246): runs maps (layer, head) to a
    list (one entry per rollout) of step-ordered external partial outputs
    [steps, rows, d]; for every adjacent step pair the row-mean cosine is one
    sample; returns {(layer, head): (mean, min)} over all samples."""
    stats = {}
    for key, rollouts in runs.items():
        vals = []
        for outs in rollouts:
            for step in range(len(outs) - 1):
                prev, curr = outs[step], outs[step + 1]
                vals.append(float(np.mean([cosine_similarity(curr[r], prev[r])
                                           for r in range(curr.shape[0])])))
        stats[key] = (float(np.mean(vals)), float(np.min(vals)))
    return stats

