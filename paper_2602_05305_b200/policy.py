"""Refresh schedule: reuse-or-recompute decision (drop-in for
flashblock/policy.py:33-107) plus the per-block schedule the engine runs.

Host logic; it must agree exactly with the reference (the driver of the GPU
kernels).  ``refresh_schedule`` is the closed form of what the reference
simulator decides per step in token-threshold mode: the Hamming distance M
seen at step s is the unmask count of step s-1 (simulator.py:388-392), and
the external cache is valid after step 0 (simulator.py:412-434).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import ShapeError

__all__ = ["Decision", "MODES", "ReuseConfig", "decide", "count_updated_tokens",
           "unmask_schedule", "refresh_schedule", "CalibrationError", "HeadGate", "HeadGateTable"]

MODES = ("token-threshold", "head-gated", "always-recompute", "always-reuse")  # policy.py:33


class Decision(Enum):
    REUSE = "Reuse"
    RECOMPUTE = "Recompute"


@dataclass(frozen=True)
class ReuseConfig:
    """tau (>= 1), gamma in [0, 1], mode in MODES (policy.py:45-68); defaults
    tau=2, gamma=0.9 as the paper."""

    tau: int = 2
    gamma: float = 0.9
    mode: str = "token-threshold"

    def __post_init__(self) -> None:
        if self.tau < 1:
            raise ValueError(f"tau must be >= 1, got {self.tau}")
        if not 0.0 <= self.gamma <= 1.0:
            raise ValueError(f"gamma must be in [0, 1], got {self.gamma}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}; expected one of {MODES}")


def decide(config: ReuseConfig, cache_valid: bool, first_visit: bool, updated_tokens: int,
           head_gate: bool = True) -> Decision:
    """policy.py:71-94: forced recompute without a valid cache, then the mode
    overrides, then the token threshold, then the head gate."""
    if first_visit or not cache_valid:
        return Decision.RECOMPUTE
    if config.mode == "always-recompute":
        return Decision.RECOMPUTE
    if config.mode == "always-reuse":
        return Decision.REUSE
    if updated_tokens >= config.tau:
        return Decision.RECOMPUTE
    if config.mode == "head-gated" and not head_gate:
        return Decision.RECOMPUTE
    return Decision.REUSE


def count_updated_tokens(prev_ids, curr_ids) -> int:
    """Hamming distance of equal-length token-id vectors (policy.py:97-107)."""
    prev = np.asarray(prev_ids)
    curr = np.asarray(curr_ids)
    if prev.shape != curr.shape or prev.ndim != 1:
        raise ShapeError(f"token id vectors differ in shape: {prev.shape} vs {curr.shape}")
    return int(np.count_nonzero(prev != curr))


def unmask_schedule(block_size: int, steps: int, per_step: int) -> list[int]:
    """Tokens revealed per step, remainder forced on the last step
    (simulator.py:258-286)."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    counts = [0] * steps
    if per_step <= 0:
        counts[-1] = block_size
        return counts
    events = min(steps, math.ceil(block_size / per_step))
    done = fired = 0
    for s in range(steps):
        target = ((s + 1) * events) // steps
        if target > fired:
            take = min(per_step * (target - fired), block_size - done)
            counts[s] = take
            done += take
            fired = target
    counts[-1] += block_size - done
    return counts


def refresh_schedule(config: ReuseConfig, block_size: int, steps: int,
                     per_step: int) -> list[Decision]:
    """Per-step decision for one block (all heads share it in token-threshold
    mode): decide(first_visit = s == 0, cache_valid = s > 0,
    M = unmask_schedule[s-1])."""
    sched = unmask_schedule(block_size, steps, per_step)
    return [decide(config, s > 0, s == 0, sched[s - 1] if s > 0 else 0) for s in range(steps)]


# ---------------------------------------------------------------- head gates


class CalibrationError(RuntimeError):
    """No usable gating signal (policy.py:41-42)."""


@dataclass(frozen=True)
class HeadGate:
    """Calibration record of one (layer, head) (policy.py:110-123): mean and
    worst adjacent-step cosine similarity of its external partials."""

    layer: int
    head: int
    similarity: float
    similarity_min: float
    enabled: bool


class HeadGateTable:
    """Per-head reuse gates (policy.py:126-181): enabled iff similarity > gamma.
    Same constructors, queries and JSON form as the reference."""

    def __init__(self, gamma: float, heads: list[HeadGate]):
        for g in heads:
            if g.enabled != (g.similarity > gamma):
                raise ValueError(f"gate for ({g.layer}, {g.head}) inconsistent with gamma={gamma}")
        self.gamma = gamma
        self.heads = list(heads)
        self._enabled = {(g.layer, g.head): g.enabled for g in heads}

    @classmethod
    def from_similarities(cls, gamma: float, stats: dict) -> "HeadGateTable":
        heads = [HeadGate(layer, head, mean, worst, mean > gamma)
                 for (layer, head), (mean, worst) in sorted(stats.items())]
        return cls(gamma, heads)

    def is_enabled(self, layer: int, head: int) -> bool:
        return self._enabled.get((layer, head), False)

    def to_json(self) -> str:
        import json

        return json.dumps({"gamma": self.gamma,
                           "heads": [{"layer": g.layer, "head": g.head, "similarity": g.similarity,
                                      "similarity_min": g.similarity_min, "enabled": g.enabled}
                                     for g in self.heads]}, indent=2, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "HeadGateTable":
        import json

        doc = json.loads(text)
        heads = [HeadGate(int(h["layer"]), int(h["head"]), float(h["similarity"]),
                          float(h.get("similarity_min", h["similarity"])), bool(h["enabled"]))
                 for h in doc["heads"]]
        return cls(float(doc["gamma"]), heads)

