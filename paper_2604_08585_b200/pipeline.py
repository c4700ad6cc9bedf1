"""Virtual-clock cost model kept for API compatibility only.

`FusionEngine.run` in the reference fills `RunResult.schedule` / `ttft_sim`
from a declared cost model (pipeline.py:18-157, marked out of scope in
SURVEY §2 row 4). This module restates just enough of it (layer_times,
the pipelined schedule, the per-policy pre-phase) for `RunResult` to carry the
same fields; the B200 engine's real timings are CUDA-event measurements
(`RunResult.timings_ms`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .model import ModelConfig
from .store import TierConfig, layer_kv_bytes


@dataclass
class CostModel:
    compute_alpha: float = 1e-9
    compute_beta: float = 1e-4
    decode_gamma: float = 1e-3
    tier: TierConfig = field(default_factory=TierConfig)

    def __post_init__(self):
        if min(self.compute_alpha, self.compute_beta, self.decode_gamma) < 0:
            raise ValueError("cost coefficients must be >= 0")


@dataclass
class ScheduleTrace:
    pre_phase: float
    fetch_start: list[float]
    fetch_end: list[float]
    compute_start: list[float]
    compute_end: list[float]
    ttft: float

    @property
    def n_layers(self) -> int:
        return len(self.fetch_start)


def layer_times(n_sel: int, n_ctx: int, config: ModelConfig, cost: CostModel) -> tuple[float, float]:
    fetch = cost.tier.fetch_seconds(layer_kv_bytes(n_ctx, config.n_kv_heads, config.d_head))
    return fetch, cost.compute_alpha * n_sel * n_ctx * config.n_heads * config.d_head + cost.compute_beta


def schedule_pipelined(fetch, compute, pre_phase: float = 0.0) -> ScheduleTrace:
    """One serialized fetch channel overlapped with layer compute."""
    if len(fetch) != len(compute):
        raise ValueError("fetch and compute must have equal length")
    if pre_phase < 0 or min(list(fetch) + list(compute) + [0.0]) < 0:
        raise ValueError("durations must be >= 0")
    fs, fe, cs, ce = [], [], [], []
    tf = tc = pre_phase
    for f, c in zip(fetch, compute):
        fs.append(tf)
        tf += f
        fe.append(tf)
        st = max(tc, tf)
        cs.append(st)
        tc = st + c
        ce.append(tc)
    return ScheduleTrace(pre_phase, fs, fe, cs, ce, ce[-1] if ce else pre_phase)


def policy_prephase(policy: str, n_ctx: int, n_query: int, config: ModelConfig, cost: CostModel) -> float:
    unit = config.n_heads * config.d_head
    full = cost.tier.fetch_seconds(layer_kv_bytes(n_ctx, config.n_kv_heads, config.d_head))
    if policy in ("FullCompute", "FullReuse", "EPIC", "Random"):
        return 0.0
    if policy in ("QCFuse", "QCLast"):
        return (cost.compute_alpha * n_query * n_ctx * unit + cost.compute_beta
                + cost.tier.fetch_seconds(layer_kv_bytes(n_ctx, config.n_kv_heads, config.d_head) // 2))
    if policy == "QCAll":
        return config.n_layers * full
    if policy in ("CacheBlend", "KVShare"):
        return full + cost.compute_alpha * n_ctx * n_ctx * unit + cost.compute_beta
    raise ValueError(f"unknown policy: {policy}")


def policy_schedule(policy: str, n_sel: int, n_ctx: int, n_query: int, config: ModelConfig,
                    cost: CostModel) -> ScheduleTrace:
    L = config.n_layers
    fetch, comp = layer_times(n_sel, n_ctx, config, cost)
    pre = policy_prephase(policy, n_ctx, n_query, config, cost)
    if policy == "FullCompute":
        return schedule_pipelined([0.0] * L, [layer_times(n_ctx, n_ctx, config, cost)[1]] * L)
    if policy == "FullReuse":
        return schedule_pipelined([fetch] * L, [0.0] * L)
    if policy == "QCAll":
        return schedule_pipelined([0.0] * L, [comp] * L, pre)
    return schedule_pipelined([fetch] * L, [comp] * L, pre)


def schedule_events(schedule: ScheduleTrace) -> list[dict]:
    ev = []
    for i in range(schedule.n_layers):
        ev.append({"kind": "fetch", "layer": i + 1, "start": schedule.fetch_start[i], "end": schedule.fetch_end[i]})
        ev.append({"kind": "compute", "layer": i + 1, "start": schedule.compute_start[i],
                   "end": schedule.compute_end[i]})
    ev.sort(key=lambda e: (e["start"], e["layer"], e["kind"] == "compute"))
    return ev
