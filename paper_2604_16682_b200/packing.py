"""Host-side packing of scenarios into the C-ABI structure-of-arrays layout.

* traces -> one CSR pool (``AsbTracePool``) shared by every scenario that
  replays the same trace (C3/C5 share one trace across many cells);
* frequency tables -> ``AsbTablePool`` (rates/powers computed on the host by
  the reference formula, instance.py:83-112, so the device never evaluates
  ``pow``);
* SimConfig -> one ``AsbScenario`` record (engine.py:57-88), validated on the
  host first so ConfigurationError surfaces exactly where the reference
  raises it (engine.py:252);
* output offsets (agent rows, instance rows, decision rows, turn rows).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigurationError
from .instance import FrequencyTable
from .workload import AgentTrace


@dataclass
class TracePool:
    trace_agent_off: np.ndarray
    trace_turn_off: np.ndarray
    arrival: np.ndarray
    agent_turn_off: np.ndarray
    prefill: np.ndarray
    decode: np.ndarray
    tool: np.ndarray
    arrival_order: np.ndarray
    agent_ids: list = field(default_factory=list)  # per trace: list[str] or None

    @property
    def n_traces(self) -> int:
        return int(self.trace_agent_off.size - 1)

    def n_agents(self, t: int) -> int:
        return int(self.trace_agent_off[t + 1] - self.trace_agent_off[t])

    def n_turns(self, t: int) -> int:
        return int(self.trace_turn_off[t + 1] - self.trace_turn_off[t])

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in _abi.TRACE_FIELDS}


@dataclass
class TablePool:
    table_off: np.ndarray
    mhz: np.ndarray
    prefill_rate: np.ndarray
    decode_rate: np.ndarray
    active_power: np.ndarray
    idle_power: np.ndarray

    @property
    def n_tables(self) -> int:
        return int(self.table_off.size - 1)

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in _abi.TABLE_FIELDS}


def trace_arrays_from_objects(traces: list[AgentTrace]) -> dict:
    """AgentTrace objects -> CSR arrays of one trace (agent order preserved)."""
    n = len(traces)
    counts = np.fromiter((len(t.turns) for t in traces), dtype=np.int64, count=n)
    turn_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=turn_off[1:])
    total = int(turn_off[-1])
    flat = [(r.prefill_tokens, r.decode_tokens, r.tool_time) for t in traces for r in t.turns]
    if total:
        pre, dec, tool = zip(*flat)
        prefill = np.asarray(pre, dtype=np.int64)
        decode = np.asarray(dec, dtype=np.int64)
        tool_a = np.asarray(tool, dtype=np.float64)
    else:
        prefill = np.zeros(0, np.int64)
        decode = np.zeros(0, np.int64)
        tool_a = np.zeros(0, np.float64)
    if total and (prefill.max() > np.iinfo(np.int32).max or decode.max() > np.iinfo(np.int32).max):
        raise ConfigurationError("turn token counts must fit in int32 for the B200 engine")
    return {
        "arrival": np.fromiter((t.arrival_time for t in traces), dtype=np.float64, count=n),
        "turn_off": turn_off,
        "prefill": prefill.astype(np.int32),
        "decode": decode.astype(np.int32),
        "tool": tool_a,
        "agent_ids": [t.agent_id for t in traces],
    }


def pack_traces(trace_arrays: list[dict]) -> TracePool:
    """Concatenate per-trace CSR arrays into one pool."""
    n_traces = len(trace_arrays)
    agent_counts = [int(t["arrival"].size) for t in trace_arrays]
    turn_counts = [int(t["turn_off"][-1]) for t in trace_arrays]
    trace_agent_off = np.zeros(n_traces + 1, dtype=np.int64)
    np.cumsum(agent_counts, out=trace_agent_off[1:])
    trace_turn_off = np.zeros(n_traces + 1, dtype=np.int64)
    np.cumsum(turn_counts, out=trace_turn_off[1:])
    n_agents = int(trace_agent_off[-1])
    agent_turn_off = np.empty(n_agents + 1, dtype=np.int64)
    orders = []
    for t, arr in enumerate(trace_arrays):
        a0, a1 = trace_agent_off[t], trace_agent_off[t + 1]
        agent_turn_off[a0:a1] = arr["turn_off"][:-1] + trace_turn_off[t]
        # arrival events sort by (time, trace index): engine.py:300-301, 315-317
        orders.append(np.argsort(arr["arrival"], kind="stable").astype(np.int32))
    agent_turn_off[n_agents] = trace_turn_off[-1]

    def cat(key, dtype):
        if not trace_arrays:
            return np.zeros(0, dtype)
        return np.ascontiguousarray(np.concatenate([np.asarray(t[key], dtype=dtype) for t in trace_arrays]))

    arrival = cat("arrival", np.float64)
    if arrival.size and (np.isnan(arrival).any() or (arrival < 0).any()):
        raise ConfigurationError("arrival_time must be a number >= 0")
    return TracePool(
        trace_agent_off=trace_agent_off,
        trace_turn_off=trace_turn_off,
        arrival=arrival,
        agent_turn_off=agent_turn_off,
        prefill=cat("prefill", np.int32),
        decode=cat("decode", np.int32),
        tool=cat("tool", np.float64),
        arrival_order=np.ascontiguousarray(np.concatenate(orders)) if orders else np.zeros(0, np.int32),
        agent_ids=[t.get("agent_ids") for t in trace_arrays],
    )


def pack_tables(tables: list[FrequencyTable]) -> TablePool:
    counts = [t.num_levels for t in tables]
    off = np.zeros(len(tables) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    levels = [lvl for t in tables for lvl in t.levels]
    return TablePool(
        table_off=off,
        mhz=np.array([lv.nominal_mhz for lv in levels], dtype=np.float64),
        prefill_rate=np.array([lv.prefill_rate for lv in levels], dtype=np.float64),
        decode_rate=np.array([lv.decode_rate for lv in levels], dtype=np.float64),
        active_power=np.array([lv.active_power for lv in levels], dtype=np.float64),
        idle_power=np.array([lv.idle_power for lv in levels], dtype=np.float64),
    )


def epoch_count(sim_duration: float, epoch_length: float) -> int:
    """#{k >= 0 : k * epoch_length < sim_duration} with the reference's
    multiplication (engine.py:306-309), without a per-epoch Python loop."""
    k = max(int(sim_duration / epoch_length) - 2, 0)
    while k > 0 and (k - 1) * epoch_length >= sim_duration:
        k -= 1
    while k * epoch_length < sim_duration:
        k += 1
    return k


MAX_AGENTS = 1 << 21  # agent ids live in 21 bits of the engine's alive-slot word (engine_core.h Slot)
MAX_INSTANCES = 127   # instance ids live in 7 bits of it (ASB_MAX_INSTANCES)
MAX_LEVELS = 64       # ASB_MAX_LEVELS: frequency tables staged in shared memory


def scenario_record(config, trace_id: int, table_id: int) -> tuple:
    """One AsbScenario row for a validated SimConfig."""
    inst = config.instance
    ctl = config.controller
    rt = config.router
    table = inst.frequency_table
    fixed_level = table.index_of_mhz(ctl.fixed_level_mhz) if ctl.variant == "fixed" else 0
    if config.instance_count > MAX_INSTANCES:
        raise ConfigurationError(
            f"instance_count: the B200 engine supports at most {MAX_INSTANCES} instances per scenario")
    if table.num_levels > MAX_LEVELS:
        raise ConfigurationError(f"frequency_table: the B200 engine supports at most {MAX_LEVELS} levels")
    rec = np.zeros((), dtype=_abi.SCENARIO_DTYPE)
    rec["trace_id"] = trace_id
    rec["table_id"] = table_id
    rec["n_instances"] = config.instance_count
    rec["n_levels"] = table.num_levels
    rec["capacity"] = int(inst.capacity_tokens)
    rec["thrash_factor"] = float(inst.thrash_latency_factor)
    rec["interference"] = float(inst.interference_coeff)
    rec["variant"] = _abi.VARIANTS[ctl.variant]
    rec["fixed_level"] = fixed_level
    rec["boost_enabled"] = int(bool(ctl.boost_enabled))
    rec["thrash_avoidance"] = int(bool(ctl.thrash_avoidance))
    rec["alpha"] = ctl.alpha
    rec["beta"] = ctl.beta
    rec["gamma"] = ctl.gamma
    rec["slo_target"] = ctl.slo_target
    rec["epoch_length"] = ctl.epoch_length
    rec["policy"] = _abi.POLICIES[rt.policy]
    rec["reassign_interval"] = int(rt.reassign_interval)
    rec["include_idle"] = int(bool(rt.include_idle_instances))
    rec["reset_only_on_reassign"] = int(bool(rt.reset_counter_only_on_reassign))
    rec["consolidation_threshold"] = rt.consolidation_threshold
    rec["imbalance_ratio"] = rt.imbalance_ratio
    rec["migration_delay"] = rt.migration_delay
    rec["sim_duration"] = config.sim_duration
    rec["n_epochs"] = epoch_count(config.sim_duration, ctl.epoch_length)
    rec["record_interval"] = config.record_interval
    return rec


def sample_count(sim_duration: float, record_interval: float) -> int:
    """#{k >= 1 : k * record_interval < sim_duration}: the sample events of
    _schedule_initial (engine.py:310-313)."""
    return max(epoch_count(sim_duration, record_interval) - 1, 0)


def timeseries_capacity(scen: np.ndarray, a_cnt: np.ndarray, t_cnt: np.ndarray) -> np.ndarray:
    """Per-scenario row bound that _mark_row can never exceed.

    * one row per instance at start, end, every sample and every epoch
      (engine.py:488, 572, 579, 603);
    * one per arrival (engine.py:507) and one per completion (engine.py:535);
    * a tool event (at most T - A of them: the last turn has none) marks its
      source and, when it migrates, its target (engine.py:549, 560-561);
    * a delayed start (engine.py:568) follows only a migration, so at most
      one per tool event.

    Every agent has at least one turn (workload.py:114-115), so T >= A."""
    m = scen["n_instances"].astype(np.int64)
    samples = np.array([sample_count(float(r["sim_duration"]), float(r["record_interval"])) for r in scen],
                       dtype=np.int64).reshape(-1)
    tools = np.maximum(t_cnt - a_cnt, 0)
    return m * (2 + samples + scen["n_epochs"].astype(np.int64)) + a_cnt + t_cnt + 3 * tools


@dataclass
class Batch:
    """Everything one engine launch needs (host numpy arrays)."""

    scen: np.ndarray          # SCENARIO_DTYPE[n]
    traces: TracePool
    tables: TablePool
    agent_off: np.ndarray     # i64[n+1]
    inst_off: np.ndarray      # i64[n+1]
    dec_off: np.ndarray       # i64[n+1]
    turn_off: np.ndarray      # i64[n+1]
    ts_off: np.ndarray        # i64[n+1] timeseries row capacity (timeseries_capacity)
    total_agents: int
    total_ring: int
    max_instances: int
    min_instances: int = 0
    max_levels: int = 0      # the largest frequency table (AsbTablePool.max_levels)

    @property
    def n(self) -> int:
        return int(self.scen.size)

    @property
    def launch_instances(self) -> int:
        """asb_run_scenarios' max_instances argument: -m when every scenario
        has exactly m instances (a fixed-count kernel), else the maximum."""
        return -self.max_instances if self.min_instances == self.max_instances else self.max_instances


def build_batch(scen: np.ndarray, traces: TracePool, tables: TablePool) -> Batch:
    n = scen.size
    tid = scen["trace_id"].astype(np.int64)
    a_cnt = traces.trace_agent_off[tid + 1] - traces.trace_agent_off[tid]
    if n and int(a_cnt.max()) >= MAX_AGENTS:
        raise ConfigurationError(f"workload: the B200 engine supports at most {MAX_AGENTS - 1} agents per scenario")
    t_cnt = traces.trace_turn_off[tid + 1] - traces.trace_turn_off[tid]
    m = scen["n_instances"].astype(np.int64)

    def offs(counts):
        o = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=o[1:])
        return o

    return Batch(
        scen=np.ascontiguousarray(scen),
        traces=traces,
        tables=tables,
        agent_off=offs(a_cnt),
        inst_off=offs(m),
        dec_off=offs(m * scen["n_epochs"].astype(np.int64)),
        turn_off=offs(t_cnt),
        ts_off=offs(timeseries_capacity(scen, a_cnt, t_cnt)) if n else np.zeros(1, dtype=np.int64),
        total_agents=int(a_cnt.sum()),
        total_ring=int((m * a_cnt).sum()),
        max_instances=int(m.max()) if n else 1,
        min_instances=int(m.min()) if n else 1,
        max_levels=int(np.diff(tables.table_off).max()) if tables.table_off.size > 1 else 0,
    )
