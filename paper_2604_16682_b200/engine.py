"""Drop-in ``run_simulation`` on the B200 engine (mirror of agentsim/engine.py).

``run_simulation(config)`` (engine.py:752-754) and the batched entry
``run_simulation_batch(configs)`` validate on the host, pack the scenarios
into the C-ABI layout (packing.py), run them with ``asb_run_scenarios`` on
the GPU (one warp per scenario) and rebuild the reference's result objects.
``DeviceBatch`` keeps a packed batch resident in HBM for repeated runs (the
benchmark's timed region).

Timeseries rows (``_mark_row``, engine.py:403-429) are produced on the
device when asked for (``timeseries=True``, the default of
``run_simulation``): those scenarios run the engine's exact serial event
loop, sample events included, instead of the optimistic batches.  Batches
default to ``timeseries=False`` (``SimulationResult.timeseries`` empty).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Mapping, Sequence

import numpy as np

from . import _abi, packing
from .controller import ControllerConfig
from .errors import ConfigurationError, SimulationError
from .instance import InstanceConfig
from .metrics import AgentMetrics, SystemMetrics
from .router import RouterConfig
from .workload import (AgentTrace, WorkloadSpec, generate_workload, generate_workload_arrays, load_trace,
                       load_trace_arrays)


@dataclass
class SimConfig:
    """Full description of one simulation run (engine.py:57-88)."""

    workload: WorkloadSpec | None = None
    trace_path: str | None = None
    traces: list[AgentTrace] | None = None
    instance_count: int = 1
    instance: InstanceConfig = field(default_factory=InstanceConfig)
    controller: ControllerConfig = field(default_factory=ControllerConfig)
    router: RouterConfig = field(default_factory=RouterConfig)
    sim_duration: float = 3600.0
    record_interval: float = 1.0
    seed: int | None = None

    def validate(self) -> None:
        if self.instance_count < 1:
            raise ConfigurationError(f"instance_count: must be >= 1, got {self.instance_count}")
        if not self.sim_duration > 0:
            raise ConfigurationError(f"sim_duration: must be > 0, got {self.sim_duration}")
        if not self.record_interval > 0:
            raise ConfigurationError(f"record_interval: must be > 0, got {self.record_interval}")
        n_sources = sum(x is not None for x in (self.workload, self.trace_path, self.traces))
        if n_sources == 0:
            raise ConfigurationError("workload: either a workload spec or a trace source is required")
        if n_sources > 1:
            raise ConfigurationError("workload: provide exactly one of workload spec, trace_path, traces")
        if self.workload is not None:
            self.workload.validate()
        self.instance.validate()
        self.controller.validate(self.instance.frequency_table)
        self.router.validate()


@dataclass(frozen=True)
class TimeseriesRow:
    time: float
    instance_id: int
    context_usage: int
    level_index: int
    level_mhz: float
    power_watts: float
    pending_depth: int
    running_requests: int
    thrashing: int


@dataclass(frozen=True)
class DecisionRow:
    time: float
    instance_id: int
    usage_observed: int
    frequency_level: int
    boosted: bool
    deferred: bool
    admitted_count: int
    min_throughput: float | None
    pending_depth: int


@dataclass(frozen=True)
class AgentResult:
    agent_id: str
    arrival_time: float
    completion_time: float | None
    completed: bool
    turns_total: int
    turns_completed: int
    max_context_tokens: int
    total_llm_time: float
    total_decode_tokens: int
    throughput: float | None
    final_instance: int | None
    migrations: int
    final_phase: str
    turn_log: tuple[tuple[int, float, float], ...]


@dataclass
class SimulationResult:
    sim_duration: float
    instance_count: int
    capacity_tokens: int
    arrived: int
    completed: int
    agents: list[AgentResult]
    timeseries: list[TimeseriesRow]
    decisions: list[DecisionRow]
    instance_energy: dict[int, float]
    instance_thrash_time: dict[int, float]
    final_pending: dict[int, int]
    final_usage: dict[int, int]
    system: SystemMetrics
    config_echo: dict
    counters: dict = field(default_factory=dict)

    def agent_metrics(self) -> list[AgentMetrics]:
        return [
            AgentMetrics(a.agent_id, a.throughput, a.completed, a.turns_completed, a.max_context_tokens,
                         a.total_llm_time, a.total_decode_tokens)
            for a in self.agents
        ]

    def power_series(self) -> dict[int, list[tuple[float, float]]]:
        series: dict[int, list[tuple[float, float]]] = {r.instance_id: [] for r in self.timeseries}
        for r in self.timeseries:
            series[r.instance_id].append((r.time, r.power_watts))
        return series

    def usage_series(self) -> dict[int, list[tuple[float, float]]]:
        series: dict[int, list[tuple[float, float]]] = {r.instance_id: [] for r in self.timeseries}
        for r in self.timeseries:
            series[r.instance_id].append((r.time, float(r.context_usage)))
        return series


def integrate_power(series: Mapping[int, Sequence[tuple[float, float]]], window: float) -> float:
    """Average watts over [0, window] of piecewise-constant series (engine.py:185-207)."""
    if not window > 0:
        raise ConfigurationError(f"window: must be > 0, got {window}")
    total = 0.0
    for iid, pts in series.items():
        if not pts or pts[0][0] > 0.0:
            raise SimulationError(f"power series for instance {iid} does not cover the window start")
        for (t0, w0), (t1, _) in zip(pts, pts[1:]):
            if t1 < t0:
                raise SimulationError(f"power series for instance {iid} is not time-ordered")
            total += w0 * (min(t1, window) - min(t0, window))
        t_last, w_last = pts[-1]
        if t_last < window:
            total += w_last * (window - t_last)
    return total / window


# --------------------------------------------------------------------------- config echo


def _dist_echo(dist) -> dict:
    return {"dist": dist.kind, "mean": dist.mean, "sigma": dist.sigma, "min": dist.minimum,
            "max": None if dist.maximum == float("inf") else dist.maximum}


def config_echo(config: SimConfig) -> dict:
    """Deterministic dict describing the run (engine.py:680-739)."""
    inst, ctl, rt = config.instance, config.controller, config.router
    echo: dict = {
        "instance_count": config.instance_count,
        "sim_duration": config.sim_duration,
        "record_interval": config.record_interval,
        "seed": config.seed,
        "instance": {
            "capacity_tokens": inst.capacity_tokens,
            "thrash_mode": inst.thrash_mode,
            "thrash_latency_factor": inst.thrash_latency_factor,
            "interference_coeff": inst.interference_coeff,
            "frequency_table": [
                {"mhz": lv.nominal_mhz, "prefill_rate": lv.prefill_rate, "decode_rate": lv.decode_rate,
                 "active_power": lv.active_power, "idle_power": lv.idle_power}
                for lv in inst.frequency_table.levels
            ],
        },
        "controller": {
            "variant": ctl.variant, "alpha": ctl.alpha, "beta": ctl.beta, "gamma": ctl.gamma,
            "slo_target": ctl.slo_target, "epoch_length": ctl.epoch_length, "boost_enabled": ctl.boost_enabled,
            "thrash_avoidance": ctl.thrash_avoidance, "fixed_level_mhz": ctl.fixed_level_mhz,
        },
        "router": {
            "policy": rt.policy, "consolidation_threshold": rt.consolidation_threshold,
            "reassign_interval": rt.reassign_interval, "imbalance_ratio": rt.imbalance_ratio,
            "migration_delay": rt.migration_delay,
        },
    }
    if config.trace_path is not None:
        echo["workload"] = {"trace_path": config.trace_path}
    elif config.workload is not None:
        spec = config.workload
        echo["workload"] = {
            "arrival_rate": spec.arrival_rate, "arrival_process": spec.arrival_process, "duration": spec.duration,
            "seed": spec.seed, "prefill_growth_per_turn": spec.prefill_growth_per_turn,
            "turn_count": _dist_echo(spec.turn_count), "prefill_tokens": _dist_echo(spec.prefill_tokens),
            "decode_tokens": _dist_echo(spec.decode_tokens), "tool_time": _dist_echo(spec.tool_time),
        }
    else:
        echo["workload"] = {"inline_traces": len(config.traces or [])}
    return echo


# --------------------------------------------------------------------------- batching


def _trace_key(config: SimConfig):
    if config.traces is not None:
        return ("objects", id(config.traces))
    if config.trace_path is not None:
        return ("path", config.trace_path)
    spec = config.workload
    if config.seed is not None and config.seed != spec.seed:
        spec = replace(spec, seed=config.seed)
    return ("spec", spec)


def _resolve(config: SimConfig, key) -> list[AgentTrace]:
    if key[0] == "objects":
        traces = list(config.traces)
    elif key[0] == "path":
        traces = load_trace(config.trace_path)
    else:
        traces = generate_workload(key[1])
    seen: set[str] = set()
    for t in traces:
        if t.agent_id in seen:
            raise ConfigurationError(f"duplicate agent_id {t.agent_id!r} in workload")
        seen.add(t.agent_id)
    return traces


def _generate_specs(specs: list, workers: int | None) -> dict:
    """generate_workload_arrays of many WorkloadSpecs, in worker processes
    when there are many (each seed is an independent numpy stream)."""
    import os

    if workers is None:
        try:
            workers = len(os.sched_getaffinity(0))
        except AttributeError:
            workers = os.cpu_count() or 1
    workers = min(workers, len(specs), 32)
    if workers <= 1 or len(specs) < 16:
        return {sp: generate_workload_arrays(sp) for sp in specs}
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        return dict(zip(specs, ex.map(generate_workload_arrays, specs)))


def prepare_batch(configs: Sequence[SimConfig], workers: int | None = None) -> packing.Batch:
    """Validate (raising ConfigurationError before any device work), resolve
    and de-duplicate traces and tables, and pack the batch.  Distinct
    WorkloadSpecs are generated in ``workers`` processes (default: the host's
    cores) when there are 16 or more."""
    for c in configs:
        c.validate()
    specs = list(dict.fromkeys(k[1] for k in map(_trace_key, configs) if k[0] == "spec"))
    generated = _generate_specs(specs, workers) if specs else {}
    trace_index: dict = {}
    trace_arrays: list[dict] = []
    table_index: dict = {}
    tables = []
    recs = []
    for c in configs:
        key = _trace_key(c)
        if key not in trace_index:
            trace_index[key] = len(trace_arrays)
            if key[0] == "path":
                arrs = load_trace_arrays(c.trace_path)  # native JSONL -> CSR (csrc/trace_io.cpp)
                ids = arrs["agent_ids"]
                if len(set(ids)) != len(ids):  # the reference's duplicate check and message
                    _resolve(c, key)
            elif key[0] == "spec":
                # generate_workload's exact draws straight into CSR arrays; its
                # ids are "a%06d" by position (unique), built only on demand
                arrs = generated[key[1]]
                arrs["agent_ids"] = None
            else:
                arrs = packing.trace_arrays_from_objects(_resolve(c, key))
            trace_arrays.append(arrs)
        tab = c.instance.frequency_table
        if tab not in table_index:
            table_index[tab] = len(tables)
            tables.append(tab)
        recs.append(packing.scenario_record(c, trace_index[key], table_index[tab]))
    scen = np.array(recs, dtype=_abi.SCENARIO_DTYPE) if recs else np.zeros(0, dtype=_abi.SCENARIO_DTYPE)
    return packing.build_batch(scen, packing.pack_traces(trace_arrays), packing.pack_tables(tables))


def alloc_host_outputs(batch: packing.Batch, decisions: bool = True, turn_log: bool = True,
                       timeseries: bool = False) -> dict:
    """numpy output buffers matching AsbOutputs (used by host-side checkers)."""
    arrays = {"agent_off": batch.agent_off, "inst_off": batch.inst_off}
    for k, dt in _abi.AGENT_OUT.items():
        arrays[k] = np.zeros(batch.total_agents, dtype=dt)
    n_inst = int(batch.inst_off[-1])
    for k, dt in _abi.INST_OUT.items():
        arrays[k] = np.zeros(n_inst, dtype=dt)
    arrays["counters"] = np.zeros(batch.n * _abi.ASB_NCOUNTERS, dtype=np.int64)
    if decisions:
        arrays["dec_off"] = batch.dec_off
        arrays["decisions"] = np.zeros(int(batch.dec_off[-1]), dtype=_abi.DECISION_DTYPE)
    if turn_log:
        arrays["turn_off"] = batch.turn_off
        arrays["turn_issue"] = np.zeros(int(batch.turn_off[-1]), dtype=np.float64)
        arrays["turn_done"] = np.zeros(int(batch.turn_off[-1]), dtype=np.float64)
    if timeseries:
        arrays["ts_off"] = batch.ts_off
        arrays["timeseries"] = np.zeros(int(batch.ts_off[-1]), dtype=_abi.TIMESERIES_DTYPE)
        arrays["ts_count"] = np.zeros(batch.n, dtype=np.int64)
    return arrays


class DeviceBatch:
    """A packed batch resident in HBM plus its outputs and workspace.

    ``run()`` enqueues the engine, the per-scenario stats and the stats
    fold on the current stream (no host sync); ``download()`` copies back.
    """

    def __init__(self, batch: packing.Batch, device=None, decisions: bool = False, turn_log: bool = False,
                 timeseries: bool = False):
        import torch

        from . import _native, ops  # noqa: F401  (registers the custom ops)

        self.batch = batch
        self.device = _native.device(device)
        dev = self.device

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self.scen = up(batch.scen.view(np.uint8))
        self.traces = [up(getattr(batch.traces, k)) for k in _abi.TRACE_FIELDS]
        self.tables = [up(getattr(batch.tables, k)) for k in _abi.TABLE_FIELDS]
        n_inst = int(batch.inst_off[-1])
        outs = {"agent_off": up(batch.agent_off), "inst_off": up(batch.inst_off)}
        for name, tdt in ops.OUT_ORDER:
            if name in outs:
                continue
            if name in _abi.AGENT_OUT:
                outs[name] = torch.empty(batch.total_agents, dtype=tdt, device=dev)
            elif name in _abi.INST_OUT:
                outs[name] = torch.empty(n_inst, dtype=tdt, device=dev)
            elif name == "counters":
                outs[name] = torch.zeros(batch.n * _abi.ASB_NCOUNTERS, dtype=tdt, device=dev)
            elif name == "dec_off":
                outs[name] = up(batch.dec_off) if decisions else torch.empty(0, dtype=tdt, device=dev)
            elif name == "decisions":
                nbytes = int(batch.dec_off[-1]) * _abi.DECISION_DTYPE.itemsize if decisions else 0
                outs[name] = torch.empty(nbytes, dtype=tdt, device=dev)
            elif name == "turn_off":
                outs[name] = up(batch.turn_off) if turn_log else torch.empty(0, dtype=tdt, device=dev)
            elif name == "ts_off":
                outs[name] = up(batch.ts_off) if timeseries else torch.empty(0, dtype=tdt, device=dev)
            elif name == "timeseries":
                nbytes = int(batch.ts_off[-1]) * _abi.TIMESERIES_DTYPE.itemsize if timeseries else 0
                outs[name] = torch.empty(nbytes, dtype=tdt, device=dev)
            elif name == "ts_count":
                outs[name] = torch.zeros(batch.n if timeseries else 0, dtype=tdt, device=dev)
            else:  # turn_issue / turn_done
                n = int(batch.turn_off[-1]) if turn_log else 0
                outs[name] = torch.empty(n, dtype=tdt, device=dev)
        self.outputs = outs
        self.out_list = [outs[k] for k in ops.OUT_NAMES]
        ws_bytes = _native.lib().asb_workspace_bytes(batch.n, batch.total_agents, batch.total_ring)
        self.workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self.stats = torch.empty(batch.n * _abi.STATS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.red = torch.zeros(_abi.ASB_NRED, dtype=torch.float64, device=dev)

    def run(self) -> None:
        import torch

        b = self.batch
        if b.n == 0:
            return
        torch.ops.agentsim_b200.run_scenarios(self.scen, self.traces, self.tables, self.out_list, self.workspace,
                                              b.launch_instances, b.total_agents, b.total_ring, b.max_levels)
        torch.ops.agentsim_b200.scenario_stats(self.scen, self.out_list, self.stats)
        torch.ops.agentsim_b200.reduce_stats(self.stats, self.outputs["counters"], b.n, self.red)

    def regime_classify(self, capacity: Sequence[float] | None = None,
                        window: Sequence[float] | None = None) -> list[tuple[dict, float]]:
        """``regime_classify(result.usage_series(), capacity, window)``
        (metrics.py:72-109) for every scenario, on the device, straight from
        the timeseries rows of the last ``run()`` (``timeseries=True``):
        ``[(segments, thrash_fraction)]`` with segments ``{instance_id:
        [(start, end, thrashing), ...]}``.  Defaults: each scenario's
        ``capacity_tokens`` and ``sim_duration``."""
        import torch

        from . import _native

        b = self.batch
        if not self.outputs["ts_count"].numel():
            raise ConfigurationError("regime_classify needs the timeseries rows: DeviceBatch(..., timeseries=True)")
        cap = np.asarray(capacity if capacity is not None else b.scen["capacity"], dtype=np.float64)
        win = np.asarray(window if window is not None else b.scen["sim_duration"], dtype=np.float64)
        if cap.shape != (b.n,) or win.shape != (b.n,):
            raise ConfigurationError("regime_classify: one capacity and one window per scenario")
        if not (win > 0).all():
            raise ConfigurationError(f"window: must be > 0, got {float(win[~(win > 0)][0])}")
        m = b.scen["n_instances"].astype(np.int64)
        room = np.diff(b.ts_off) + m
        span_off = np.zeros(b.n + 1, dtype=np.int64)
        np.cumsum(room, out=span_off[1:])
        dev = self.device

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        d_m, d_cap, d_win, d_off = up(m.astype(np.int32)), up(cap), up(win), up(span_off)
        spans = torch.empty(int(span_off[-1]) * _abi.REGIME_SPAN_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        count = torch.empty(b.n, dtype=torch.int64, device=dev)
        frac = torch.empty(b.n, dtype=torch.float64, device=dev)
        status = torch.empty(b.n, dtype=torch.int32, device=dev)
        o = self.outputs
        with torch.cuda.device(dev):
            rc = _native.lib().asb_regime_classify(
                o["timeseries"].data_ptr(), o["ts_off"].data_ptr(), o["ts_count"].data_ptr(), b.n, d_m.data_ptr(),
                d_cap.data_ptr(), d_win.data_ptr(), d_off.data_ptr(), spans.data_ptr(), count.data_ptr(),
                frac.data_ptr(), status.data_ptr(), _native.stream_handle(dev))
        _native.check(rc, "asb_regime_classify")
        spans_h = spans.cpu().numpy().view(_abi.REGIME_SPAN_DTYPE)
        count_h, frac_h, status_h = count.cpu().numpy(), frac.cpu().numpy(), status.cpu().numpy()
        out = []
        for s in range(b.n):
            if status_h[s] > 0:
                raise SimulationError(f"usage series for instance {int(status_h[s])} does not cover the window start")
            if status_h[s] < 0:
                raise SimulationError("regime_classify: span buffer overflow")
            rows = spans_h[int(span_off[s]): int(span_off[s]) + int(count_h[s])]
            seg: dict = {i + 1: [] for i in range(int(m[s]))}
            for r in rows:
                seg[int(r["instance_id"])].append((float(r["start"]), float(r["end"]), bool(r["thrashing"])))
            out.append((seg, float(frac_h[s])))
        return out

    def download(self) -> tuple[dict, np.ndarray]:
        host = {}
        for k, t in self.outputs.items():
            host[k] = t.cpu().numpy()
        if host["decisions"].size:
            host["decisions"] = host["decisions"].view(_abi.DECISION_DTYPE)
        else:
            host.pop("decisions")
            host.pop("dec_off")
        if not host["turn_issue"].size and int(self.batch.turn_off[-1]):
            for k in ("turn_off", "turn_issue", "turn_done"):
                host.pop(k)
        if host["ts_count"].size:
            host["timeseries"] = host["timeseries"].view(_abi.TIMESERIES_DTYPE)
        else:
            for k in ("ts_off", "timeseries", "ts_count"):
                host.pop(k)
        stats = self.stats.cpu().numpy().view(_abi.STATS_DTYPE)
        return host, stats


def _none_if_nan(x: float):
    return None if x != x else float(x)


def check_status(host: Mapping, n: int) -> None:
    ctr = host["counters"].reshape(n, _abi.ASB_NCOUNTERS)
    bad = np.nonzero(ctr[:, _abi.CTR["status"]])[0]
    if bad.size:
        code = int(ctr[bad[0], _abi.CTR["status"]])
        raise SimulationError(f"scenario {int(bad[0])}: engine reported {_abi.SIMERR.get(code, code)}")


def build_results(batch: packing.Batch, host: Mapping, stats: np.ndarray, configs: Sequence[SimConfig],
                  echos: Sequence[dict | None], only: Sequence[int] | None = None,
                  checked: bool = False) -> list[SimulationResult]:
    """Rebuild the reference's SimulationResult objects from output arrays
    (every scenario, or the scenarios listed in ``only``)."""
    if not checked:
        check_status(host, batch.n)
    tp = batch.traces
    results = []
    ctr_all = host["counters"].reshape(batch.n, _abi.ASB_NCOUNTERS)
    for s in (range(len(configs)) if only is None else only):
        cfg = configs[s]
        rec = batch.scen[s]
        t = int(rec["trace_id"])
        a0, a1 = int(batch.agent_off[s]), int(batch.agent_off[s + 1])
        g0 = int(tp.trace_agent_off[t])
        ids = tp.agent_ids[t]
        rank = host["arrival_rank"][a0:a1]
        arrived = np.nonzero(rank >= 0)[0]
        order = arrived[np.argsort(rank[arrived], kind="stable")]
        turn_ok = "turn_issue" in host
        agents = []
        for a in order.tolist():
            o = a0 + a
            steps = int(host["turns_completed"][o])
            llm = float(host["llm_time"][o])
            dec = int(host["decode_total"][o])
            ct = float(host["completion_time"][o])
            ph = int(host["phase"][o])
            inst = int(host["final_instance"][o])
            n_turns = int(tp.agent_turn_off[g0 + a + 1] - tp.agent_turn_off[g0 + a])
            log = ()
            if turn_ok:
                base = int(batch.turn_off[s]) + int(tp.agent_turn_off[g0 + a] - tp.trace_turn_off[t])
                iss = host["turn_issue"][base: base + steps]
                don = host["turn_done"][base: base + steps]
                log = tuple((j, float(iss[j]), float(don[j])) for j in range(steps))
            agents.append(
                AgentResult(
                    agent_id=ids[a] if ids is not None else f"a{a:06d}",
                    arrival_time=float(tp.arrival[g0 + a]),
                    completion_time=None if ct != ct else ct,
                    completed=ph == 5,
                    turns_total=n_turns,
                    turns_completed=steps,
                    max_context_tokens=int(host["max_context"][o]),
                    total_llm_time=llm,
                    total_decode_tokens=dec,
                    throughput=dec / llm if llm > 0 else None,
                    final_instance=inst if inst > 0 else None,
                    migrations=int(host["migrations"][o]),
                    final_phase=_abi.PHASES[ph],
                    turn_log=log,
                )
            )
        m = int(rec["n_instances"])
        i0 = int(batch.inst_off[s])
        decisions = []
        if "decisions" in host:
            rows = host["decisions"][int(batch.dec_off[s]): int(batch.dec_off[s + 1])]
            decisions = [
                DecisionRow(float(r["time"]), int(r["instance_id"]), int(r["usage_observed"]),
                            int(r["frequency_level"]), bool(r["boosted"]), bool(r["deferred"]),
                            int(r["admitted_count"]), _none_if_nan(float(r["min_throughput"])),
                            int(r["pending_depth"]))
                for r in rows
            ]
        timeseries = []
        if "timeseries" in host:
            t0 = int(batch.ts_off[s])
            rows = host["timeseries"][t0: t0 + int(host["ts_count"][s])]
            table = cfg.instance.frequency_table
            timeseries = [
                TimeseriesRow(float(r["time"]), int(r["instance_id"]), int(r["context_usage"]),
                              int(r["level_index"]), float(table.level(int(r["level_index"])).nominal_mhz),
                              float(r["power_watts"]), int(r["pending_depth"]), int(r["running_requests"]),
                              int(r["thrashing"]))
                for r in rows
            ]
        st = stats[s]
        ctr = ctr_all[s]
        system = SystemMetrics(
            slo_attainment=_none_if_nan(float(st["slo_attainment"])),
            p5_throughput=_none_if_nan(float(st["p5_throughput"])),
            job_throughput=float(st["job_throughput"]),
            average_power=float(st["average_power"]),
            energy=float(st["energy"]),
            thrash_fraction=float(st["thrash_fraction"]),
        )
        echo = echos[s] if echos is not None and echos[s] is not None else config_echo(cfg)
        results.append(
            SimulationResult(
                sim_duration=cfg.sim_duration,
                instance_count=cfg.instance_count,
                capacity_tokens=cfg.instance.capacity_tokens,
                arrived=int(ctr[_abi.CTR["arrived"]]),
                completed=int(ctr[_abi.CTR["completed"]]),
                agents=agents,
                timeseries=timeseries,
                decisions=decisions,
                instance_energy={i + 1: float(host["energy"][i0 + i]) for i in range(m)},
                instance_thrash_time={i + 1: float(host["thrash_time"][i0 + i]) for i in range(m)},
                final_pending={i + 1: int(host["final_pending"][i0 + i]) for i in range(m)},
                final_usage={i + 1: int(host["final_usage"][i0 + i]) for i in range(m)},
                system=system,
                config_echo=echo,
                counters={k: int(ctr[v]) for k, v in _abi.CTR.items()},
            )
        )
    return results


class BatchResult(Sequence):
    """Columnar results of ``run_simulation_batch(..., columnar=True)``.

    The engine's output arrays as downloaded, without a Python object per
    agent: ``system`` (one SystemMetrics row per scenario: slo_attainment,
    p5_throughput, job_throughput, average_power, energy, thrash_fraction;
    NaN = None), ``counters`` (arrived, completed, agent-ticks, ... per
    scenario), ``agents(s)`` / ``instances(s)`` (numpy columns of scenario s,
    agents in arrival order like ``SimulationResult.agents``) and ``arrays``
    (every output array; agent rows of scenario s at
    ``batch.agent_off[s]:batch.agent_off[s+1]``).  Indexing builds scenario
    s's full ``SimulationResult`` (the reference's types) on first access.
    Device status words are checked at construction (SimulationError).
    """

    def __init__(self, batch: packing.Batch, host: Mapping, stats: np.ndarray, configs: Sequence[SimConfig],
                 echos: Sequence[dict | None] | None):
        check_status(host, batch.n)
        self.batch, self.arrays, self.system = batch, host, stats
        self.configs, self.echos = list(configs), echos
        self.counters = host["counters"].reshape(batch.n, _abi.ASB_NCOUNTERS)
        self._cache: dict[int, SimulationResult] = {}

    def __len__(self) -> int:
        return self.batch.n

    def __getitem__(self, s):
        if isinstance(s, slice):
            return [self[i] for i in range(*s.indices(len(self)))]
        s = range(len(self))[s]
        if s not in self._cache:
            (self._cache[s],) = build_results(self.batch, self.arrays, self.system, self.configs, self.echos,
                                              only=[s], checked=True)
        return self._cache[s]

    def counter(self, name: str) -> np.ndarray:
        return self.counters[:, _abi.CTR[name]]

    def agents(self, s: int) -> dict[str, np.ndarray]:
        """Per-agent columns of scenario s (arrived agents, arrival order)."""
        a0, a1 = int(self.batch.agent_off[s]), int(self.batch.agent_off[s + 1])
        rank = self.arrays["arrival_rank"][a0:a1]
        arrived = np.nonzero(rank >= 0)[0]
        order = arrived[np.argsort(rank[arrived], kind="stable")]
        t = int(self.batch.scen[s]["trace_id"])
        g0 = int(self.batch.traces.trace_agent_off[t])
        cols = {k: self.arrays[k][a0:a1][order] for k in _abi.AGENT_OUT}
        cols["arrival_time"] = self.batch.traces.arrival[g0 + order]
        llm, dec = cols["llm_time"], cols["decode_total"]
        with np.errstate(divide="ignore", invalid="ignore"):
            cols["throughput"] = np.where(llm > 0, dec / np.where(llm > 0, llm, 1.0), np.nan)
        cols["index"] = order
        return cols

    def instances(self, s: int) -> dict[str, np.ndarray]:
        i0, i1 = int(self.batch.inst_off[s]), int(self.batch.inst_off[s + 1])
        return {k: self.arrays[k][i0:i1] for k in _abi.INST_OUT}


def run_simulation_batch(configs: Sequence[SimConfig], config_echos: Sequence[dict | None] | None = None, *,
                         device=None, decisions: bool = True, turn_log: bool = True,
                         timeseries: bool = False, columnar: bool = False):
    """Run many independent simulations on one GPU; each result equals the
    reference's ``run_simulation`` of the same config (``timeseries`` rows
    only when asked for: those scenarios take the exact serial loop).

    ``columnar=True`` returns a ``BatchResult`` (numpy columns, per-scenario
    ``SimulationResult`` built lazily) instead of a list of results: at
    sweep scale the per-agent objects would cost far more than the run."""
    batch = prepare_batch(configs)
    dev_batch = DeviceBatch(batch, device=device, decisions=decisions, turn_log=turn_log, timeseries=timeseries)
    dev_batch.run()
    host, stats = dev_batch.download()
    if columnar:
        return BatchResult(batch, host, stats, configs, config_echos)
    return build_results(batch, host, stats, configs, config_echos)


def run_simulation(config: SimConfig, config_echo: dict | None = None, *, timeseries: bool = True) -> SimulationResult:
    """Run one simulation (engine.py:752-754) on the B200 engine, timeseries
    rows included like the reference's (``timeseries=False`` skips them and
    takes the optimistic-batch engine)."""
    return run_simulation_batch([config], [config_echo], timeseries=timeseries)[0]


def agent_ticks_closed_form(arrival: np.ndarray, completion: np.ndarray, epoch_length: float,
                            n_epochs: int) -> int:
    """Σ_a #{k : arrival_a < k·E ≤ completion_a (or not completed), k < K}
    (SURVEY §0): the agent-tick count implied by a result."""
    total = 0
    for arr, comp in zip(arrival.tolist(), completion.tolist()):
        k0 = math.floor(arr / epoch_length) + 1
        while k0 > 0 and (k0 - 1) * epoch_length > arr:
            k0 -= 1
        while k0 * epoch_length <= arr:
            k0 += 1
        k1 = n_epochs - 1
        if comp == comp:
            k1 = min(k1, math.floor(comp / epoch_length))
            while k1 >= 0 and k1 * epoch_length > comp:
                k1 -= 1
        total += max(0, k1 - k0 + 1)
    return total
