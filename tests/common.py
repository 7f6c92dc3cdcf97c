"""Shared test helpers: scenario factories, canonical result form, comparisons.

Configs are described by plain dicts so the same case can be instantiated
with the reference's classes (``agentsim``, only importable in the build
container) or with this package's mirror, and stored in golden fixtures.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"

import paper_2604_16682_b200 as asb  # noqa: E402
from paper_2604_16682_b200 import _abi  # noqa: E402
from paper_2604_16682_b200.engine import build_results, prepare_batch  # noqa: E402


REF_INSTALLED = os.path.join(ROOT, "baseline", "_ref")  # pip install --target of the reference (travels)


def reference_module(installed: bool = False):
    """The reference package: the read-only tree in the build container, or
    (``installed=True``) its pip install under baseline/_ref, which also
    exists on the GPU box when it was installed; None when absent."""
    path = REF_SRC if os.path.isdir(REF_SRC) else None
    if path is None and installed and os.path.isdir(os.path.join(REF_INSTALLED, "agentsim")):
        path = REF_INSTALLED
    if path is None:
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import agentsim  # noqa: F401

    return sys.modules["agentsim"]


# --------------------------------------------------------------------------- case description


def traces_to_json(traces) -> list:
    return [[t.agent_id, t.arrival_time, [[r.prefill_tokens, r.decode_tokens, r.tool_time] for r in t.turns]]
            for t in traces]


def traces_from_json(mod, rows) -> list:
    return [mod.AgentTrace(a, float(arr), tuple(mod.TurnRecord(int(p), int(d), float(tt)) for p, d, tt in turns))
            for a, arr, turns in rows]


def config_from_dict(mod, d: dict, traces):
    table = mod.default_frequency_table(**({"mhz": tuple(d["mhz"])} if d.get("mhz") else {}))
    inst = mod.InstanceConfig(
        capacity_tokens=d.get("capacity", 500_000),
        frequency_table=table,
        thrash_mode=d.get("thrash_mode", "recompute"),
        thrash_latency_factor=d.get("thrash_factor", 3.0),
        interference_coeff=d.get("interference", 0.0),
    )
    ctl = mod.ControllerConfig(**d.get("controller", {}))
    rt = mod.RouterConfig(**d.get("router", {}))
    return mod.SimConfig(
        traces=traces,
        instance_count=d.get("instances", 1),
        instance=inst,
        controller=ctl,
        router=rt,
        sim_duration=d.get("duration", 3600.0),
        record_interval=d.get("record_interval", 1.0),
    )


def spec_from_dict(mod, d: dict):
    kw = dict(d)
    return mod.WorkloadSpec(**kw)


# --------------------------------------------------------------------------- canonical results


def _f(x):
    return None if x is None else float(x)


def canonical(result) -> dict:
    """Result fields the parity contract covers, in a comparable form."""
    return {
        "arrived": result.arrived,
        "completed": result.completed,
        "agents": [
            [a.agent_id, _f(a.arrival_time), _f(a.completion_time), bool(a.completed), a.turns_total,
             a.turns_completed, a.max_context_tokens, _f(a.total_llm_time), a.total_decode_tokens,
             _f(a.throughput), a.final_instance, a.migrations, a.final_phase,
             [[i, _f(s), _f(e)] for i, s, e in a.turn_log]]
            for a in result.agents
        ],
        "decisions": [
            [_f(d.time), d.instance_id, d.usage_observed, d.frequency_level, bool(d.boosted), bool(d.deferred),
             d.admitted_count, _f(d.min_throughput), d.pending_depth]
            for d in result.decisions
        ],
        "instance_energy": {str(k): _f(v) for k, v in sorted(result.instance_energy.items())},
        "instance_thrash_time": {str(k): _f(v) for k, v in sorted(result.instance_thrash_time.items())},
        "final_pending": {str(k): v for k, v in sorted(result.final_pending.items())},
        "final_usage": {str(k): v for k, v in sorted(result.final_usage.items())},
        "system": [_f(result.system.slo_attainment), _f(result.system.p5_throughput),
                   _f(result.system.job_throughput), _f(result.system.average_power), _f(result.system.energy),
                   _f(result.system.thrash_fraction)],
    }


def canonical_timeseries(result) -> list:
    """SimulationResult.timeseries (engine.py:91-101) in a comparable form."""
    return [[_f(r.time), r.instance_id, r.context_usage, r.level_index, _f(r.level_mhz), _f(r.power_watts),
             r.pending_depth, r.running_requests, int(r.thrashing)] for r in result.timeseries]


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True, allow_nan=True).encode()).hexdigest()


def first_difference(a, b, path="") -> str | None:
    """Human-readable location of the first difference (exact compare)."""
    if type(a) is not type(b) and not (isinstance(a, (int, float)) and isinstance(b, (int, float))):
        return f"{path}: type {type(a).__name__} != {type(b).__name__} ({a!r} vs {b!r})"
    if isinstance(a, dict):
        if set(a) != set(b):
            return f"{path}: keys differ"
        for k in sorted(a):
            d = first_difference(a[k], b[k], f"{path}.{k}")
            if d:
                return d
        return None
    if isinstance(a, list):
        if len(a) != len(b):
            return f"{path}: length {len(a)} != {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            d = first_difference(x, y, f"{path}[{i}]")
            if d:
                return d
        return None
    if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
        return None
    if a != b:
        return f"{path}: {a!r} != {b!r}"
    return None


def close_difference(a, b, rel=1e-5, path="") -> str | None:
    """Like first_difference but floats within `rel` relative tolerance."""
    if isinstance(a, float) and isinstance(b, float):
        if math.isnan(a) and math.isnan(b):
            return None
        if a == b or abs(a - b) <= rel * max(abs(a), abs(b)):
            return None
        return f"{path}: {a!r} !~ {b!r}"
    if isinstance(a, dict):
        if set(a) != set(b):
            return f"{path}: keys differ"
        for k in sorted(a):
            d = close_difference(a[k], b[k], rel, f"{path}.{k}")
            if d:
                return d
        return None
    if isinstance(a, list):
        if len(a) != len(b):
            return f"{path}: length {len(a)} != {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            d = close_difference(x, y, rel, f"{path}[{i}]")
            if d:
                return d
        return None
    if a != b:
        return f"{path}: {a!r} != {b!r}"
    return None


# --------------------------------------------------------------------------- runners over a batch


def results_via(runner, configs, decisions=True, turn_log=True, timeseries=False):
    """Run configs through a host runner (oracle / host engine) and rebuild results."""
    batch = prepare_batch(configs)
    host, stats = runner(batch, timeseries=True) if timeseries else runner(batch)
    return build_results(batch, host, stats, configs, None), host


def array_outputs_equal(h1: dict, h2: dict, keys=None) -> str | None:
    keys = keys or [k for k in h1 if k in h2 and k not in ("agent_off", "inst_off", "dec_off", "turn_off")]
    for k in keys:
        a, b = h1[k], h2[k]
        if k == "counters":
            a = a.reshape(-1, _abi.ASB_NCOUNTERS).copy()
            b = b.reshape(-1, _abi.ASB_NCOUNTERS).copy()
            a[:, _abi.CTR["batches"]] = 0
            b[:, _abi.CTR["batches"]] = 0
        if a.dtype.names:
            for f in a.dtype.names:
                if not np.array_equal(a[f], b[f], equal_nan=np.issubdtype(a[f].dtype, np.floating)):
                    idx = np.nonzero(~((a[f] == b[f]) | (np.isnan(a[f]) & np.isnan(b[f])) if np.issubdtype(a[f].dtype, np.floating) else (a[f] != b[f])))[0]
                    return f"{k}.{f} differs at {idx[:5].tolist()}"
            continue
        eq = np.array_equal(a, b, equal_nan=np.issubdtype(a.dtype, np.floating))
        if not eq:
            if np.issubdtype(a.dtype, np.floating):
                bad = np.nonzero(~((a == b) | (np.isnan(a) & np.isnan(b))))[0]
            else:
                bad = np.nonzero(a != b)[0]
            return f"{k} differs at {bad[:5].tolist()} ({a[bad[:3]].tolist()} vs {b[bad[:3]].tolist()})"
    return None


def load_golden(name: str) -> dict:
    path = os.path.join(GOLDEN, name)
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return json.load(fh)
