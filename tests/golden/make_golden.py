"""Generate the golden fixtures from the REFERENCE itself (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

    python tests/golden/make_golden.py

Each fixture: the case description (config dict + either the full trace or
the WorkloadSpec that regenerates it), and the reference's results in the
canonical form of tests/common.py: full for small cases, SHA-256 digests
(plus a few summary fields) for the large ones.  Agent-tick counts are the
closed form of SURVEY §0, computed from the reference's own result.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import canonical, config_from_dict, digest, reference_module, traces_to_json  # noqa: E402

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"
import numpy as np  # noqa: E402


def ticks_closed_form(result, epoch_length: float, sim_duration: float) -> int:
    k_max = 0
    while k_max * epoch_length < sim_duration:
        k_max += 1
    total = 0
    for a in result.agents:
        k0 = 0
        while not (a.arrival_time < k0 * epoch_length):
            k0 += 1
        k1 = k_max - 1
        if a.completion_time is not None:
            while k1 >= 0 and not (k1 * epoch_length <= a.completion_time):
                k1 -= 1
        total += max(0, k1 - k0 + 1)
    return total


def tr(aid, arr, turns):
    return ref.AgentTrace(aid, arr, tuple(ref.TurnRecord(*t) for t in turns))


def known_answer_cases():
    """The hand-walked scenarios of the reference's test_engine.py."""
    yield "ka_single_agent", {"controller": {"variant": "off"}, "duration": 10.0}, [tr("a1", 0.5, [(1000, 100, 0.0)])]
    yield "ka_zero_agents_1", {"duration": 120.0}, []
    yield "ka_zero_agents_3", {"duration": 120.0, "instances": 3}, []
    yield "ka_boost_retime", {"controller": {"slo_target": 50.0}, "duration": 135.0}, [
        tr("A", 0.2, [(2000, 200, 200.0), (1, 1, 0.0)]),
        tr("B", 0.3, [(100, 10000, 0.0)]),
    ]
    yield "ka_migration_delay", {
        "instances": 2, "capacity": 1000, "thrash_factor": 1.0, "controller": {"variant": "off"},
        "router": {"reassign_interval": 2, "migration_delay": 5.0}, "duration": 12.0,
    }, [tr("X", 0.1, [(1000, 80, 1.0)] * 8), tr("Y", 2.5, [(100, 80, 1.0)] * 8)]
    yield "ka_closed_form", {"controller": {"variant": "off"}, "duration": 60.0}, [
        tr("x", 0.0, [(100, 50, 0.5), (25, 25, 0.5), (10, 5, 0.0)])
    ]
    # tie storms: identical agents admitted together
    base = ref.generate_workload(ref.WorkloadSpec(arrival_rate=0.5, duration=20.0, seed=5))[0]
    yield "tie_storm_rr", {"instances": 4, "router": {"policy": "round_robin"}, "duration": 400.0}, [
        ref.AgentTrace(f"r{i:02d}", base.arrival_time, base.turns) for i in range(48)
    ]
    yield "tie_storm_ctx", {
        "instances": 4, "capacity": 60000,
        "router": {"reassign_interval": 2, "include_idle_instances": True}, "duration": 400.0,
    }, [ref.AgentTrace(f"r{i:02d}", base.arrival_time, base.turns[:18]) for i in range(64)]
    yield "tool_zero", {"instances": 2, "duration": 200.0}, [
        tr(f"z{i}", 0.25 * i, [(300 + i, 40, 0.0)] * 6) for i in range(12)
    ]


def rand_case(rng):
    spec = dict(arrival_rate=rng.choice([0.05, 0.2, 0.5, 2.0]), duration=rng.choice([50.0, 200.0, 400.0]),
                seed=rng.randrange(1000))
    if rng.random() < 0.2:
        spec["arrival_process"] = "fixed_interval"
    if rng.random() < 0.2:
        spec["prefill_growth_per_turn"] = 20.0
    d = {
        "instances": rng.choice([1, 2, 3, 4, 8]),
        "capacity": rng.choice([2000, 10000, 50000, 200000, 500000]),
        "duration": rng.choice([100.0, 300.0, 500.0, 333.3]),
        "thrash_factor": rng.choice([1.0, 3.0]),
        "interference": rng.choice([0.0, 0.0, 0.0, 0.1]),
        "controller": {"variant": rng.choice(["context_aware", "off", "fixed"]),
                       "slo_target": rng.choice([20.0, 35.0, 50.0]), "boost_enabled": rng.random() < 0.8,
                       "thrash_avoidance": rng.random() < 0.7, "epoch_length": rng.choice([1.0, 1.0, 2.0, 0.7])},
        "router": {"policy": rng.choice(["context_aware", "round_robin", "least_loaded"]),
                   "reassign_interval": rng.choice([1, 2, 8]), "migration_delay": rng.choice([0.0, 0.0, 5.0]),
                   "include_idle_instances": rng.random() < 0.3,
                   "reset_counter_only_on_reassign": rng.random() < 0.3},
    }
    if d["controller"]["variant"] == "fixed":
        d["controller"]["fixed_level_mhz"] = rng.choice([660.0, 810.0, 1680.0])
    return spec, d


C3_MHZ = [660, 810, 900, 1035, 1185, 1350, 1515, 1680]


def config_cases():
    """BASELINE configurations, full size."""
    yield "c1", dict(arrival_rate=64 / 600, arrival_process="fixed_interval", duration=600.0, seed=1), {
        "controller": {"variant": "fixed", "fixed_level_mhz": 810.0}, "duration": 3600.0}
    yield "c2", dict(arrival_rate=1000 / 3600, duration=3600.0, seed=1), {"instances": 8, "duration": 3600.0}
    yield "c3_s0_660_250k", dict(arrival_rate=0.08, duration=12500.0, seed=0), {
        "mhz": C3_MHZ, "capacity": 250_000, "controller": {"variant": "fixed", "fixed_level_mhz": 660.0},
        "duration": 12500.0}
    yield "c3_s5_1185_1m", dict(arrival_rate=0.08, duration=12500.0, seed=5), {
        "mhz": C3_MHZ, "capacity": 1_000_000, "controller": {"variant": "fixed", "fixed_level_mhz": 1185.0},
        "duration": 12500.0}
    yield "c4_trim5k", dict(arrival_rate=5000 / 3600, duration=3600.0, seed=11, prefill_growth_per_turn=20.0), {
        "instances": 64, "capacity": 25_000, "controller": {"thrash_avoidance": False}, "duration": 3600.0}
    yield "c5_s7_ca_ca_20", dict(arrival_rate=10000 / 3600, duration=3600.0, seed=7), {
        "instances": 16, "duration": 3600.0}
    yield "c5_s7_rr_off_35", dict(arrival_rate=10000 / 3600, duration=3600.0, seed=7), {
        "instances": 16, "duration": 3600.0, "router": {"policy": "round_robin"},
        "controller": {"variant": "off", "slo_target": 35.0}}


def save(name, payload):
    path = os.path.join(HERE, name + ".json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(payload, fh, separators=(",", ":"), allow_nan=True)
    return os.path.getsize(path)


def main():
    meta = {"numpy": np.__version__, "python": sys.version.split()[0]}
    index = []
    for name, d, traces in known_answer_cases():
        r = ref.run_simulation(config_from_dict(ref, d, traces))
        e = d.get("controller", {}).get("epoch_length", 1.0)
        payload = {"name": name, "config": d, "trace": traces_to_json(traces), "meta": meta,
                   "ticks": ticks_closed_form(r, e, d.get("duration", 3600.0)), "expected": canonical(r)}
        index.append((name, save(name, payload)))
    rng = random.Random(20261017)
    for i in range(24):
        spec, d = rand_case(rng)
        traces = ref.generate_workload(ref.WorkloadSpec(**spec))
        r = ref.run_simulation(config_from_dict(ref, d, traces))
        e = d["controller"].get("epoch_length", 1.0)
        name = f"rand_{i:02d}"
        payload = {"name": name, "config": d, "trace": traces_to_json(traces), "meta": meta,
                   "ticks": ticks_closed_form(r, e, d["duration"]), "expected": canonical(r)}
        index.append((name, save(name, payload)))
    for name, spec, d in config_cases():
        traces = ref.generate_workload(ref.WorkloadSpec(**spec))
        t0 = time.time()
        r = ref.run_simulation(config_from_dict(ref, d, traces))
        wall = time.time() - t0
        can = canonical(r)
        full = name in ("c1", "c2")
        payload = {
            "name": name, "config": d, "spec": spec, "meta": meta, "ref_wall_s": wall,
            "trace_digest": digest(traces_to_json(traces)),
            "ticks": ticks_closed_form(r, 1.0, d["duration"]),
            "summary": {"arrived": r.arrived, "completed": r.completed, "system": can["system"],
                        "n_agents": len(traces), "n_turns": sum(len(t.turns) for t in traces)},
            "digests": {k: digest(v) for k, v in can.items()},
        }
        if full:
            payload["trace"] = traces_to_json(traces)
            payload["expected"] = can
        index.append((name, save(name, payload)))
        print(name, f"{wall:.1f}s", flush=True)
    for name, size in index:
        print(f"{name:24s} {size/1024:8.1f} KiB")


if __name__ == "__main__":
    main()
