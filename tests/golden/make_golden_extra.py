"""Round-2 golden fixtures, generated from the REFERENCE itself (build
container only; the fixtures travel, the reference does not).

    python tests/golden/make_golden_extra.py

* ``ka_migration_storm``: a migration-heavy case (2 instances, a
  reassignment check at every turn, idle instances as candidates, imbalance
  ratio 1.0001, migration delay 1 s) whose series has more rows than the
  round-1 bound of 3 per turn: every tool event that migrates marks two
  instances (engine.py:560-561) and is followed by a delayed start (568).  Full trace, full expected result, and its timeseries
  (tests/golden/timeseries/ka_migration_storm.json.gz, record interval 1.0).
* ``c4_full_recompute`` / ``c4_full_offload``: the full-size C4 thrashing
  regime of SURVEY §8d (seed 11, 99,955 agents / 3.39 M turns, 64 instances,
  context-aware control with thrash_avoidance=False), once per thrash_mode.
  The two modes are numerically identical in the reference (instance.py:121,
  201-203); only the config echo differs (engine.py:689), so the fixture
  also stores the reference's ``_config_echo`` for each.
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import (canonical, canonical_timeseries, config_from_dict, digest, reference_module,  # noqa: E402
                    traces_to_json)
from make_golden import save, ticks_closed_form  # noqa: E402

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"
import numpy as np  # noqa: E402

META = {"numpy": np.__version__, "python": sys.version.split()[0]}


def migration_storm():
    # six agents of 24 short turns, all consolidated on instance 1; with idle
    # instances as candidates every tool event migrates (ping-pong), so a
    # turn produces four rows: completion, source + target, delayed start
    traces = [ref.AgentTrace(f"m{i:02d}", 0.1 * i, tuple(ref.TurnRecord(200 + 10 * i, 20, 0.05) for _ in range(24)))
              for i in range(6)]
    d = {"instances": 2, "capacity": 500_000, "thrash_factor": 1.0, "controller": {"variant": "off"},
         "router": {"reassign_interval": 1, "imbalance_ratio": 1.0001, "migration_delay": 1.0,
                    "include_idle_instances": True},
         "duration": 45.0}
    cfg = config_from_dict(ref, d, traces)
    r = ref.run_simulation(cfg)
    name = "ka_migration_storm"
    payload = {"name": name, "config": d, "trace": traces_to_json(traces), "meta": META,
               "ticks": ticks_closed_form(r, 1.0, d["duration"]), "expected": canonical(r)}
    save(name, payload)
    rows = canonical_timeseries(r)
    path = os.path.join(HERE, "timeseries", name + ".json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump({"name": name + ".json.gz", "config": d, "n_rows": len(rows), "digest": digest(rows),
                   "rows": rows}, fh, separators=(",", ":"), allow_nan=True)
    n_turns = sum(len(t.turns) for t in traces)
    mig = sum(a.migrations for a in r.agents)
    print(f"{name}: {len(traces)} agents, {n_turns} turns, {mig} migrations, {len(rows)} rows", flush=True)


def c4_full():
    spec = dict(arrival_rate=100000 / 3600, duration=3600.0, seed=11, prefill_growth_per_turn=20.0)
    t0 = time.time()
    traces = ref.generate_workload(ref.WorkloadSpec(**spec))
    print(f"c4 trace: {len(traces)} agents in {time.time() - t0:.1f}s", flush=True)
    for mode in ("recompute", "offload"):
        d = {"instances": 64, "thrash_mode": mode, "controller": {"thrash_avoidance": False}, "duration": 3600.0}
        cfg = config_from_dict(ref, d, traces)
        t0 = time.time()
        r = ref.run_simulation(cfg)
        wall = time.time() - t0
        can = canonical(r)
        name = f"c4_full_{mode}"
        payload = {
            "name": name, "config": d, "spec": spec, "meta": META, "ref_wall_s": wall,
            "trace_digest": digest(traces_to_json(traces)),
            "ticks": ticks_closed_form(r, 1.0, d["duration"]),
            "summary": {"arrived": r.arrived, "completed": r.completed, "system": can["system"],
                        "n_agents": len(traces), "n_turns": sum(len(t.turns) for t in traces)},
            "digests": {k: digest(v) for k, v in can.items()},
            "config_echo": sys.modules["agentsim.engine"]._config_echo(cfg),
        }
        save(name, payload)
        print(f"{name}: {wall:.1f}s, ticks {payload['ticks']}, system {can['system']}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["storm", "c4"]
    if "storm" in which:
        migration_storm()
    if "c4" in which:
        c4_full()
