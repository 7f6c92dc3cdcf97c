"""The GPU engine's batching logic (engine_core.h) compiled as a 1-lane CPU
harness, differential-tested against the oracle on CPU: optimistic epoch
batches, tie resolution, coupling points, and — with deliberately tiny
buffers — the horizon / window-bisection / serial-step overflow paths."""

import random

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import array_outputs_equal, config_from_dict, load_golden, traces_from_json
from oracle.oracle import run_host_engine, run_oracle
from paper_2604_16682_b200.engine import prepare_batch

CASES = ["ka_single_agent", "ka_boost_retime", "ka_migration_delay", "tie_storm_rr", "tie_storm_ctx", "tool_zero",
         "rand_00", "rand_03", "rand_07", "rand_11", "rand_16", "rand_21", "c1"]


def golden_batch(names):
    cfgs = []
    for n in names:
        g = load_golden(n + ".json.gz")
        cfgs.append(config_from_dict(asb, g["config"], traces_from_json(asb, g["trace"])))
    return prepare_batch(cfgs)


@pytest.mark.parametrize("small", [False, True])
def test_host_engine_matches_oracle_on_golden(small):
    batch = golden_batch(CASES)
    want, _ = run_oracle(batch)
    got, _ = run_host_engine(batch, small_buffers=small)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff


def random_configs(seed, n):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        spec = asb.WorkloadSpec(arrival_rate=rng.choice([0.1, 0.5, 2.0]), duration=rng.choice([60.0, 200.0]),
                                seed=rng.randrange(10_000))
        traces = asb.generate_workload(spec)
        if traces and rng.random() < 0.25:
            base = traces[0]
            traces = [asb.AgentTrace(f"t{i}", base.arrival_time, base.turns) for i in range(rng.choice([8, 40]))]
        d = {
            "instances": rng.choice([1, 2, 4, 8]),
            "capacity": rng.choice([3000, 20_000, 100_000, 500_000]),
            "duration": rng.choice([150.0, 300.0, 301.5]),
            "interference": rng.choice([0.0, 0.0, 0.05]),
            "controller": {"variant": rng.choice(["context_aware", "off", "fixed"]),
                           "slo_target": rng.choice([20.0, 50.0]), "thrash_avoidance": rng.random() < 0.6,
                           "epoch_length": rng.choice([1.0, 2.5])},
            "router": {"policy": rng.choice(["context_aware", "round_robin", "least_loaded"]),
                       "reassign_interval": rng.choice([1, 3, 8]), "migration_delay": rng.choice([0.0, 2.0]),
                       "include_idle_instances": rng.random() < 0.3,
                       "reset_counter_only_on_reassign": rng.random() < 0.3},
        }
        if d["controller"]["variant"] == "fixed":
            d["controller"]["fixed_level_mhz"] = 810.0
        out.append(config_from_dict(asb, d, traces))
    return out


@pytest.mark.parametrize("seed", [1, 2])
def test_host_engine_matches_oracle_random(seed):
    batch = prepare_batch(random_configs(seed, 24))
    want, _ = run_oracle(batch)
    for small in (False, True):
        got, _ = run_host_engine(batch, small_buffers=small)
        diff = array_outputs_equal(want, got)
        assert diff is None, (small, diff)


def test_host_engine_c5_scenario():
    from paper_2604_16682_b200 import packing, _abi
    from paper_2604_16682_b200.workload import generate_arrays

    arr = generate_arrays(asb.WorkloadSpec(arrival_rate=10000 / 3600, duration=3600.0, seed=3))
    cfg = asb.SimConfig(traces=[], instance_count=16, sim_duration=3600.0)
    scen = np.array([packing.scenario_record(cfg, 0, 0)], dtype=_abi.SCENARIO_DTYPE)
    batch = packing.build_batch(scen, packing.pack_traces([arr]), packing.pack_tables([asb.default_frequency_table()]))
    want, _ = run_oracle(batch, decisions=False)
    got, _ = run_host_engine(batch, decisions=False)
    assert array_outputs_equal(want, got) is None


@pytest.mark.parametrize("small", [False, True])
def test_host_engine_serial_due_windows(small):
    """The single-warp teams' small-window serial loop (serial_due: the exact
    event loop over the window's due list, batches when the list outgrows
    the buffer) against the oracle, on the goldens and random configs."""
    for batch in (golden_batch(CASES), prepare_batch(random_configs(3, 24))):
        want, _ = run_oracle(batch)
        got, _ = run_host_engine(batch, small_buffers=small, serial_due=True)
        diff = array_outputs_equal(want, got)
        assert diff is None, (small, diff)
