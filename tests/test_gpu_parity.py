"""GPU parity: the sm_100a engine through the C ABI against the reference's
golden vectors and the (pinned) oracle — bit-exact for every integer,
index and decision field, and (stricter than the 1e-5 contract) for the
floats too."""

import glob
import os
import random

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import (GOLDEN, array_outputs_equal, canonical, config_from_dict, digest, first_difference,
                    load_golden, traces_from_json, traces_to_json)
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import _abi, packing
from paper_2604_16682_b200.engine import DeviceBatch, build_results, prepare_batch
from paper_2604_16682_b200.workload import generate_arrays

pytestmark = pytest.mark.gpu

FULL = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "*.json.gz"))
              if not os.path.basename(p).startswith(("c3", "c4", "c5")))
DIGEST = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "c[345]*.json.gz"))
                if not os.path.basename(p).startswith("c4_full"))  # full C4: test_gpu_fullsize.py


def gpu(batch, decisions=True, turn_log=True):
    dev = DeviceBatch(batch, device="cuda:0", decisions=decisions, turn_log=turn_log)
    dev.run()
    return dev.download()


def test_golden_full_cases_in_one_batch(cuda_device):
    goldens = [load_golden(n) for n in FULL]
    cfgs = [config_from_dict(asb, g["config"], traces_from_json(asb, g["trace"])) for g in goldens]
    batch = prepare_batch(cfgs)
    host, stats = gpu(batch)
    results = build_results(batch, host, stats, cfgs, None)
    for g, r in zip(goldens, results):
        diff = first_difference(g["expected"], canonical(r))
        assert diff is None, (g["name"], diff)
        assert r.counters["ticks"] == g["ticks"], g["name"]


@pytest.mark.parametrize("name", DIGEST)
def test_golden_config_digests(cuda_device, name):
    g = load_golden(name)
    traces = asb.generate_workload(asb.WorkloadSpec(**g["spec"]))
    if digest(traces_to_json(traces)) != g["trace_digest"]:
        pytest.skip("numpy RNG stream differs from the golden trace's")
    cfg = config_from_dict(asb, g["config"], traces)
    batch = prepare_batch([cfg])
    host, stats = gpu(batch)
    (r,) = build_results(batch, host, stats, [cfg], None)
    can = canonical(r)
    bad = [k for k in g["digests"] if digest(can[k]) != g["digests"][k]]
    assert not bad, (bad, can["system"], g["summary"]["system"])
    assert r.counters["ticks"] == g["ticks"]


def _random_configs(seed, n):
    from test_host_engine import random_configs

    return random_configs(seed, n)


@pytest.fixture
def team(request, monkeypatch):
    """Force the engine's team shape (ASB_TEAM, read by asb_run_scenarios)."""
    if request.param:
        monkeypatch.setenv("ASB_TEAM", request.param)
    return request.param


@pytest.mark.parametrize("seed,team", [(11, None), (12, "quad"), (13, "big"), (14, "solo")], indirect=["team"])
def test_random_batch_matches_oracle(cuda_device, seed, team):
    """Random configurations on every team shape: solo warp (the default for
    these small scenarios), 4-warp quad team, 16-warp big team."""
    batch = prepare_batch(_random_configs(seed, 96))
    got, gst = gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(gst[f], wst[f], equal_nan=True), f


def c5_batch(seeds, cells=None):
    arrs = [generate_arrays(asb.WorkloadSpec(arrival_rate=10000 / 3600, duration=3600.0, seed=s)) for s in seeds]
    cfgs = []
    for pol in ("context_aware", "round_robin"):
        for var in ("context_aware", "off"):
            for tau in (20.0, 35.0):
                cfgs.append(asb.SimConfig(traces=[], instance_count=16, sim_duration=3600.0,
                                          controller=asb.ControllerConfig(variant=var, slo_target=tau),
                                          router=asb.RouterConfig(policy=pol)))
    cfgs = cfgs if cells is None else [cfgs[c] for c in cells]
    recs = [packing.scenario_record(c, t, 0) for t in range(len(seeds)) for c in cfgs]
    scen = np.array(recs, dtype=_abi.SCENARIO_DTYPE)
    return packing.build_batch(scen, packing.pack_traces(arrs), packing.pack_tables([asb.default_frequency_table()]))


def test_c5_full_size_scenarios_match_oracle(cuda_device):
    """Full-size C5 scenarios (16 instances x ~10k agents x 3600 epochs), all 8 cells."""
    batch = c5_batch([101, 102, 103, 104])
    got, gst = gpu(batch, decisions=True, turn_log=False)
    want, wst = run_oracle(batch, decisions=True, turn_log=False)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    ctr = got["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
    assert (ctr[:, _abi.CTR["ticks"]] > 5_000_000).all()


def test_c5_size_independent_properties(cuda_device):
    """Conservation laws at full size: final instance usage equals the summed
    context of the agents still resident on it; agent-ticks equal the closed
    form of SURVEY §0; completed agents consumed all their turns."""
    batch = c5_batch([7, 8], cells=[0, 3, 5, 6])
    host, _ = gpu(batch, decisions=False, turn_log=False)
    ctr = host["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
    tp = batch.traces
    for s in range(batch.n):
        a0, a1 = batch.agent_off[s], batch.agent_off[s + 1]
        t = int(batch.scen[s]["trace_id"])
        g0 = tp.trace_agent_off[t]
        phase = host["phase"][a0:a1]
        inst = host["final_instance"][a0:a1]
        ctx = host["context"][a0:a1]
        resident = np.isin(phase, [2, 3, 4])
        m = int(batch.scen[s]["n_instances"])
        usage = np.bincount(inst[resident], weights=ctx[resident], minlength=m + 1)[1:]
        assert np.array_equal(usage.astype(np.int64), host["final_usage"][batch.inst_off[s]: batch.inst_off[s + 1]])
        n_turns = tp.agent_turn_off[g0 + 1: g0 + (a1 - a0) + 1] - tp.agent_turn_off[g0: g0 + (a1 - a0)]
        done = phase == 5
        assert np.array_equal(host["turns_completed"][a0:a1][done], n_turns[done])
        arr = tp.arrival[g0: g0 + (a1 - a0)]
        comp = host["completion_time"][a0:a1]
        arrived = host["arrival_rank"][a0:a1] >= 0
        want = asb.engine.agent_ticks_closed_form(arr[arrived], comp[arrived], 1.0, int(batch.scen[s]["n_epochs"]))
        assert ctr[s, _abi.CTR["ticks"]] == want


@pytest.mark.parametrize("team", [None, "quad", "big"], indirect=True)
def test_wide_scenarios_64_instance_team(cuda_device, team):
    """Scenarios with 17..64 instances on the MAXM=64 kernels: the solo warp
    (default for these sizes) and the multi-warp teams, whose walk runs the
    snapshots / checks / routing of more than 32 instances as a team job."""
    import random as _random

    rng = _random.Random(5)
    cfgs = []
    for k in range(24):
        spec = asb.WorkloadSpec(arrival_rate=rng.choice([0.5, 2.0]), duration=120.0, seed=100 + k)
        d = {
            "instances": rng.choice([17, 32, 64]),
            "capacity": rng.choice([3000, 20_000, 100_000]),
            "duration": 200.0,
            "controller": {"variant": rng.choice(["context_aware", "off"]), "thrash_avoidance": rng.random() < 0.5},
            "router": {"policy": rng.choice(["context_aware", "round_robin", "least_loaded"]),
                       "reassign_interval": rng.choice([1, 3, 8]), "migration_delay": rng.choice([0.0, 2.0])},
        }
        cfgs.append(config_from_dict(asb, d, asb.generate_workload(spec)))
    batch = prepare_batch(cfgs)
    assert batch.max_instances > 16
    got, gst = gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(gst[f], wst[f], equal_nan=True), f


def test_run_sharded_single_rank(cuda_device):
    """parallel.run_sharded on one rank: the LPT shard is everything, the
    gathered per-scenario rows and the stats vector match the oracle."""
    from paper_2604_16682_b200.parallel import run_sharded

    cfgs = _random_configs(21, 12)
    res = run_sharded(cfgs, device="cuda:0", results=True)
    assert res.world == 1 and list(res.local_index) == list(range(len(cfgs)))
    batch = prepare_batch(cfgs)
    want, wst = run_oracle(batch, decisions=False, turn_log=False)
    ctr = want["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
    assert np.array_equal(res.counters[:, :9], ctr[:, :9])
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(res.stats[f], wst[f], equal_nan=True), f
    assert res.totals["ticks"] == float(ctr[:, _abi.CTR["ticks"]].sum())
    assert res.totals["completed"] == float(ctr[:, _abi.CTR["completed"]].sum())
    assert len(res.local_results) == len(cfgs)


@pytest.mark.parametrize("team", ["big", "quad"], indirect=True)
def test_large_tie_storm_batches(cuda_device, team):
    """Hundreds of identical agents: batches of several hundred records with
    exact (time, priority) ties ordered by push sequence, past the 256th
    record of the big team's 1,024-record buffer."""
    base = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.5, duration=20.0, seed=5))[0]
    cfgs = []
    for n, inst, pol in ((600, 4, "round_robin"), (400, 2, "context_aware"), (700, 8, "least_loaded")):
        traces = [asb.AgentTrace(f"r{i:04d}", base.arrival_time, base.turns[:12]) for i in range(n)]
        cfgs.append(config_from_dict(asb, {"instances": inst, "capacity": 2_000_000, "duration": 300.0,
                                           "router": {"policy": pol, "reassign_interval": 3}}, traces))
    batch = prepare_batch(cfgs)
    got, gst = gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff


def _with_instances(cfgs, m):
    import dataclasses

    return [dataclasses.replace(c, instance_count=m) for c in cfgs]


@pytest.mark.parametrize("seed", [21, 22])
def test_single_instance_kernel_matches_oracle(cuda_device, seed):
    """Every scenario single-instance: the batch runs the kernel whose
    instance count is the compile-time 1 (asb_run_scenarios(-1)), across all
    controller variants, interference, thrash avoidance and tie storms."""
    batch = prepare_batch(_with_instances(_random_configs(seed, 96), 1))
    assert batch.launch_instances == -1
    got, gst = gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(gst[f], wst[f], equal_nan=True), f


@pytest.mark.parametrize("seed,team", [(23, "quad"), (24, "solo"), (25, "big")], indirect=["team"])
def test_fixed_count_kernel_matches_oracle(cuda_device, seed, team, monkeypatch):
    """Every scenario with 16 instances: the quad team runs the kernel whose
    instance count is the compile-time 16; the result equals the oracle and
    the run-time-count kernel's (ASB_NO_FIXED_M) bit for bit."""
    batch = prepare_batch(_with_instances(_random_configs(seed, 48), 16))
    assert batch.launch_instances == -16
    got, gst = gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    monkeypatch.setenv("ASB_NO_FIXED_M", "1")
    got2, _ = gpu(batch)
    assert array_outputs_equal(got, got2) is None


def test_mixed_instance_counts_take_the_general_kernel(cuda_device):
    """A batch mixing instance counts passes the maximum (not -m) and matches
    the oracle."""
    cfgs = _with_instances(_random_configs(26, 16), 16) + _with_instances(_random_configs(27, 16), 3)
    batch = prepare_batch(cfgs)
    assert batch.launch_instances == 16
    got, _ = gpu(batch)
    want, _ = run_oracle(batch)
    assert array_outputs_equal(want, got) is None
