"""GPU edge cases through the C ABI against the pinned oracle: an empty
batch, ragged batches (zero-agent, one-agent and ~10k-agent scenarios side by
side on every team shape), the frequency-table extremes (two levels, sixteen
levels) and scenarios whose instance count differs from the batch maximum."""

import dataclasses

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import array_outputs_equal
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import _abi
from paper_2604_16682_b200.engine import DeviceBatch, prepare_batch

pytestmark = pytest.mark.gpu


def _gpu(batch):
    dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=True)
    dev.run()
    return dev.download()


def _check(batch):
    got, gst = _gpu(batch)
    want, wst = run_oracle(batch)
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(gst[f], wst[f], equal_nan=True), f
    return got


def test_empty_batch(cuda_device):
    assert asb.run_simulation_batch([]) == []
    res = asb.run_simulation_batch([], columnar=True)
    assert len(res) == 0


def _ragged_configs():
    big = asb.generate_workload(asb.WorkloadSpec(arrival_rate=10000 / 3600, duration=600.0, seed=5))
    one = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.05, duration=40.0, seed=6))[:1]
    mid = asb.generate_workload(asb.WorkloadSpec(arrival_rate=1.0, duration=120.0, seed=7))
    cfgs = []
    for traces, m in ((big, 16), ([], 4), (one, 1), (mid, 8), (big, 3), (one, 16)):
        cfgs.append(asb.SimConfig(traces=traces, instance_count=m, sim_duration=650.0,
                                  instance=asb.InstanceConfig(capacity_tokens=400_000)))
    return cfgs


@pytest.mark.parametrize("team", [None, "quad", "big", "solo"])
def test_ragged_batch_every_team(cuda_device, team, monkeypatch):
    """Scenario sizes from 0 to ~1.7k agents and 1 to 16 instances in one
    launch, on every team shape."""
    if team:
        monkeypatch.setenv("ASB_TEAM", team)
    batch = prepare_batch(_ragged_configs())
    assert batch.launch_instances == 16  # mixed counts: the run-time-count kernels
    got = _check(batch)
    ctr = got["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
    assert ctr[1, _abi.CTR["ticks"]] == 0  # the zero-agent scenario
    assert ctr[0, _abi.CTR["ticks"]] > 100_000


@pytest.mark.parametrize("mhz", [(660.0, 1680.0), tuple(660.0 + 68.0 * k for k in range(16))])
def test_frequency_table_extremes(cuda_device, mhz):
    """The two-level minimum a FrequencyTable validates (instance.py) and the
    sixteen-level maximum, under the context-aware controller with boost."""
    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.5, duration=300.0, seed=9))
    table = asb.default_frequency_table(mhz=mhz)
    base = asb.SimConfig(traces=traces, instance_count=4, sim_duration=400.0,
                         instance=asb.InstanceConfig(frequency_table=table, capacity_tokens=30_000),
                         controller=asb.ControllerConfig(variant="context_aware", slo_target=35.0))
    cfgs = [base, dataclasses.replace(base, instance_count=1),
            dataclasses.replace(base, controller=asb.ControllerConfig(variant="off"))]
    _check(prepare_batch(cfgs))


def test_single_config_batches_take_the_fixed_kernels(cuda_device):
    """run_simulation_batch of one config (a fixed-count launch) equals the
    same config inside a mixed batch (a run-time-count launch)."""
    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=2.0, duration=200.0, seed=3))
    a = asb.SimConfig(traces=traces, instance_count=16, sim_duration=250.0)
    b = dataclasses.replace(a, instance_count=5)
    alone = prepare_batch([a])
    assert alone.launch_instances == -16
    got_alone, _ = _gpu(alone)
    mixed = prepare_batch([a, b])
    got_mixed, _ = _gpu(mixed)
    n0 = int(alone.agent_off[1])
    for k in ("completion_time", "llm_time", "turns_completed", "final_instance", "migrations"):
        assert np.array_equal(got_alone[k][:n0], got_mixed[k][:n0], equal_nan=got_alone[k].dtype.kind == "f"), k
    assert np.array_equal(got_alone["counters"][:_abi.ASB_NCOUNTERS], got_mixed["counters"][:_abi.ASB_NCOUNTERS])


def _wide_configs(seed):
    """Up to 127 instances and up to 64 DVFS levels (the wide kernel), with
    every controller variant and router policy."""
    import random

    rng = random.Random(seed)
    out = []
    for m, n_lv in ((100, 24), (127, 8), (70, 64), (3, 40)):
        traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=rng.choice([2.0, 5.0]), duration=150.0,
                                                        seed=rng.randrange(10_000)))
        table = asb.default_frequency_table(mhz=tuple(600.0 + 20.0 * k for k in range(n_lv)))
        var = rng.choice(["context_aware", "off", "fixed"])
        ctl = asb.ControllerConfig(variant=var, slo_target=rng.choice([20.0, 50.0]),
                                   fixed_level_mhz=table.levels[n_lv // 2].nominal_mhz if var == "fixed" else None)
        out.append(asb.SimConfig(traces=traces, instance_count=m, sim_duration=200.0,
                                 instance=asb.InstanceConfig(frequency_table=table,
                                                             capacity_tokens=rng.choice([3000, 30_000])),
                                 controller=ctl,
                                 router=asb.RouterConfig(policy=rng.choice(["context_aware", "round_robin",
                                                                            "least_loaded"]),
                                                         reassign_interval=rng.choice([1, 3]))))
    return out


@pytest.mark.parametrize("seed", [31, 32])
def test_wide_kernel_matches_oracle(cuda_device, seed):
    """More than 64 instances / more than 16 levels: the 128-instance,
    64-level kernel, bit-exact against the oracle, rows included."""
    batch = prepare_batch(_wide_configs(seed))
    assert batch.max_levels > 16 and batch.max_instances > 64
    _check(batch)
    dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=True, timeseries=True)
    dev.run()
    got, _ = dev.download()
    want, _ = run_oracle(batch, timeseries=True)
    assert np.array_equal(got["ts_count"], want["ts_count"])
    for s in range(batch.n):
        o, n = int(batch.ts_off[s]), int(want["ts_count"][s])
        assert got["timeseries"][o: o + n].tobytes() == want["timeseries"][o: o + n].tobytes(), s
