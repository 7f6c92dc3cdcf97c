"""The drop-in adapter (paper_2604_16682_b200/adapter.py): the reference's
own SimConfig / AgentTrace objects in, the reference's own SimulationResult
out.  CPU: the conversion and packing against the mirror, and the full
round trip with the oracle as the engine stand-in, compared field by field
(``==`` on the reference's dataclasses, floats exact) with
``agentsim.run_simulation``.  GPU: ``adapter.run_simulation`` itself."""

import dataclasses

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import config_from_dict, reference_module, results_via
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import adapter
from paper_2604_16682_b200.engine import prepare_batch

CASES = [
    ({"instances": 3, "capacity": 20_000, "router": {"reassign_interval": 2, "migration_delay": 2.0},
      "duration": 300.0}, dict(arrival_rate=0.3, duration=200.0, seed=4)),
    ({"instances": 2, "controller": {"variant": "fixed", "fixed_level_mhz": 810.0},
      "router": {"policy": "round_robin"}, "interference": 0.1, "thrash_mode": "offload", "duration": 250.0},
     dict(arrival_rate=0.2, duration=200.0, seed=9, prefill_growth_per_turn=20.0)),
    ({"instances": 4, "controller": {"variant": "off", "epoch_length": 0.7}, "router": {"policy": "least_loaded"},
      "mhz": [660, 900, 1185, 1680], "duration": 200.0}, dict(arrival_rate=0.5, duration=100.0, seed=2)),
]


def _ref():
    ref = reference_module(installed=True)
    if ref is None:
        pytest.skip("the reference is not importable here")
    return ref


@pytest.mark.parametrize("d,spec", CASES)
def test_from_reference_packs_like_the_mirror(d, spec):
    ref = _ref()
    ref_cfg = config_from_dict(ref, d, ref.generate_workload(ref.WorkloadSpec(**spec)))
    mine = config_from_dict(asb, d, asb.generate_workload(asb.WorkloadSpec(**spec)))
    conv = adapter.from_reference(ref_cfg)
    assert isinstance(conv, asb.SimConfig) and conv.traces is ref_cfg.traces
    assert conv.instance == mine.instance and conv.controller == mine.controller and conv.router == mine.router
    b1, b2 = prepare_batch([conv]), prepare_batch([mine])
    assert b1.scen.tobytes() == b2.scen.tobytes()
    for k in ("arrival", "agent_turn_off", "prefill", "decode", "tool", "arrival_order"):
        assert np.array_equal(getattr(b1.traces, k), getattr(b2.traces, k)), k


def test_workload_spec_configs_convert():
    """A SimConfig carrying a WorkloadSpec (the reference CLI's `run` path)."""
    ref = _ref()
    spec = ref.WorkloadSpec(arrival_rate=0.2, duration=100.0, seed=3,
                            tool_time=ref.Distribution("exponential", 1.5, minimum=0.0))
    ref_cfg = ref.SimConfig(workload=spec, instance_count=2, sim_duration=150.0, seed=8)
    conv = adapter.from_reference(ref_cfg)
    assert conv.workload == asb.WorkloadSpec(arrival_rate=0.2, duration=100.0, seed=3,
                                             tool_time=asb.Distribution("exponential", 1.5, minimum=0.0))
    assert conv.seed == 8 and conv.instance_count == 2


@pytest.mark.parametrize("d,spec", CASES)
def test_round_trip_equals_reference_run_simulation(d, spec):
    """reference objects -> adapter -> packed batch -> engine stand-in (the
    oracle on CPU) -> the reference's SimulationResult, equal (==) to
    agentsim.run_simulation's, timeseries and echo included."""
    ref = _ref()
    ref_cfg = config_from_dict(ref, d, ref.generate_workload(ref.WorkloadSpec(**spec)))
    want = ref.run_simulation(ref_cfg)
    (mine,), _ = results_via(run_oracle, [adapter.from_reference(ref_cfg)], timeseries=True)
    got = adapter.to_reference(mine, ref)
    assert type(got) is ref.SimulationResult and type(got.system) is ref.SystemMetrics
    assert type(got.agents[0]) is ref.AgentResult and type(got.decisions[0]) is ref.DecisionRow
    for f in dataclasses.fields(ref.SimulationResult):
        assert getattr(got, f.name) == getattr(want, f.name), f.name
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("d,spec", CASES)
def test_gpu_adapter_run_simulation(cuda_device, d, spec):
    """The drop-in itself on the B200: adapter.run_simulation(reference
    config) == agentsim.run_simulation(reference config).  (On the GPU box the
    reference comes from its pip install in baseline/_ref.)"""
    ref = _ref()
    ref_cfg = config_from_dict(ref, d, ref.generate_workload(ref.WorkloadSpec(**spec)))
    want = ref.run_simulation(ref_cfg)
    got = adapter.run_simulation(ref_cfg)
    assert type(got) is ref.SimulationResult
    assert got == want
    (got2,) = adapter.run_simulation_batch([ref_cfg])  # batched path, no timeseries rows
    assert got2.agents == want.agents and got2.decisions == want.decisions and got2.system == want.system
