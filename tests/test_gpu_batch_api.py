"""run_simulation_batch's columnar mode (BatchResult) against its object
mode on the GPU, and the WorkloadSpec fast path of prepare_batch (the
reference's generate_workload draws straight into CSR arrays)."""

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import canonical
from paper_2604_16682_b200.engine import BatchResult, prepare_batch


def _configs():
    cfgs = []
    for k, (pol, var) in enumerate([("context_aware", "context_aware"), ("round_robin", "off"),
                                    ("least_loaded", "fixed")]):
        ctl = asb.ControllerConfig(variant=var, fixed_level_mhz=900.0 if var == "fixed" else None)
        cfgs.append(asb.SimConfig(workload=asb.WorkloadSpec(arrival_rate=0.4, duration=150.0, seed=k),
                                  instance_count=3, sim_duration=220.0, controller=ctl,
                                  router=asb.RouterConfig(policy=pol),
                                  instance=asb.InstanceConfig(capacity_tokens=40_000)))
    return cfgs


def test_spec_fast_path_packs_like_generated_objects():
    cfgs = _configs()
    objs = [asb.SimConfig(traces=asb.generate_workload(c.workload), instance_count=c.instance_count,
                          sim_duration=c.sim_duration, controller=c.controller, router=c.router,
                          instance=c.instance) for c in cfgs]
    b1, b2 = prepare_batch(cfgs), prepare_batch(objs)
    assert b1.scen.tobytes() == b2.scen.tobytes()
    for k in ("arrival", "agent_turn_off", "prefill", "decode", "tool", "arrival_order"):
        assert np.array_equal(getattr(b1.traces, k), getattr(b2.traces, k)), k
    assert b1.traces.agent_ids[0] is None and b2.traces.agent_ids[0][0] == "a000000"


@pytest.mark.gpu
def test_columnar_results_match_objects(cuda_device):
    cfgs = _configs()
    objs = asb.run_simulation_batch(cfgs)
    col = asb.run_simulation_batch(cfgs, columnar=True)
    assert isinstance(col, BatchResult) and len(col) == len(cfgs)
    for s, r in enumerate(objs):
        assert canonical(col[s]) == canonical(r)
        a = col.agents(s)
        assert a["turns_completed"].tolist() == [x.turns_completed for x in r.agents]
        assert a["arrival_time"].tolist() == [x.arrival_time for x in r.agents]
        tp = [np.nan if x.throughput is None else x.throughput for x in r.agents]
        assert np.array_equal(a["throughput"], np.array(tp), equal_nan=True)
        assert col.counter("completed")[s] == r.completed
        sysm = col.system[s]
        assert float(sysm["energy"]) == r.system.energy
        assert col.instances(s)["final_usage"].tolist() == [r.final_usage[i + 1] for i in range(3)]
