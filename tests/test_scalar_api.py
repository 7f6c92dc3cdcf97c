"""The per-call API mirror (controller / instance / router helpers) is host
arithmetic; it must agree with the reference's own functions exactly
(controller.py:81-109, instance.py:184-204, router.py:75-151)."""

import random
import sys

import pytest

import paper_2604_16682_b200 as asb
from common import reference_module


def test_scalar_api_mirror_known_answers():
    assert asb.select_frequency_level(37_500, 100_000, 7, 0.75) == 4
    assert asb.select_frequency_level(75_000, 100_000, 7, 0.75) == 7
    assert asb.select_frequency_level(0.5, 1.0, 4, 0.75) == 3  # float inputs are not truncated
    lvl = asb.FrequencyLevel(1000.0, 10000.0, 1000.0, 300.0, 50.0)
    cfg = asb.InstanceConfig(thrash_latency_factor=3.0)
    assert asb.service_time(asb.TurnRecord(1000, 100, 0.0), lvl, 0, 1, True, cfg) == pytest.approx(0.6, rel=1e-12)
    state = asb.RouterState(instance_ids=[1, 2, 3, 4])
    agent = asb.AgentRuntimeState("a")
    assert asb.assign_agent(agent, {1: 60_000, 2: 10_000, 3: 0, 4: 0}, 100_000, asb.RouterConfig(), state) == 2
    agent = asb.AgentRuntimeState("b", instance_id=1, steps_since_assignment=7)
    assert asb.maybe_reassign(agent, {1: 80_000, 2: 30_000}, asb.RouterConfig(), asb.RouterState([1, 2])) == 2
    a = asb.AgentRuntimeState("c", decode_tokens_total=300, llm_time_total=15.0)
    assert asb.running_throughput(a) == 20.0
    assert asb.running_throughput(asb.AgentRuntimeState("d")) is None
    assert asb.slo_boost_check([a, asb.AgentRuntimeState("e", decode_tokens_total=50, llm_time_total=10.0)], 20.0)
    with pytest.raises(asb.ConfigurationError):
        asb.service_time(asb.TurnRecord(1, 1, 0.0), asb.FrequencyLevel(1.0, 0.0, 1.0, 1.0, 1.0), 0, 1, False, cfg)


ref = reference_module()


@pytest.mark.skipif(ref is None, reason="reference not present (GPU box)")
def test_scalar_api_matches_reference_on_random_grids():
    rng = random.Random(11)
    for _ in range(5000):
        u, c = rng.uniform(0, 3.0) * rng.choice([1, 1e5]), rng.uniform(0.01, 2.0) * rng.choice([1, 1e5])
        L, al = rng.randint(1, 16), rng.choice([0.3, 0.5, 0.75, 1.0])
        assert asb.select_frequency_level(u, c, L, al) == ref.select_frequency_level(u, c, L, al)
    for _ in range(2000):
        m = rng.randint(1, 9)
        ids = sorted(rng.sample(range(1, 40), m))
        us = {i: rng.choice([0, 0, rng.randint(0, 10**6), rng.uniform(0, 1e6)]) for i in ids}
        rc = dict(consolidation_threshold=rng.choice([0.2, 0.5, 0.9]), reassign_interval=rng.randint(1, 4),
                  imbalance_ratio=rng.choice([1.01, 2.0, 4.0]), include_idle_instances=rng.random() < 0.5,
                  reset_counter_only_on_reassign=rng.random() < 0.5)
        cap = rng.choice([10_000, 500_000])
        got = asb.assign_agent(asb.AgentRuntimeState("x"), us, cap, asb.RouterConfig(**rc), asb.RouterState(ids))
        want = ref.assign_agent(ref.AgentRuntimeState("x"), us, cap, ref.RouterConfig(**rc), ref.RouterState(ids))
        assert got == want
        got = asb.route_least_loaded(asb.AgentRuntimeState("x"), us, asb.RouterState(ids))
        assert got == ref.route_least_loaded(ref.AgentRuntimeState("x"), us, ref.RouterState(ids))
        cur, sa = rng.choice(ids), rng.randint(0, 5)
        a1 = asb.AgentRuntimeState("y", instance_id=cur, steps_since_assignment=sa)
        a2 = ref.AgentRuntimeState("y", instance_id=cur, steps_since_assignment=sa)
        assert asb.maybe_reassign(a1, us, asb.RouterConfig(**rc), asb.RouterState(ids)) == ref.maybe_reassign(
            a2, us, ref.RouterConfig(**rc), ref.RouterState(ids))
        assert a1.steps_since_assignment == a2.steps_since_assignment
    lv_args = (1185.0, 15000.0, 60.0, 300.0, 50.0)
    for _ in range(2000):
        p, d = rng.randint(1, 32768), rng.randint(1, 8192)
        n, th = rng.randint(0, 12), rng.random() < 0.5
        ic, tf = rng.choice([0.0, 0.1, 0.37]), rng.choice([1.0, 3.0, 2.5])
        got = asb.service_time(asb.TurnRecord(p, d, 0.0), asb.FrequencyLevel(*lv_args), 0, n, th,
                               asb.InstanceConfig(interference_coeff=ic, thrash_latency_factor=tf))
        want = ref.service_time(ref.TurnRecord(p, d, 0.0), ref.FrequencyLevel(*lv_args), 0, n, th,
                                ref.InstanceConfig(interference_coeff=ic, thrash_latency_factor=tf))
        assert got == want
    agents = [(rng.randint(0, 10**6), rng.choice([0.0, rng.uniform(0, 100)])) for _ in range(200)]
    got = asb.min_throughput([asb.AgentRuntimeState(str(i), decode_tokens_total=d, llm_time_total=t)
                              for i, (d, t) in enumerate(agents)])
    want = sys.modules["agentsim.controller"].min_throughput([ref.AgentRuntimeState(str(i), decode_tokens_total=d, llm_time_total=t)
                               for i, (d, t) in enumerate(agents)])
    assert got == want
