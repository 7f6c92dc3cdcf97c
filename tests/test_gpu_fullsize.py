"""Full-size BASELINE configurations on the GPU:

* C4 — the 100k-agent thrashing regime (seed 11, 99,955 agents, 3.39 M
  turns, 64 instances, context-aware without thrash avoidance), run with
  thrash_mode "recompute" and "offload": every result field against the
  digests the REFERENCE itself produced (tests/golden/make_golden_c4.py),
  the config echo included, and every output array against the oracle;
* C3 — the whole 2,048-scenario DVFS sweep (64 seeds x 8 fixed levels x 4
  capacities, 1 instance x ~1k agents, 12,500 epochs) against the oracle,
  bit-exact, on the same workload bench.py times.
"""

import os
import sys

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import array_outputs_equal, canonical, config_from_dict, digest, load_golden, traces_to_json
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import _abi
from paper_2604_16682_b200.engine import DeviceBatch, build_results, prepare_batch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c4_traces():
    g = load_golden("c4_full_recompute.json.gz")
    traces = asb.generate_workload(asb.WorkloadSpec(**g["spec"]))
    if digest(traces_to_json(traces)) != g["trace_digest"]:
        pytest.skip("numpy RNG stream differs from the golden trace's")
    return traces


@pytest.mark.parametrize("mode", ["recompute", "offload"])
def test_c4_full_matches_reference_and_oracle(cuda_device, c4_traces, mode):
    g = load_golden(f"c4_full_{mode}.json.gz")
    cfg = config_from_dict(asb, g["config"], c4_traces)
    assert cfg.instance.thrash_mode == mode
    batch = prepare_batch([cfg])
    dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=True)
    dev.run()
    host, stats = dev.download()
    # the oracle on the same packed batch: every output array, bit-exact
    want, wstats = run_oracle(batch, decisions=True, turn_log=True)
    diff = array_outputs_equal(want, host)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(stats[f], wstats[f], equal_nan=True), f
    # the reference's own results (digests of every canonical field)
    (r,) = build_results(batch, host, stats, [cfg], None)
    can = canonical(r)
    bad = [k for k in g["digests"] if digest(can[k]) != g["digests"][k]]
    assert not bad, (bad, can["system"], g["summary"]["system"])
    assert r.counters["ticks"] == g["ticks"]
    assert len(r.decisions) == g["summary"]["n_decisions"]
    assert digest(r.config_echo) == g["echo_digest"]
    assert r.config_echo["instance"]["thrash_mode"] == mode


def test_c3_full_sweep_matches_oracle(cuda_device):
    """All 2,048 C3 scenarios in one launch (the single-warp teams, 14 per SM)."""
    sys.path.insert(0, ROOT)
    import bench

    batch, seeds = bench.build_shard(0, None, "c3")
    assert batch.n == 2048 and len(seeds) == 64
    dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=False)
    dev.run()
    got, gst = dev.download()
    want, wst = run_oracle(batch, decisions=True, turn_log=False, threads=len(os.sched_getaffinity(0)))
    diff = array_outputs_equal(want, got)
    assert diff is None, diff
    for f in _abi.STATS_DTYPE.names:
        assert np.array_equal(gst[f], wst[f], equal_nan=True), f
    ctr = got["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
    assert ctr[:, _abi.CTR["ticks"]].sum() > 4_000_000_000
