"""Timeseries rows (``_mark_row``, engine.py:403-429; ``_on_sample``,
engine.py:570-572): the oracle against golden series produced by the
reference itself (tests/golden/make_golden_timeseries.py), the engine core's
serial loop against the oracle on CPU (host build), and the sm_100a engine
against both (``-m gpu``).  Exact equality, floats included."""

import glob
import gzip
import json
import os

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from common import (GOLDEN, array_outputs_equal, canonical, canonical_timeseries, config_from_dict, digest,
                    first_difference, load_golden, results_via, traces_from_json)
from oracle.oracle import run_host_engine, run_oracle
from paper_2604_16682_b200 import packing
from paper_2604_16682_b200.engine import prepare_batch

TS_DIR = os.path.join(GOLDEN, "timeseries")
TS = sorted(os.path.basename(p) for p in glob.glob(os.path.join(TS_DIR, "*.json.gz")))


def load_ts(name):
    with gzip.open(os.path.join(TS_DIR, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


def ts_config(name):
    t = load_ts(name)
    g = load_golden(name)
    return t, g, config_from_dict(asb, t["config"], traces_from_json(asb, g["trace"]))


def check_rows(t, rows):
    assert len(rows) == t["n_rows"]
    if "rows" in t:
        diff = first_difference(t["rows"], rows)
        assert diff is None, diff
    else:
        diff = first_difference(t["head"], rows[: len(t["head"])])
        assert diff is None, diff
        assert digest(rows) == t["digest"]


def test_fixtures_present():
    assert len(TS) >= 30


@pytest.mark.parametrize("name", TS)
def test_oracle_timeseries_matches_reference(name):
    t, g, cfg = ts_config(name)
    (res,), _ = results_via(run_oracle, [cfg], timeseries=True)
    check_rows(t, canonical_timeseries(res))


@pytest.mark.parametrize("name", [n for n in TS if n.startswith(("ka_", "tie_", "tool_", "rand_0"))])
def test_host_engine_serial_loop_matches_reference(name):
    """The engine core's serial loop (the GPU's timeseries mode), CPU build."""
    t, g, cfg = ts_config(name)
    (res,), _ = results_via(run_host_engine, [cfg], timeseries=True)
    check_rows(t, canonical_timeseries(res))
    if "expected" in g:  # the serial loop's other results equal the batched engine's golden ones
        diff = first_difference(g["expected"], canonical(res))
        assert diff is None, diff


def test_samples_change_no_other_result():
    """Sample events only emit rows (engine.py:570-572): every other output is
    identical with and without the series."""
    cfgs = [ts_config(n)[2] for n in ("rand_03.json.gz", "tie_storm_ctx.json.gz", "ka_migration_delay.json.gz")]
    batch = prepare_batch(cfgs)
    a, _ = run_oracle(batch, timeseries=True)
    b, _ = run_oracle(batch)
    assert array_outputs_equal(b, a, keys=[k for k in b if k not in ("agent_off", "inst_off", "dec_off",
                                                                      "turn_off")]) is None


def test_capacity_bounds_the_rows():
    cfgs = [ts_config(n)[2] for n in TS if n.startswith(("rand_", "tie_"))]
    batch = prepare_batch(cfgs)
    host, _ = run_oracle(batch, timeseries=True)
    cap = np.diff(batch.ts_off)
    assert (host["ts_count"] <= cap).all()
    assert (host["ts_count"] > 0).all()


def test_sample_count_matches_the_reference_loop():
    for dur, iv in ((10.0, 1.0), (10.5, 1.0), (0.3, 1.0), (1.0, 0.1), (3600.0, 0.7), (100.0, 2.5), (333.3, 0.7)):
        k, n = 1, 0
        while k * iv < dur:
            n += 1
            k += 1
        assert packing.sample_count(dur, iv) == n, (dur, iv)


def test_series_helpers():
    """power_series / usage_series / integrate_power over the rows
    (engine.py:164-205): the integral of the power series is the energy."""
    t, g, cfg = ts_config("rand_01.json.gz")
    (res,), _ = results_via(run_oracle, [cfg], timeseries=True)
    ps = res.power_series()
    assert sorted(ps) == list(range(1, cfg.instance_count + 1))
    assert all(p[0][0] == 0.0 for p in ps.values())
    avg = asb.integrate_power(ps, cfg.sim_duration)
    assert avg == pytest.approx(sum(res.instance_energy.values()) / cfg.sim_duration, rel=1e-9)
    us = res.usage_series()
    assert all(u[-1][1] == float(res.final_usage[i]) for i, u in us.items())


# --------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", TS)
def test_gpu_run_simulation_timeseries_matches_reference(cuda_device, name):
    """``run_simulation`` (timeseries on by default, like the reference)."""
    t, g, cfg = ts_config(name)
    res = asb.run_simulation(cfg)
    check_rows(t, canonical_timeseries(res))
    if "expected" in g:
        diff = first_difference(g["expected"], canonical(res))
        assert diff is None, diff


@pytest.fixture
def team(request, monkeypatch):
    if request.param:
        monkeypatch.setenv("ASB_TEAM", request.param)
    return request.param


@pytest.mark.gpu
@pytest.mark.parametrize("seed,team", [(21, None), (22, "quad"), (23, "big")], indirect=["team"])
def test_gpu_timeseries_batch_matches_oracle(cuda_device, seed, team):
    """A batch of random scenarios in timeseries mode on every team shape:
    every output array, rows included, equals the oracle's."""
    from test_host_engine import random_configs

    from paper_2604_16682_b200.engine import DeviceBatch

    batch = prepare_batch(random_configs(seed, 24))
    dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=True, timeseries=True)
    dev.run()
    got, _ = dev.download()
    want, _ = run_oracle(batch, timeseries=True)
    assert np.array_equal(got["ts_count"], want["ts_count"])
    for s in range(batch.n):
        o, n = int(batch.ts_off[s]), int(want["ts_count"][s])
        assert got["timeseries"][o: o + n].tobytes() == want["timeseries"][o: o + n].tobytes(), s
    diff = array_outputs_equal(want, got, keys=[k for k in want if k not in (
        "agent_off", "inst_off", "dec_off", "turn_off", "ts_off", "timeseries")])
    assert diff is None, diff


@pytest.mark.gpu
def test_gpu_rows_without_offsets_are_rejected(cuda_device):
    """asb_run_scenarios returns ASB_ERR_ARG for a row buffer without its
    offsets / counts (include/agentsim_b200.h), raised by the host mirror."""
    import torch

    from paper_2604_16682_b200 import ops
    from paper_2604_16682_b200.engine import DeviceBatch

    t, g, cfg = ts_config("ka_single_agent.json.gz")
    dev = DeviceBatch(prepare_batch([cfg]), device="cuda:0", timeseries=True)
    dev.outputs["ts_off"] = torch.empty(0, dtype=torch.int64, device="cuda:0")
    dev.out_list = [dev.outputs[k] for k in ops.OUT_NAMES]
    with pytest.raises(RuntimeError):
        dev.run()
