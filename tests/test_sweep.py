"""Batched sweep driver (paper_2604_16682_b200/sweep.py) against the
reference's own ``agentsim sweep`` CLI: the ``sweep.csv`` it wrote
(tests/golden/make_golden_sweep.py → tests/golden/sweep/) is reproduced
byte for byte — with the oracle as the runner on CPU, and with the one-launch
GPU batch under ``-m gpu``."""

import glob
import json
import os

import pytest

import paper_2604_16682_b200 as asb
from common import GOLDEN, results_via
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import sweep

SWEEP_DIR = os.path.join(GOLDEN, "sweep")
CASES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(SWEEP_DIR, "*.json")))
AXIS_FLAGS = {"--axis-level-mhz": ("level_mhz", float), "--axis-rate": ("arrival_rate", float),
              "--axis-slo": ("slo_target", float), "--axis-policy": ("policy", str)}


def load_case(name):
    with open(os.path.join(SWEEP_DIR, name + ".json")) as fh:
        return json.load(fh)


def base_config(doc):
    """The experiment YAML's sections (config.py:1-45) as a SimConfig."""
    w, i, r, s = doc.get("workload", {}), doc.get("instance", {}), doc.get("router", {}), doc.get("sim", {})
    return asb.SimConfig(
        workload=asb.WorkloadSpec(arrival_rate=w["arrival_rate"], duration=float(w["duration"]), seed=w["seed"]),
        instance_count=i.get("count", 1),
        instance=asb.InstanceConfig(capacity_tokens=i.get("capacity_tokens", 500_000),
                                    interference_coeff=i.get("interference_coeff", 0.0)),
        router=asb.RouterConfig(**{k: v for k, v in r.items()}),
        sim_duration=float(s.get("duration", 3600.0)),
    )


def axes_of(case):
    """CLI axis flags override the YAML's sweep section (cli.py:136-158)."""
    axes = {k: v for k, v in case["experiment"].get("sweep", {}).items() if v}
    flag, vals = None, []
    for tok in case["axes"] + ["--end"]:
        if tok.startswith("--"):
            if flag:
                name, conv = AXIS_FLAGS[flag]
                axes[name] = [conv(v) for v in vals]
            flag, vals = (tok if tok != "--end" else None), []
        else:
            vals.append(tok)
    return axes


def oracle_runner(cfgs):
    return results_via(run_oracle, cfgs, decisions=False, turn_log=False)[0]


def test_fixtures_present():
    assert len(CASES) >= 3


@pytest.mark.parametrize("name", CASES)
def test_sweep_csv_matches_reference_cli(tmp_path, name):
    case = load_case(name)
    outcomes = sweep.run_cells(base_config(case["experiment"]), sweep.sweep_cells(axes_of(case)),
                               runner=oracle_runner)
    path = tmp_path / "sweep.csv"
    assert sweep.write_sweep_table(str(path), outcomes) == 0
    assert path.read_text(encoding="utf-8") == case["sweep_csv"]


def test_cells_order_and_errors():
    cells = sweep.sweep_cells({"policy": ["round-robin"], "level_mhz": [660.0, 810.0]})
    assert cells == [{"level_mhz": 660.0, "policy": "round-robin"}, {"level_mhz": 810.0, "policy": "round-robin"}]
    with pytest.raises(asb.ConfigurationError):
        sweep.sweep_cells({})
    with pytest.raises(asb.ConfigurationError):
        sweep.sweep_cells({"slo_target": []})
    with pytest.raises(asb.ConfigurationError):
        sweep.sweep_cells({"bogus": [1]})


def test_failing_cell_is_recorded_and_the_sweep_continues(tmp_path):
    base = base_config(load_case(CASES[0])["experiment"])
    cells = sweep.sweep_cells({"level_mhz": [660.0, 700.0], "slo_target": [-1.0, 20.0]})
    outcomes = sweep.run_cells(base, cells, runner=oracle_runner)
    ok = [c for c, s, e in outcomes if s is not None]
    bad = [c for c, s, e in outcomes if s is None]
    assert ok == [{"level_mhz": 660.0, "slo_target": 20.0}]
    assert len(bad) == 3 and all(e for _, s, e in outcomes if s is None)
    path = tmp_path / "sweep.csv"
    assert sweep.write_sweep_table(str(path), outcomes) == 3
    rows = path.read_text().splitlines()
    assert rows[1].endswith(",nan,nan,nan,nan,nan,nan,nan,nan,error," + outcomes[0][2].replace(",", ";"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_sweep_csv_matches_reference_cli(cuda_device, tmp_path, name):
    """All cells of the sweep in one engine launch."""
    case = load_case(name)
    outcomes = sweep.run_cells(base_config(case["experiment"]), sweep.sweep_cells(axes_of(case)))
    path = tmp_path / "sweep.csv"
    assert sweep.write_sweep_table(str(path), outcomes) == 0
    assert path.read_text(encoding="utf-8") == case["sweep_csv"]


def test_extra_axes_express_the_baseline_sweeps(tmp_path):
    """seed / capacity / variant axes (beyond the reference's four): a
    C3-shaped sweep (level x capacity x seed) through run_cells equals the
    configs built by hand, and sweep.csv gets the extra columns last."""
    table = asb.default_frequency_table(mhz=(660, 810, 900, 1035, 1185, 1350, 1515, 1680))
    base = asb.SimConfig(workload=asb.WorkloadSpec(arrival_rate=0.1, duration=150.0, seed=0), sim_duration=200.0,
                         instance=asb.InstanceConfig(frequency_table=table))
    cells = sweep.sweep_cells({"seed": [3, 4], "level_mhz": [660.0, 1185.0], "capacity": [20_000, 60_000]})
    assert len(cells) == 8 and list(cells[0]) == ["level_mhz", "capacity", "seed"]
    assert [c["seed"] for c in cells[:2]] == [3, 4]  # the last axis varies fastest
    cfgs = [sweep.apply_cell(base, c) for c in cells]
    assert cfgs[1].seed == 4 and cfgs[2].instance.capacity_tokens == 60_000
    assert cfgs[0].controller.variant == "fixed" and cfgs[0].controller.fixed_level_mhz == 660.0
    outcomes = sweep.run_cells(base, cells, runner=oracle_runner)
    by_hand = [asb.SimConfig(workload=asb.WorkloadSpec(arrival_rate=0.1, duration=150.0, seed=c["seed"]),
                             sim_duration=200.0,
                             instance=asb.InstanceConfig(capacity_tokens=c["capacity"], frequency_table=table),
                             controller=asb.ControllerConfig(variant="fixed", fixed_level_mhz=c["level_mhz"]))
               for c in cells]
    for (cell, summary, err), r in zip(outcomes, oracle_runner(by_hand)):
        assert err is None and summary["energy"] == r.system.energy and summary["completed"] == r.completed
    sweep.write_sweep_table(str(tmp_path / "sweep.csv"), outcomes)
    header = (tmp_path / "sweep.csv").read_text().splitlines()[0].split(",")
    assert header[:2] == ["level_mhz", "capacity"] and header[2] == "seed"
    v = sweep.sweep_cells({"variant": ["off", "context-aware"], "policy": ["round-robin"]})
    assert sweep.apply_cell(base, v[1]).controller.variant == "context_aware"
    with pytest.raises(asb.ConfigurationError, match="unknown axis"):
        sweep.sweep_cells({"seeds": [1]})
