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
