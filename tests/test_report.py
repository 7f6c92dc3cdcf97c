"""export_report byte identity: the report directory this
package writes for a B200 result equals, byte for byte, the one the
reference's own CLI wrote (`agentsim run --config cfg.yaml --out dir`,
cli.py:121-135; the reference's check is test_cli.py:109-116).  Fixtures:
tests/golden/make_golden_report.py.  The YAML front end is the reference's
(ExperimentConfig, config.py), reached through the drop-in adapter; the
reference is imported from the build container's tree or from its pip
install in baseline/_ref (on the GPU box)."""

import os

import pytest

from common import GOLDEN, reference_module, results_via
from oracle.oracle import run_oracle
from paper_2604_16682_b200 import adapter, export_report, run_simulation

REPORT = os.path.join(GOLDEN, "report")
CASES = sorted(os.listdir(REPORT)) if os.path.isdir(REPORT) else []
FILES = ("summary.csv", "agents.csv", "timeseries.csv", "decisions.csv", "config.yaml")


def _experiment(name):
    ref = reference_module(installed=True)
    if ref is None:
        pytest.skip("the reference's YAML config layer is not importable here")
    from agentsim.config import load_config

    exp = load_config(os.path.join(REPORT, name, "cfg.yaml"))
    return adapter.from_reference(exp.to_sim_config()), exp.resolved_dict()


def _same_bytes(name, outdir):
    for f in FILES:
        with open(os.path.join(REPORT, name, "out", f), "rb") as a, open(os.path.join(outdir, f), "rb") as b:
            assert a.read() == b.read(), (name, f)


@pytest.mark.parametrize("name", CASES)
def test_report_bytes_oracle(tmp_path, name):
    """The report writer over results rebuilt from the oracle's arrays."""
    cfg, echo = _experiment(name)
    batch_results, _ = results_via(run_oracle, [cfg], timeseries=True)
    res = batch_results[0]
    res.config_echo = echo
    export_report(res, str(tmp_path))
    _same_bytes(name, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_report_bytes_gpu(cuda_device, tmp_path, name):
    """run_simulation on the B200 (timeseries rows from the device) ->
    export_report == the reference CLI's report, every file."""
    cfg, echo = _experiment(name)
    res = run_simulation(cfg, config_echo=echo)
    export_report(res, str(tmp_path))
    _same_bytes(name, tmp_path)
