"""Report directories written by the REFERENCE's own CLI (`agentsim run
--config cfg.yaml --out dir`, cli.py:121-135 -> export_report,
metrics.py:184-252), frozen for the byte-identity test of this package's
export_report on B200 results (tests/test_report.py).

    python tests/golden/make_golden_report.py      # build container only
"""

from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import reference_module  # noqa: E402

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"
from agentsim.cli import main  # noqa: E402

CONFIGS = {
    # the reference's own test_cli.py SMALL_CONFIG
    "small": """
workload:
  arrival_rate: 0.05
  duration: 300
  seed: 5
  turn_count: {dist: lognormal, mean: 8.0, sigma: 1.0, min: 1, max: 40}
sim:
  duration: 400
""",
    "ctx_migrate": """
workload:
  arrival_rate: 0.2
  duration: 300
  seed: 11
  turn_count: {dist: lognormal, mean: 12.0, sigma: 1.0, min: 1, max: 60}
instance:
  count: 4
  capacity_tokens: 30000
controller:
  slo_target: 35.0
router:
  reassign_interval: 2
  migration_delay: 3.0
sim:
  duration: 420
  record_interval: 2.5
""",
    "rr_fixed_interference": """
workload:
  arrival_rate: 0.1
  arrival_process: fixed_interval
  duration: 200
  seed: 2
  turn_count: {dist: lognormal, mean: 6.0, sigma: 1.0, min: 1, max: 30}
instance:
  count: 3
  capacity_tokens: 20000
  thrash_mode: offload
  interference_coeff: 0.1
controller:
  variant: fixed
  fixed_level_mhz: 900
router:
  policy: round-robin
sim:
  duration: 300
  record_interval: 0.7
""",
}

FILES = ("summary.csv", "agents.csv", "timeseries.csv", "decisions.csv", "config.yaml")


def main_():
    for name, text in CONFIGS.items():
        d = os.path.join(HERE, "report", name)
        shutil.rmtree(d, ignore_errors=True)
        os.makedirs(d)
        cfg = os.path.join(d, "cfg.yaml")
        with open(cfg, "w") as fh:
            fh.write(text.lstrip())
        out = os.path.join(d, "out")
        assert main(["run", "--config", cfg, "--out", out]) == 0
        print(name, {f: os.path.getsize(os.path.join(out, f)) for f in FILES})


if __name__ == "__main__":
    main_()
