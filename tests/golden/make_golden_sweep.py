"""Generate the sweep golden fixtures by running the REFERENCE's own CLI
(``agentsim sweep``, cli.py:177-211) in the build container:

    python tests/golden/make_golden_sweep.py

Each case: an experiment YAML (written to a temp dir), the CLI axis flags,
and the resulting ``sweep.csv`` text, saved as tests/golden/sweep/<case>.json.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import yaml

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from common import reference_module  # noqa: E402

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"
from agentsim import cli  # noqa: E402

CASES = {
    "levels_x_policy": (
        {"workload": {"arrival_rate": 0.2, "duration": 300, "seed": 3},
         "instance": {"count": 2, "capacity_tokens": 60000}, "sim": {"duration": 400}},
        ["--axis-level-mhz", "660", "1185", "1680", "--axis-policy", "round-robin", "context-aware"],
    ),
    "rate_x_slo": (
        {"workload": {"arrival_rate": 0.1, "duration": 400, "seed": 8},
         "instance": {"count": 3, "capacity_tokens": 40000}, "sim": {"duration": 500}},
        ["--axis-rate", "0.05", "0.2", "0.5", "--axis-slo", "20", "35"],
    ),
    "yaml_axes": (
        {"workload": {"arrival_rate": 0.3, "duration": 200, "seed": 1},
         "instance": {"count": 4, "capacity_tokens": 30000, "interference_coeff": 0.05},
         "router": {"reassign_interval": 2, "migration_delay": 2.0}, "sim": {"duration": 300},
         "sweep": {"policy": ["least-loaded", "context-aware"], "slo_target": [25.0]}},
        [],
    ),
}


def main():
    out_dir = os.path.join(HERE, "sweep")
    os.makedirs(out_dir, exist_ok=True)
    for name, (doc, axes) in CASES.items():
        with tempfile.TemporaryDirectory() as tmp:
            cfg = os.path.join(tmp, "exp.yaml")
            with open(cfg, "w") as fh:
                yaml.safe_dump(doc, fh)
            rc = cli.main(["sweep", "--config", cfg, "--out", os.path.join(tmp, "o"), *axes])
            with open(os.path.join(tmp, "o", "sweep.csv"), encoding="utf-8") as fh:
                csv = fh.read()
        with open(os.path.join(out_dir, name + ".json"), "w") as fh:
            json.dump({"name": name, "experiment": doc, "axes": axes, "rc": rc, "sweep_csv": csv}, fh, indent=1)
        print(name, rc, csv.count("\n") - 1, "cells")


if __name__ == "__main__":
    main()
