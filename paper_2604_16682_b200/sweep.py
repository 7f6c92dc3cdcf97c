"""Batched sweep driver: the caller side of the hot path.

The reference's ``agentsim sweep`` (cli.py:136-211) expands the sweep axes
into cells (``_sweep_cells``, cli.py:136-158), applies each cell to the base
experiment (``apply_cell``, config.py:302-315), runs every cell with
``run_simulation`` in a process pool (``_run_cell``, cli.py:161-174) and
writes ``sweep.csv``.  Here the cells of a sweep run in ONE engine launch
(one CTA team per cell), with the same per-cell outcome tuples:

    outcomes = run_cells(base, sweep_cells({"level_mhz": [660.0, 1680.0], "policy": ["round_robin"]}))
    write_sweep_table("out/sweep.csv", outcomes)

Beyond the reference's four axes (config.py:64), ``capacity``, ``variant``
and ``seed`` express the BASELINE sweeps: C3 is
``{"level_mhz": 8 levels, "capacity": 4 caps, "seed": range(64)}`` and C5
``{"slo_target": [20, 35], "policy": [...], "variant": [...], "seed": ...}``.

A cell that fails validation is recorded with its error and the sweep
continues (cli.py:172-174); the others still share the launch.  The YAML
front end (``ExperimentConfig``) is out of scope, so cells apply to a
``SimConfig`` and a failing cell's message is ``SimConfig.validate``'s.
"""

from __future__ import annotations

import itertools
import os
from dataclasses import replace
from typing import Mapping, Sequence

from .engine import SimConfig, run_simulation_batch
from .errors import ConfigurationError, SimulationError
from .metrics import SUMMARY_FIELDS, format_value

SWEEP_AXES = ("level_mhz", "arrival_rate", "slo_target", "policy")  # config.py:64
# axes beyond the reference's four, for the BASELINE sweeps the reference CLI
# cannot express (C3: seed x level x capacity; C5: seed x policy x variant x
# SLO target).  They come after the reference's axes in the cell order and
# the sweep.csv columns, so a sweep over the reference's axes alone is
# unchanged.
EXTRA_AXES = ("capacity", "variant", "seed")
ALL_AXES = SWEEP_AXES + EXTRA_AXES


def sweep_cells(axes: Mapping[str, Sequence]) -> list[dict]:
    """Cartesian product of the given axes in ALL_AXES order (cli.py:136-158):
    the last axis varies fastest."""
    unknown = [a for a in axes if a not in ALL_AXES]
    if unknown:
        raise ConfigurationError(f"sweep: unknown axis {unknown[0]!r}")
    for axis, values in axes.items():
        if values is not None and not list(values):
            raise ConfigurationError(f"sweep.{axis}: axis must be non-empty")
    names = [a for a in ALL_AXES if axes.get(a) is not None]
    if not names:
        raise ConfigurationError("sweep: at least one non-empty axis is required")
    return [dict(zip(names, combo)) for combo in itertools.product(*(list(axes[n]) for n in names))]


def apply_cell(base: SimConfig, cell: Mapping) -> SimConfig:
    """One cell's axis values applied to a copy of ``base`` (config.py:302-315)."""
    out = base
    if "level_mhz" in cell:
        out = replace(out, controller=replace(out.controller, variant="fixed", fixed_level_mhz=float(cell["level_mhz"])))
    if "arrival_rate" in cell:
        if out.workload is None:
            raise ConfigurationError("sweep.arrival_rate: the base config needs a workload spec")
        out = replace(out, workload=replace(out.workload, arrival_rate=float(cell["arrival_rate"])))
    if "slo_target" in cell:
        out = replace(out, controller=replace(out.controller, slo_target=float(cell["slo_target"])))
    if "policy" in cell:
        out = replace(out, router=replace(out.router, policy=str(cell["policy"]).replace("-", "_")))
    if "capacity" in cell:
        out = replace(out, instance=replace(out.instance, capacity_tokens=int(cell["capacity"])))
    if "variant" in cell:
        out = replace(out, controller=replace(out.controller, variant=str(cell["variant"]).replace("-", "_")))
    if "seed" in cell:
        # SimConfig.seed overrides the workload's seed (engine.py:70, 286-289)
        out = replace(out, seed=int(cell["seed"]))
    return out


def _summary(result) -> dict:
    s = {name: getattr(result.system, name) for name in SUMMARY_FIELDS}
    s["arrived"] = result.arrived
    s["completed"] = result.completed
    return s


def run_cells(base: SimConfig, cells: Sequence[Mapping], *, device=None,
              runner=None) -> list[tuple[dict, dict | None, str | None]]:
    """``[(cell, summary, error)]`` like ``_run_cell`` (cli.py:161-174) for every
    cell; the valid cells run in one batched launch.  ``runner`` (configs ->
    results) replaces the GPU batch, for tests."""
    if runner is None:
        def runner(cfgs):
            return run_simulation_batch(cfgs, device=device, decisions=False, turn_log=False)
    outcomes: list = [None] * len(cells)
    configs, where = [], []
    for k, cell in enumerate(cells):
        try:
            cfg = apply_cell(base, cell)
            cfg.validate()
        except (ConfigurationError, ValueError) as exc:
            outcomes[k] = (dict(cell), None, str(exc))
            continue
        configs.append(cfg)
        where.append(k)
    if configs:
        try:
            results = runner(configs)
        except (ConfigurationError, SimulationError):
            # one cell broke the batch (a trace error, a device status):
            # run cell by cell so the others are still recorded
            results = []
            for cfg in configs:
                try:
                    results.append(runner([cfg])[0])
                except (ConfigurationError, SimulationError) as exc:
                    results.append(exc)
        for k, res in zip(where, results):
            if isinstance(res, Exception):
                outcomes[k] = (dict(cells[k]), None, str(res))
            else:
                outcomes[k] = (dict(cells[k]), _summary(res), None)
    return outcomes


def write_sweep_table(path: str, outcomes: Sequence[tuple[dict, dict | None, str | None]]) -> int:
    """``sweep.csv`` in the reference's format (cli.py:190-210); returns the
    number of failed cells."""
    axis_names = [a for a in ALL_AXES if outcomes and a in outcomes[0][0]]
    header = axis_names + list(SUMMARY_FIELDS) + ["arrived", "completed", "status", "error"]
    failed = 0
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(",".join(header) + "\n")
        for cell, summary, error in outcomes:
            values = [format_value(cell[name]) for name in axis_names]
            if summary is None:
                failed += 1
                values += ["nan"] * (len(SUMMARY_FIELDS) + 2) + ["error", (error or "").replace(",", ";")]
            else:
                values += [format_value(summary[name]) for name in SUMMARY_FIELDS]
                values += [str(summary["arrived"]), str(summary["completed"]), "ok", ""]
            fh.write(",".join(values) + "\n")
    return failed
