"""Drop-in adapter for the reference's own objects.

A caller of the reference (``agentsim``) keeps its objects: ``SimConfig``
with ``WorkloadSpec`` / ``AgentTrace`` / ``InstanceConfig`` /
``ControllerConfig`` / ``RouterConfig`` (agentsim/engine.py:57-88,
workload.py:83-116) go in, the reference's ``SimulationResult`` with its
``AgentResult`` / ``DecisionRow`` / ``TimeseriesRow`` / ``SystemMetrics``
(engine.py:91-182, metrics.py) comes out, and the simulation runs on the
B200 engine.  The two packages' configuration and result types have the same
class names and fields, so the conversion is structural: a dataclass tree is
rebuilt class by class in the target module.  Trace objects are not copied:
the packer reads their attributes (``arrival_time``, ``turns`` of
``prefill_tokens`` / ``decode_tokens`` / ``tool_time``) directly.

    import agentsim
    from paper_2604_16682_b200 import adapter
    result = adapter.run_simulation(agentsim_config)   # an agentsim.SimulationResult

This is what a maintainer binds behind ``agentsim.run_simulation``
(engine.py:752-754) or a ``--backend b200`` switch of ``cmd_run`` /
``_run_cell`` (cli.py:126, 161-174).
"""

from __future__ import annotations

import dataclasses
import sys
from typing import Sequence

from . import engine as _engine

_THIS = sys.modules[__package__]


def convert(obj, mod):
    """Rebuild a tree of dataclass instances with ``mod``'s classes of the
    same names (fields the target class does not declare are dropped, e.g.
    this package's ``SimulationResult.counters``).  Lists, tuples and dicts
    are converted element-wise; everything else is kept as is."""
    if dataclasses.is_dataclass(obj) and not isinstance(obj, type):
        cls = getattr(mod, type(obj).__name__, None)
        if cls is None:
            raise TypeError(f"{mod.__name__} has no class {type(obj).__name__!r}")
        if cls is type(obj):
            return obj
        kwargs = {f.name: convert(getattr(obj, f.name), mod)
                  for f in dataclasses.fields(cls) if f.init and hasattr(obj, f.name)}
        return cls(**kwargs)
    if isinstance(obj, list):
        return [convert(x, mod) for x in obj]
    if isinstance(obj, tuple):
        return tuple(convert(x, mod) for x in obj)
    if isinstance(obj, dict):
        return {k: convert(v, mod) for k, v in obj.items()}
    return obj


def from_reference(config) -> _engine.SimConfig:
    """This package's SimConfig for a reference (or duck-typed) SimConfig;
    ``traces`` keep the caller's objects (read by attribute when packed)."""
    if isinstance(config, _engine.SimConfig):
        return config
    traces = getattr(config, "traces", None)
    shell = dataclasses.replace(config, traces=None) if traces is not None else config
    mine = convert(shell, _THIS)
    if traces is not None:
        mine.traces = traces
    return mine


def _module_of(config):
    return sys.modules[type(config).__module__.split(".")[0]]


def to_reference(result, mod):
    """The reference's SimulationResult (``mod``'s types) for one of ours."""
    return convert(result, mod)


def run_simulation_batch(configs: Sequence, config_echos: Sequence[dict | None] | None = None, *,
                         device=None, timeseries: bool = False) -> list:
    """``agentsim.run_simulation`` for every config, as one B200 launch;
    results come back in the callers' own result types."""
    mine = [from_reference(c) for c in configs]
    res = _engine.run_simulation_batch(mine, config_echos, device=device, timeseries=timeseries)
    return [to_reference(r, _module_of(c)) for r, c in zip(res, configs)]


def run_simulation(config, config_echo: dict | None = None, *, device=None, timeseries: bool = True):
    """Drop-in for ``agentsim.run_simulation(config, config_echo)``
    (engine.py:752-754): same result type, fields and values."""
    return run_simulation_batch([config], [config_echo], device=device, timeseries=timeseries)[0]
