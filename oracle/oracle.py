"""TEST INFRASTRUCTURE ONLY — ctypes driver for the C oracle (des_oracle.c).

`run_oracle(batch)` executes the serial restatement of the reference engine
(/root/reference/pkg/src/agentsim/engine.py) on the host over the same packed
batch the GPU consumes, and returns the same output arrays.  Parity pin:
tests/test_oracle_golden.py compares it with golden vectors produced by the
reference itself (tests/golden/make_golden.py).

`run_host_engine(batch)` runs the 1-lane CPU build of the GPU engine core
(tests/native/host_engine.cpp) — a harness for debugging the batching logic
on CPU; it is not the product either.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from paper_2604_16682_b200 import _abi, _build
from paper_2604_16682_b200.engine import alloc_host_outputs

_LIBS: dict = {}


def _np_ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def _load(path: str, fn: str, extra: list):
    if path not in _LIBS:
        lib = C.CDLL(path)
        f = getattr(lib, fn)
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(_abi.AsbTracePool), C.POINTER(_abi.AsbTablePool),
                      C.POINTER(_abi.AsbOutputs), *extra]
        if fn == "oracle_run_scenarios":
            g = lib.oracle_scenario_stats
            g.restype = C.c_int
            g.argtypes = [C.c_void_p, C.c_int32, C.POINTER(_abi.AsbOutputs), C.c_void_p]
        _LIBS[path] = lib
    return _LIBS[path]


def _structs(batch, arrays):
    tp = _abi.make_pool(_abi.AsbTracePool, _np_ptr, batch.traces.arrays(), "n_traces", batch.traces.n_traces)
    tb = _abi.make_pool(_abi.AsbTablePool, _np_ptr, batch.tables.arrays(), "n_tables", batch.tables.n_tables,
                        max_levels=batch.max_levels)
    out = _abi.make_outputs(_np_ptr, arrays)
    return tp, tb, out


def run_oracle(batch, decisions: bool = True, turn_log: bool = True, threads: int = 0, timing: dict | None = None,
               timeseries: bool = False):
    """Serial C oracle over every scenario; returns (outputs, stats)."""
    lib = _load(_build.build_oracle(), "oracle_run_scenarios", [C.c_int32])
    arrays = alloc_host_outputs(batch, decisions, turn_log, timeseries)
    tp, tb, out = _structs(batch, arrays)
    scen = np.ascontiguousarray(batch.scen)
    t0 = time.perf_counter()
    lib.oracle_run_scenarios(scen.ctypes.data, batch.n, C.byref(tp), C.byref(tb), C.byref(out), threads)
    stats = np.zeros(batch.n, dtype=_abi.STATS_DTYPE)
    lib.oracle_scenario_stats(scen.ctypes.data, batch.n, C.byref(out), stats.ctypes.data)
    if timing is not None:
        timing["seconds"] = time.perf_counter() - t0
    return arrays, stats


def run_host_engine(batch, small_buffers: bool = False, decisions: bool = True, turn_log: bool = True,
                    timeseries: bool = False, serial_due: bool = False):
    """1-lane CPU build of the GPU engine core (test harness); returns (outputs, stats)."""
    lib = _load(_build.build_host_engine(), "host_engine_run", [C.c_int32])
    olib = _load(_build.build_oracle(), "oracle_run_scenarios", [C.c_int32])
    arrays = alloc_host_outputs(batch, decisions, turn_log, timeseries)
    tp, tb, out = _structs(batch, arrays)
    scen = np.ascontiguousarray(batch.scen)
    lib.host_engine_run(scen.ctypes.data, batch.n, C.byref(tp), C.byref(tb), C.byref(out), int(small_buffers) | (2 if serial_due else 0))
    stats = np.zeros(batch.n, dtype=_abi.STATS_DTYPE)
    olib.oracle_scenario_stats(scen.ctypes.data, batch.n, C.byref(out), stats.ctypes.data)
    return arrays, stats
