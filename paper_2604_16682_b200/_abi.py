"""ctypes / numpy mirrors of the C ABI structs in include/agentsim_b200.h.

Kept byte-compatible with the header; ``tests/test_abi.py`` checks the sizes
against ``asb_struct_sizes`` exported by the built library.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

ASB_NCOUNTERS = 16
CTR = {
    "ticks": 0,
    "arrived": 1,
    "completed": 2,
    "turns": 3,
    "events": 4,
    "migrations": 5,
    "thrash_flips": 6,
    "retimes": 7,
    "status": 8,
    "batches": 9,
}
ASB_NRED = 8
RED = ("energy", "thrash_fraction_sum", "completed", "slo_met", "ticks", "thrash_flips", "migrations", "turns")

VARIANTS = {"context_aware": 0, "off": 1, "fixed": 2}
POLICIES = {"context_aware": 0, "round_robin": 1, "least_loaded": 2}
PHASES = ("arriving", "pending", "running", "tool", "waiting_start", "done")
SIMERR = {0: "ok", 1: "invariant violation", 2: "engine buffer overflow", 3: "event scheduled before its parent",
          4: "engine watchdog (no progress inside a window)"}

SCENARIO_DTYPE = np.dtype(
    [
        ("trace_id", "<i4"),
        ("table_id", "<i4"),
        ("n_instances", "<i4"),
        ("n_levels", "<i4"),
        ("capacity", "<i8"),
        ("thrash_factor", "<f8"),
        ("interference", "<f8"),
        ("variant", "<i4"),
        ("fixed_level", "<i4"),
        ("boost_enabled", "<i4"),
        ("thrash_avoidance", "<i4"),
        ("alpha", "<f8"),
        ("beta", "<f8"),
        ("gamma", "<f8"),
        ("slo_target", "<f8"),
        ("epoch_length", "<f8"),
        ("policy", "<i4"),
        ("reassign_interval", "<i4"),
        ("include_idle", "<i4"),
        ("reset_only_on_reassign", "<i4"),
        ("consolidation_threshold", "<f8"),
        ("imbalance_ratio", "<f8"),
        ("migration_delay", "<f8"),
        ("sim_duration", "<f8"),
        ("n_epochs", "<i8"),
        ("record_interval", "<f8"),
    ],
    align=True,
)

DECISION_DTYPE = np.dtype(
    [
        ("time", "<f8"),
        ("min_throughput", "<f8"),
        ("usage_observed", "<i8"),
        ("instance_id", "<i4"),
        ("frequency_level", "<i4"),
        ("admitted_count", "<i4"),
        ("pending_depth", "<i4"),
        ("boosted", "<i4"),
        ("deferred", "<i4"),
    ],
    align=True,
)

TIMESERIES_DTYPE = np.dtype(
    [
        ("time", "<f8"),
        ("power_watts", "<f8"),
        ("context_usage", "<i8"),
        ("instance_id", "<i4"),
        ("level_index", "<i4"),
        ("pending_depth", "<i4"),
        ("running_requests", "<i4"),
        ("thrashing", "<i4"),
        ("pad_", "<i4"),
    ],
    align=True,
)

REGIME_SPAN_DTYPE = np.dtype(
    [("start", "<f8"), ("end", "<f8"), ("instance_id", "<i4"), ("thrashing", "<i4")], align=True)

STATS_DTYPE = np.dtype(
    [
        ("slo_attainment", "<f8"),
        ("p5_throughput", "<f8"),
        ("job_throughput", "<f8"),
        ("average_power", "<f8"),
        ("energy", "<f8"),
        ("thrash_fraction", "<f8"),
        ("slo_met", "<i8"),
        ("n_completed_with_tp", "<i8"),
    ],
    align=True,
)

P = C.c_void_p


class AsbTracePool(C.Structure):
    _fields_ = [
        ("n_traces", C.c_int32),
        ("pad_", C.c_int32),
        ("trace_agent_off", P),
        ("trace_turn_off", P),
        ("arrival", P),
        ("agent_turn_off", P),
        ("prefill", P),
        ("decode", P),
        ("tool", P),
        ("arrival_order", P),
    ]


class AsbTablePool(C.Structure):
    _fields_ = [
        ("n_tables", C.c_int32),
        ("max_levels", C.c_int32),  # host-side: the largest level count (0: at most 16)
        ("table_off", P),
        ("mhz", P),
        ("prefill_rate", P),
        ("decode_rate", P),
        ("active_power", P),
        ("idle_power", P),
    ]


class AsbOutputs(C.Structure):
    _fields_ = [
        ("agent_off", P),
        ("inst_off", P),
        ("completion_time", P),
        ("llm_time", P),
        ("decode_total", P),
        ("max_context", P),
        ("context", P),
        ("turns_completed", P),
        ("final_instance", P),
        ("migrations", P),
        ("phase", P),
        ("arrival_rank", P),
        ("energy", P),
        ("thrash_time", P),
        ("final_usage", P),
        ("final_pending", P),
        ("final_level", P),
        ("pad_", C.c_int32),
        ("counters", P),
        ("dec_off", P),
        ("decisions", P),
        ("turn_off", P),
        ("turn_issue", P),
        ("turn_done", P),
        ("ts_off", P),
        ("timeseries", P),
        ("ts_count", P),
    ]


TRACE_FIELDS = ("trace_agent_off", "trace_turn_off", "arrival", "agent_turn_off", "prefill", "decode", "tool",
                "arrival_order")
TABLE_FIELDS = ("table_off", "mhz", "prefill_rate", "decode_rate", "active_power", "idle_power")
AGENT_OUT = {
    "completion_time": np.float64,
    "llm_time": np.float64,
    "decode_total": np.int64,
    "max_context": np.int64,
    "context": np.int64,
    "turns_completed": np.int32,
    "final_instance": np.int32,
    "migrations": np.int32,
    "phase": np.int32,
    "arrival_rank": np.int32,
}
INST_OUT = {
    "energy": np.float64,
    "thrash_time": np.float64,
    "final_usage": np.int64,
    "final_pending": np.int32,
    "final_level": np.int32,
}


def struct_sizes() -> list[int]:
    """Sizes in header order, as the C side reports them via asb_struct_sizes."""
    return [SCENARIO_DTYPE.itemsize, C.sizeof(AsbTracePool), C.sizeof(AsbTablePool), C.sizeof(AsbOutputs),
            DECISION_DTYPE.itemsize, STATS_DTYPE.itemsize, TIMESERIES_DTYPE.itemsize, REGIME_SPAN_DTYPE.itemsize]


def make_outputs(ptr_of, arrays: dict) -> AsbOutputs:
    """Fill an AsbOutputs from a dict of arrays; ``ptr_of`` maps array -> address (None -> NULL)."""
    out = AsbOutputs()
    for name, _ in AsbOutputs._fields_:
        if name == "pad_":
            continue
        arr = arrays.get(name)
        setattr(out, name, ptr_of(arr) if arr is not None else None)
    return out


def make_pool(cls, ptr_of, arrays: dict, count_field: str, count: int, **scalars):
    pool = cls()
    setattr(pool, count_field, count)
    for name, value in scalars.items():
        setattr(pool, name, value)
    for name, ctype in cls._fields_:
        if name in (count_field, "pad_") or name in scalars or ctype is not P:
            continue
        setattr(pool, name, ptr_of(arrays[name]))
    return pool
