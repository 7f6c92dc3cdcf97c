"""PyTorch custom ops over the C ABI (``torch.ops.agentsim_b200.*``).

Each op takes device tensors, passes raw pointers + sizes + the current CUDA
stream to the C ABI of include/agentsim_b200.h, and returns device tensors.
The list-taking helpers below (``select_level_batch`` …) are the convenience
layer used by the scalar API mirror and the SPEC acceptance grids.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi, _native

_NS = "agentsim_b200"

# AsbOutputs slots, in the order the run_scenarios op receives them
OUT_ORDER = (
    ("agent_off", torch.int64),
    ("inst_off", torch.int64),
    *((k, {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[v]) for k, v in _abi.AGENT_OUT.items()),
    *((k, {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[v]) for k, v in _abi.INST_OUT.items()),
    ("counters", torch.int64),
    ("dec_off", torch.int64),
    ("decisions", torch.uint8),
    ("turn_off", torch.int64),
    ("turn_issue", torch.float64),
    ("turn_done", torch.float64),
    ("ts_off", torch.int64),
    ("timeseries", torch.uint8),
    ("ts_count", torch.int64),
)
OUT_NAMES = tuple(k for k, _ in OUT_ORDER)


def _ptr(t: torch.Tensor | None):
    return t.data_ptr() if t is not None and t.numel() > 0 else None


def _stream(t: torch.Tensor) -> int:
    return _native.stream_handle(t.device)


def _on(t: torch.Tensor):
    """The C ABI launches on the CURRENT device (cudaGetDevice, kernel
    attributes, the launch itself): make it the tensors' device, so that
    ``device='cuda:1'`` with cuda:0 current gets cuda:1's stream and memory."""
    return torch.cuda.device(t.device)


# --------------------------------------------------------------------------- engine


@torch.library.custom_op(f"{_NS}::run_scenarios", mutates_args=("outputs", "workspace"))
def run_scenarios(
    scen: torch.Tensor,
    traces: list[torch.Tensor],
    tables: list[torch.Tensor],
    outputs: list[torch.Tensor],
    workspace: torch.Tensor,
    max_instances: int,
    total_agents: int,
    total_ring: int,
    max_levels: int = 0,
) -> None:
    """Run every scenario of the batch on the GPU (asb_run_scenarios).
    ``max_levels``: the largest frequency table of the batch (0: at most 16)."""
    lib = _native.lib()
    n_scen = scen.numel() // _abi.SCENARIO_DTYPE.itemsize
    tp = _abi.make_pool(_abi.AsbTracePool, _ptr, dict(zip(_abi.TRACE_FIELDS, traces)), "n_traces",
                        traces[0].numel() - 1)
    tb = _abi.make_pool(_abi.AsbTablePool, _ptr, dict(zip(_abi.TABLE_FIELDS, tables)), "n_tables",
                        tables[0].numel() - 1, max_levels=max_levels)
    out = _abi.make_outputs(_ptr, dict(zip(OUT_NAMES, outputs)))
    with _on(scen):
        rc = lib.asb_run_scenarios(_ptr(scen), n_scen, max_instances, tp, tb, out, total_agents, total_ring,
                                   _ptr(workspace), workspace.numel(), _stream(scen))
    _native.check(rc, "asb_run_scenarios")


@torch.library.custom_op(f"{_NS}::scenario_stats", mutates_args=("stats",))
def scenario_stats(scen: torch.Tensor, outputs: list[torch.Tensor], stats: torch.Tensor) -> None:
    """Per-scenario SystemMetrics on device (asb_scenario_stats)."""
    lib = _native.lib()
    n_scen = scen.numel() // _abi.SCENARIO_DTYPE.itemsize
    out = _abi.make_outputs(_ptr, dict(zip(OUT_NAMES, outputs)))
    with _on(scen):
        rc = lib.asb_scenario_stats(_ptr(scen), n_scen, out, _ptr(stats), None, 0, _stream(scen))
    _native.check(rc, "asb_scenario_stats")


@torch.library.custom_op(f"{_NS}::reduce_stats", mutates_args=("red",))
def reduce_stats(stats: torch.Tensor, counters: torch.Tensor, n_scen: int, red: torch.Tensor) -> None:
    with _on(red):
        rc = _native.lib().asb_reduce_stats(_ptr(stats), _ptr(counters), n_scen, _ptr(red), _stream(red))
    _native.check(rc, "asb_reduce_stats")


# --------------------------------------------------------------------------- unit ops


@torch.library.custom_op(f"{_NS}::select_frequency_level", mutates_args=())
def select_frequency_level(usage: torch.Tensor, capacity: torch.Tensor, num_levels: torch.Tensor,
                           alpha: torch.Tensor) -> torch.Tensor:
    out = torch.empty(usage.shape, dtype=torch.int32, device=usage.device)
    with _on(usage):
        rc = _native.lib().asb_select_level_batch(_ptr(usage), _ptr(capacity), _ptr(num_levels), _ptr(alpha),
                                                  _ptr(out), usage.numel(), _stream(usage))
    _native.check(rc, "asb_select_level_batch")
    return out


@select_frequency_level.register_fake
def _(usage, capacity, num_levels, alpha):
    return torch.empty(usage.shape, dtype=torch.int32, device=usage.device)


@torch.library.custom_op(f"{_NS}::service_time", mutates_args=())
def service_time(prefill: torch.Tensor, decode: torch.Tensor, prefill_rate: torch.Tensor,
                 decode_rate: torch.Tensor, concurrent: torch.Tensor, thrashing: torch.Tensor,
                 interference: float, thrash_factor: float) -> torch.Tensor:
    out = torch.empty(prefill.shape, dtype=torch.float64, device=prefill.device)
    with _on(prefill):
        rc = _native.lib().asb_service_time_batch(_ptr(prefill), _ptr(decode), _ptr(prefill_rate), _ptr(decode_rate),
                                                  _ptr(concurrent), _ptr(thrashing), interference, thrash_factor,
                                                  _ptr(out), prefill.numel(), _stream(prefill))
    _native.check(rc, "asb_service_time_batch")
    return out


@service_time.register_fake
def _(prefill, decode, prefill_rate, decode_rate, concurrent, thrashing, interference, thrash_factor):
    return torch.empty(prefill.shape, dtype=torch.float64, device=prefill.device)


@torch.library.custom_op(f"{_NS}::route_assign", mutates_args=())
def route_assign(usages: torch.Tensor, m: torch.Tensor, capacity: int, threshold: float, policy: int) -> torch.Tensor:
    out = torch.empty(usages.shape[0], dtype=torch.int32, device=usages.device)
    with _on(usages):
        rc = _native.lib().asb_assign_batch(_ptr(usages), _ptr(m), usages.shape[1], capacity, threshold, policy,
                                            _ptr(out), usages.shape[0], _stream(usages))
    _native.check(rc, "asb_assign_batch")
    return out


@route_assign.register_fake
def _(usages, m, capacity, threshold, policy):
    return torch.empty(usages.shape[0], dtype=torch.int32, device=usages.device)


@torch.library.custom_op(f"{_NS}::route_reassign", mutates_args=("counters",))
def route_reassign(usages: torch.Tensor, m: torch.Tensor, current: torch.Tensor, counters: torch.Tensor,
                   interval: int, ratio: float, include_idle: bool, reset_only: bool) -> torch.Tensor:
    out = torch.empty(usages.shape[0], dtype=torch.int32, device=usages.device)
    with _on(usages):
        rc = _native.lib().asb_reassign_batch(_ptr(usages), _ptr(m), usages.shape[1], _ptr(current), _ptr(counters),
                                              interval, ratio, int(include_idle), int(reset_only), _ptr(out),
                                              usages.shape[0], _stream(usages))
    _native.check(rc, "asb_reassign_batch")
    return out


@torch.library.custom_op(f"{_NS}::min_throughput", mutates_args=())
def min_throughput(decode_total: torch.Tensor, llm_time: torch.Tensor, segment: torch.Tensor,
                   n_seg: int) -> torch.Tensor:
    out = torch.empty(n_seg, dtype=torch.float64, device=decode_total.device)
    scratch = torch.empty(n_seg, dtype=torch.float64, device=decode_total.device)
    with _on(decode_total):
        rc = _native.lib().asb_min_throughput_batch(_ptr(decode_total), _ptr(llm_time), _ptr(segment),
                                                    decode_total.numel(), n_seg, _ptr(scratch), _ptr(out),
                                                    _stream(decode_total))
    _native.check(rc, "asb_min_throughput_batch")
    return out


# --------------------------------------------------------------------------- list helpers


def _dev(device=None):
    return _native.device(device)


def select_level_batch(usage, capacity, num_levels, alpha, device=None) -> np.ndarray:
    d = _dev(device)
    out = torch.ops.agentsim_b200.select_frequency_level(
        torch.as_tensor(np.asarray(usage, dtype=np.float64), device=d),
        torch.as_tensor(np.asarray(capacity, dtype=np.float64), device=d),
        torch.as_tensor(np.asarray(num_levels, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(alpha, dtype=np.float64), device=d),
    )
    return out.cpu().numpy()


def service_time_batch(prefill, decode, prefill_rate, decode_rate, concurrent, thrashing, interference,
                       thrash_factor, device=None) -> np.ndarray:
    d = _dev(device)
    out = torch.ops.agentsim_b200.service_time(
        torch.as_tensor(np.asarray(prefill, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(decode, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(prefill_rate, dtype=np.float64), device=d),
        torch.as_tensor(np.asarray(decode_rate, dtype=np.float64), device=d),
        torch.as_tensor(np.asarray(concurrent, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(thrashing, dtype=np.int32), device=d),
        float(interference), float(thrash_factor),
    )
    return out.cpu().numpy()


def _usage_matrix(rows):
    m = np.array([len(r) for r in rows], dtype=np.int32)
    width = max(int(m.max()), 1)
    mat = np.zeros((len(rows), width), dtype=np.float64)
    for k, r in enumerate(rows):
        mat[k, : len(r)] = r
    return mat, m


def assign_batch(usage_rows, capacity, threshold, policy: str, device=None) -> np.ndarray:
    """1-based position of the chosen instance in each usage row."""
    d = _dev(device)
    mat, m = _usage_matrix(usage_rows)
    out = torch.ops.agentsim_b200.route_assign(torch.as_tensor(mat, device=d), torch.as_tensor(m, device=d),
                                               int(capacity), float(threshold), _abi.POLICIES[policy])
    return out.cpu().numpy()


def reassign_batch(usage_rows, current, counters, interval, ratio, include_idle, reset_only, device=None):
    """(target positions (0 = none), updated counters)."""
    d = _dev(device)
    mat, m = _usage_matrix(usage_rows)
    ctr = torch.as_tensor(np.asarray(counters, dtype=np.int32), device=d).clone()
    out = torch.ops.agentsim_b200.route_reassign(
        torch.as_tensor(mat, device=d), torch.as_tensor(m, device=d),
        torch.as_tensor(np.asarray(current, dtype=np.int32), device=d), ctr,
        int(interval), float(ratio), bool(include_idle), bool(reset_only),
    )
    return out.cpu().numpy(), ctr.cpu().numpy()


def min_throughput_batch(decode_total, llm_time, segment, n_seg, device=None) -> np.ndarray:
    d = _dev(device)
    out = torch.ops.agentsim_b200.min_throughput(
        torch.as_tensor(np.asarray(decode_total, dtype=np.int64), device=d),
        torch.as_tensor(np.asarray(llm_time, dtype=np.float64), device=d),
        torch.as_tensor(np.asarray(segment, dtype=np.int32), device=d),
        int(n_seg),
    )
    return out.cpu().numpy()
