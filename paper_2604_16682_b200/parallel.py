"""Scenario sharding across GPUs (one process per GPU) — SURVEY §8(e).

Scenarios are fully independent (the reference runs sweep cells in separate
processes with zero shared state, /root/reference/pkg/src/agentsim/cli.py:
186-188), so the data path has no collective at all: each rank
runs its own shard of scenarios to completion with ``asb_run_scenarios``.
The only exchange step is at the end:

* ``allreduce_stats`` — one ``all_reduce(sum)`` of the ASB_NRED-double stats
  vector that ``asb_reduce_stats`` folds on each device (Σ energy, Σ thrash
  fraction, completed, SLO-met, agent-ticks, thrash flips, migrations,
  turns);
* ``gather_rows`` — an optional ``all_gather`` of the per-scenario
  ``SystemMetrics`` rows (AsbStats, 64 B each) plus the scenario counters,
  reassembled in global scenario order, so per-scenario results are
  bit-identical for every world size.

Partitioning (``partition_lpt``) is static longest-processing-time-first by
Σ trace turns per scenario, a proxy for its event count; inside a GPU the
engine's persistent grid pulls scenarios from an atomic queue, which absorbs
the remaining heavy-tail imbalance.

Everything here is host logic over ``torch.distributed``; on GPUs the group
is NCCL over NVLink/NVSwitch, and the CPU tests run the same functions over
gloo with world size 2 (tests/test_parallel.py).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _abi

STATS_WORDS = _abi.STATS_DTYPE.itemsize // 8  # AsbStats as float64/int64 words


def scenario_weights(batch) -> np.ndarray:
    """Σ trace turns per scenario of a packed batch (the LPT cost proxy)."""
    tto = batch.traces.trace_turn_off
    tid = batch.scen["trace_id"].astype(np.int64)
    return (tto[tid + 1] - tto[tid]).astype(np.int64)


def config_weights(configs) -> np.ndarray:
    """LPT cost proxy per SimConfig without packing anything (every rank
    computes it identically from the configs alone): Σ trace turns for
    inline traces, the expected turn count (arrival_rate · duration · mean
    turns, workload.py:134-152) for a WorkloadSpec, the file size for a
    trace path."""
    import os

    from .engine import _trace_key

    out = np.zeros(len(configs), dtype=np.int64)
    memo: dict = {}
    for s, c in enumerate(configs):
        key = _trace_key(c)
        if key not in memo:
            if key[0] == "objects":
                w = sum(len(t.turns) for t in c.traces)
            elif key[0] == "path":
                w = os.path.getsize(c.trace_path) // 64 if os.path.exists(c.trace_path) else 1
            else:
                spec = key[1]
                w = int(spec.arrival_rate * spec.duration * spec.turn_count.mean)
            memo[key] = max(int(w), 1)
        out[s] = memo[key]
    return out


def check_status_all(counters, group=None) -> None:
    """Raise SimulationError on EVERY rank when any scenario on any rank
    reported a device status (overflow, livelock, invariant violation): one
    all_reduce(MAX) of the local worst status, so no rank returns partial
    aggregates."""
    import torch
    import torch.distributed as dist

    from .errors import SimulationError

    ctr = counters.view(-1, _abi.ASB_NCOUNTERS) if counters.numel() else counters.view(0, _abi.ASB_NCOUNTERS)
    st = ctr[:, _abi.CTR["status"]]
    worst = torch.zeros(1, dtype=torch.int64, device=counters.device)
    if st.numel():
        worst = torch.maximum(worst, st.max().reshape(1))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(worst, op=dist.ReduceOp.MAX, group=group)
    code = int(worst.item())
    if code:
        raise SimulationError(f"a scenario of the sharded run reported {_abi.SIMERR.get(code, code)}")


def partition_lpt(weights: Sequence[int] | np.ndarray, world: int) -> list[np.ndarray]:
    """Static LPT partition of scenarios over ``world`` ranks.

    Scenarios are placed heaviest first (ties: lower index first) on the
    currently lightest rank (ties: lower rank).  Returns, per rank, the
    ascending array of global scenario indices it owns.  Deterministic, so
    every rank computes the same partition without communicating.
    """
    if world < 1:
        raise ValueError(f"world must be >= 1, got {world}")
    w = np.asarray(weights, dtype=np.int64)
    order = sorted(range(w.size), key=lambda s: (-int(w[s]), s))
    heap = [(0, r) for r in range(world)]
    owned: list[list[int]] = [[] for _ in range(world)]
    for s in order:
        load, r = heapq.heappop(heap)
        owned[r].append(s)
        heapq.heappush(heap, (load + int(w[s]), r))
    return [np.array(sorted(o), dtype=np.int64) for o in owned]


def allreduce_stats(red, group=None):
    """Sum the per-rank stats vector across ranks in place (no-op at world 1)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(red, op=dist.ReduceOp.SUM, group=group)
    return red


def gather_rows(local_index, stats_rows, counters, n_total: int, group=None):
    """All-gather per-scenario rows into global scenario order.

    local_index: int64 tensor [n_local] of global scenario ids owned here;
    stats_rows: uint8 tensor [n_local * sizeof(AsbStats)];
    counters: int64 tensor [n_local * ASB_NCOUNTERS].
    Returns (stats uint8 [n_total * 64], counters int64 [n_total * 16]) on
    every rank.  Shards are padded to the largest one for the collective.
    """
    import torch
    import torch.distributed as dist

    dev = stats_rows.device
    sz = _abi.STATS_DTYPE.itemsize
    nc = _abi.ASB_NCOUNTERS
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    n_local = int(local_index.numel())
    words = 1 + sz // 8 + nc  # index, stats row, counters: one int64 record per scenario
    rec = torch.empty((n_local, words), dtype=torch.int64, device=dev)
    rec[:, 0] = local_index.to(dev)
    rec[:, 1:1 + sz // 8] = stats_rows.view(torch.int64).view(n_local, sz // 8)
    rec[:, 1 + sz // 8:] = counters.view(n_local, nc)
    if world > 1:
        sizes = torch.tensor([n_local], dtype=torch.int64, device=dev)
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        mx = int(max(int(s) for s in all_sizes))
        pad = torch.full((mx, words), -1, dtype=torch.int64, device=dev)
        pad[:n_local] = rec
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        rec = torch.cat([p[: int(n)] for p, n in zip(parts, all_sizes)], dim=0)
    out = torch.empty((n_total, words), dtype=torch.int64, device=dev)
    out[rec[:, 0]] = rec
    stats = out[:, 1:1 + sz // 8].contiguous().view(torch.uint8).reshape(-1)
    ctr = out[:, 1 + sz // 8:].contiguous().reshape(-1)
    return stats, ctr


@dataclass
class ShardedResult:
    """What one rank holds after ``run_sharded``."""

    rank: int
    world: int
    local_index: np.ndarray          # global scenario ids run on this rank
    local_results: list              # SimulationResult per local scenario (if requested)
    totals: dict                     # allreduced stats vector, by _abi.RED name
    stats: np.ndarray                # AsbStats rows for ALL scenarios, global order (gather=True)
    counters: np.ndarray             # [n_total, ASB_NCOUNTERS] for ALL scenarios (gather=True)


def run_sharded(configs, *, group=None, device=None, results: bool = False, gather: bool = True,
                decisions: bool = False, turn_log: bool = False) -> ShardedResult:
    """Run a list of SimConfigs sharded over the ranks of ``group``.

    Each rank takes its LPT share, runs it on its GPU (one persistent engine
    launch), folds the stats on device and joins one all_reduce; a device
    status on any rank raises SimulationError on every rank; with
    ``gather`` the per-scenario SystemMetrics rows are all-gathered into
    global order.  There is no CPU fallback.
    """
    import torch
    import torch.distributed as dist

    from . import _native
    from .engine import DeviceBatch, build_results, prepare_batch

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    dev = _native.device(device)
    for c in configs:
        c.validate()
    # weights from the configs alone: no rank packs scenarios it does not run
    owned = partition_lpt(config_weights(configs), world)[rank]
    mine = [configs[int(s)] for s in owned]
    local_res: list = []
    if mine:
        batch = prepare_batch(mine)
        db = DeviceBatch(batch, device=dev, decisions=decisions, turn_log=turn_log)
        db.run()
        red = db.red
        stats_rows, ctr = db.stats, db.outputs["counters"]
    else:
        batch = db = None
        red = torch.zeros(_abi.ASB_NRED, dtype=torch.float64, device=dev)
        stats_rows = torch.empty(0, dtype=torch.uint8, device=dev)
        ctr = torch.empty(0, dtype=torch.int64, device=dev)
    check_status_all(ctr, group)
    red = allreduce_stats(red.clone(), group)
    all_stats = np.zeros(0, dtype=_abi.STATS_DTYPE)
    all_ctr = np.zeros((0, _abi.ASB_NCOUNTERS), dtype=np.int64)
    if gather:
        idx = torch.from_numpy(owned).to(dev)
        s_all, c_all = gather_rows(idx, stats_rows, ctr, len(configs), group)
        all_stats = s_all.cpu().numpy().view(_abi.STATS_DTYPE)
        all_ctr = c_all.cpu().numpy().reshape(-1, _abi.ASB_NCOUNTERS)
    if results and db is not None:
        host, st = db.download()
        local_res = build_results(batch, host, st, mine, None)
    totals = {k: float(v) for k, v in zip(_abi.RED, red.cpu().tolist())}
    return ShardedResult(rank, world, owned, local_res, totals, all_stats, all_ctr)
