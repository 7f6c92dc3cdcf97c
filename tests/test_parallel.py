"""Multi-rank host logic of the scenario sharding (paper_2604_16682_b200/
parallel.py) on CPU: LPT partition properties, and — over a real gloo
process group with world size 2 — the stats all_reduce and the
per-scenario row all_gather.  Per-scenario rows come from the oracle here
(test infrastructure standing in for each rank's device shard); the
collectives and the reassembly in global order are the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2604_16682_b200 as asb
from paper_2604_16682_b200 import _abi
from paper_2604_16682_b200.engine import prepare_batch
from paper_2604_16682_b200.parallel import (allreduce_stats, check_status_all, config_weights, gather_rows,
                                            partition_lpt, scenario_weights)


def test_partition_lpt_covers_and_balances():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        w = rng.pareto(1.2, size=257).astype(np.float64) * 1000 + 1
        w = w.astype(np.int64)
        parts = partition_lpt(w, world)
        assert len(parts) == world
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(w.size))
        loads = [int(w[p].sum()) for p in parts]
        # LPT bound: max load <= mean load + max single weight
        assert max(loads) <= w.sum() / world + w.max()
        assert all(np.all(np.diff(p) > 0) for p in parts)
        # deterministic
        again = partition_lpt(w, world)
        assert all(np.array_equal(a, b) for a, b in zip(parts, again))


def test_partition_lpt_more_ranks_than_scenarios():
    parts = partition_lpt([5, 3], 4)
    assert sorted(len(p) for p in parts) == [0, 0, 1, 1]
    with pytest.raises(ValueError):
        partition_lpt([1], 0)


def test_config_weights_without_packing():
    tr = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.4, duration=50.0, seed=1))
    spec = asb.WorkloadSpec(arrival_rate=2.0, duration=100.0, seed=3)
    cfgs = [asb.SimConfig(traces=tr), asb.SimConfig(workload=spec), asb.SimConfig(workload=spec, seed=9)]
    w = config_weights(cfgs)
    assert w[0] == sum(len(t.turns) for t in tr)
    assert w[1] == w[2] == int(2.0 * 100.0 * spec.turn_count.mean)
    assert np.array_equal(w, config_weights(cfgs))


def _configs():
    cfgs = []
    for seed in range(3):
        tr = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.4, duration=150.0, seed=seed))
        cfgs.append(asb.SimConfig(traces=tr, instance_count=3, sim_duration=220.0,
                                  instance=asb.InstanceConfig(capacity_tokens=30_000)))
        cfgs.append(asb.SimConfig(traces=tr, instance_count=2, sim_duration=220.0,
                                  controller=asb.ControllerConfig(variant="off"),
                                  router=asb.RouterConfig(policy="round_robin")))
    return cfgs


def host_fold(stats: np.ndarray, ctr: np.ndarray) -> np.ndarray:
    """numpy restatement of reduce_stats_kernel's fold (unit_ops.cu)."""
    c = _abi.CTR
    out = np.zeros(_abi.ASB_NRED)
    out[0] = stats["energy"].sum()
    out[1] = stats["thrash_fraction"].sum()
    out[2] = ctr[:, c["completed"]].sum()
    out[3] = stats["slo_met"].sum()
    out[4] = ctr[:, c["ticks"]].sum()
    out[5] = ctr[:, c["thrash_flips"]].sum()
    out[6] = ctr[:, c["migrations"]].sum()
    out[7] = ctr[:, c["turns"]].sum()
    return out


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import run_oracle

        cfgs = _configs()
        batch = prepare_batch(cfgs)
        host, stats = run_oracle(batch, decisions=False, turn_log=False)
        ctr = host["counters"].reshape(batch.n, _abi.ASB_NCOUNTERS)
        owned = partition_lpt(scenario_weights(batch), world)[rank]
        red = torch.from_numpy(host_fold(stats[owned], ctr[owned]))
        red = allreduce_stats(red)
        rows = torch.from_numpy(np.ascontiguousarray(stats[owned]).view(np.uint8).copy())
        c_loc = torch.from_numpy(np.ascontiguousarray(ctr[owned]).reshape(-1).copy())
        s_all, c_all = gather_rows(torch.from_numpy(owned), rows, c_loc, batch.n)
        got_stats = s_all.numpy().view(_abi.STATS_DTYPE)
        got_ctr = c_all.numpy().reshape(-1, _abi.ASB_NCOUNTERS)
        ok_rows = np.array_equal(got_stats.view(np.uint8), stats.view(np.uint8)) and np.array_equal(got_ctr, ctr)
        want = host_fold(stats, ctr)
        ok_red = np.allclose(red.numpy(), want, rtol=1e-12, atol=0) and np.array_equal(red.numpy()[2:], want[2:])
        # a device status on ONE rank raises on EVERY rank (no partial aggregates)
        check_status_all(c_loc)
        bad = c_loc.clone()
        if rank == 1 and bad.numel():
            bad[_abi.CTR["status"]] = 3
        try:
            check_status_all(bad)
            ok_red = False
        except asb.SimulationError:
            pass
        q.put((rank, bool(ok_rows), bool(ok_red), len(owned)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, False, repr(e)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_allreduce_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok_rows, ok_red, n_owned in res:
        assert ok_rows, (rank, n_owned)
        assert ok_red, (rank, n_owned)
    assert sum(r[3] for r in res) == 6
