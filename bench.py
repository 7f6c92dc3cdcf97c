#!/usr/bin/env python
"""bench.py — agent-ticks/s of the batched scenario engine on B200.

Workload (default, BASELINE.json configs[4] "C5"): the
Monte-Carlo sweep, 4096 scenarios = 512 seeds x 8 cells {router
context_aware|round_robin} x {controller context_aware|off} x {SLO tau 20|35};
each scenario 16 instances x ~10k agents (WorkloadSpec arrival_rate=10000/3600,
3600 s), 3600 control epochs.  The whole job fits one B200, so N=1 runs all of
it; at N GPUs rank r takes seeds [512r/N, 512(r+1)/N) (strong scaling: the job
is fixed, N=8 is the 512-scenario-per-GPU split BASELINE names).  One step =
every scenario of the rank's share run to completion (engine kernel +
per-scenario stats + stats fold), plus the NCCL allreduce of the 8-double
stats vector when N > 1.  `--config c5` keeps the fixed 512-scenario shard per
GPU (weak scaling).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config c5full|c5|c3|c4]

--config selects another BASELINE.json workload for the same line format:
c3 = the DVFS sweep (8 fixed levels x 4 capacities x 64 seeds per GPU, 1
instance x ~1k agents, 12500 epochs), c4 = the 100k-agent thrashing regime
(one scenario, 64 instances).  The driver's headline is the default (c5full).

`--impl reference` times the CPU restatement of the reference (oracle/,
serial C DES, OpenMP over scenarios on all host cores) on the same shard.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "agent-ticks/sec (batched scenarios)"
UNIT = "agent-ticks/s"
HBM_FALLBACK = 6538.6


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--config", choices=tuple(CONFIGS), default="c5full",
                   help="workload (BASELINE.json configs): c5full = the headline Monte-Carlo sweep, all 4096 "
                        "scenarios split over the GPUs (strong scaling); c5 = a fixed 512-scenario shard per GPU")
    p.add_argument("--seeds-per-gpu", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- workload


C3_MHZ = (660.0, 810.0, 900.0, 1035.0, 1185.0, 1350.0, 1515.0, 1680.0)
C3_CAPS = (250_000, 500_000, 750_000, 1_000_000)


def base_config(config: str):
    """The experiment every cell of a BASELINE sweep applies to."""
    import paper_2604_16682_b200 as asb

    if config == "c5":
        return asb.SimConfig(workload=workload_spec("c5", 0), instance_count=16, sim_duration=3600.0)
    if config == "c3":
        return asb.SimConfig(workload=workload_spec("c3", 0), instance_count=1, sim_duration=12500.0,
                             instance=asb.InstanceConfig(frequency_table=asb.default_frequency_table(mhz=C3_MHZ)))
    if config == "c4":
        return asb.SimConfig(workload=workload_spec("c4", 0), instance_count=64, sim_duration=3600.0,
                             controller=asb.ControllerConfig(thrash_avoidance=False))
    raise ValueError(f"unknown config {config!r}")


def sweep_axes(config: str, seeds: list[int]) -> dict:
    """The BASELINE sweep as axes of the sweep driver (sweep.ALL_AXES)."""
    if config == "c5":  # 8 cells: router x controller x SLO target, per seed
        return {"slo_target": [20.0, 35.0], "policy": ["context_aware", "round_robin"],
                "variant": ["context_aware", "off"], "seed": seeds}
    if config == "c3":  # 8 fixed levels x 4 capacities, per seed
        return {"level_mhz": list(C3_MHZ), "capacity": list(C3_CAPS), "seed": seeds}
    if config == "c4":
        return {"seed": [11 + s for s in seeds]}
    raise ValueError(f"unknown config {config!r}")


# workload table: seeds per GPU (weak scaling: rank r takes seeds [r*k, (r+1)*k)), generator, cells
CONFIGS = {
    "c5": {"seeds_per_gpu": 64, "desc": "C5 Monte-Carlo sweep shard: 512 scenarios/GPU (64 seeds x 8 cells "
                                        "{ctx-aware,round-robin} router x {ctx-aware,off} controller x tau {20,35}), "
                                        "16 instances x ~10k agents, 3600 s",
           "instances": 16, "epochs": 3600, "sim_duration_s": 3600.0},
    "c3": {"seeds_per_gpu": 64, "desc": "C3 DVFS sweep: 2048 scenarios/GPU (64 seeds x 8 fixed frequency levels "
                                        "x 4 capacities {250k,500k,750k,1M}), 1 instance x ~1k agents, 12500 s",
           "instances": 1, "epochs": 12500, "sim_duration_s": 12500.0},
    "c4": {"seeds_per_gpu": 1, "desc": "C4 long-tail thrashing regime: 1 scenario/GPU, ~100k agents with "
                                       "prefill growth 20/turn, 64 instances, context-aware without thrash avoidance, "
                                       "3600 s",
           "instances": 64, "epochs": 3600, "sim_duration_s": 3600.0},
    # the whole C5 job (4096 scenarios) split over the N GPUs: strong scaling,
    # N=1 runs all of it on one GPU
    "c5full": {"seeds_total": 512, "desc": "C5 Monte-Carlo sweep, whole job: 4096 scenarios (512 seeds x 8 cells) "
                                          "split over the GPUs, 16 instances x ~10k agents, 3600 s",
               "instances": 16, "epochs": 3600, "sim_duration_s": 3600.0, "same_as": "c5"},
}


def scaling_of(config: str) -> str:
    return "strong" if "seeds_total" in CONFIGS[config] else "weak"


def workload_spec(config: str, seed: int):
    """The WorkloadSpec of one seed of a BASELINE config."""
    import paper_2604_16682_b200 as asb

    if config == "c5":
        return asb.WorkloadSpec(arrival_rate=10000 / 3600, duration=3600.0, seed=seed)
    if config == "c3":
        return asb.WorkloadSpec(arrival_rate=0.08, duration=12500.0, seed=seed)
    if config == "c4":
        return asb.WorkloadSpec(arrival_rate=100000 / 3600, duration=3600.0, seed=seed, prefill_growth_per_turn=20)
    raise ValueError(f"unknown config {config!r}")


def build_shard(rank: int, seeds_per_gpu: int | None = None, config: str = "c5"):
    """This rank's share of a BASELINE sweep, built through the public API:
    sweep.sweep_cells over the sweep's axes (seed included), apply_cell to
    the base experiment, prepare_batch (the reference's generate_workload
    draws as CSR arrays, one trace per seed shared by its cells)."""
    from paper_2604_16682_b200 import sweep
    from paper_2604_16682_b200.engine import prepare_batch

    cfg = CONFIGS[config]
    if "seeds_total" in cfg:  # strong scaling: the job's seeds split over the ranks
        world = int(os.environ.get("WORLD_SIZE", "1"))
        total = seeds_per_gpu or cfg["seeds_total"]
        seeds = list(range(total * rank // world, total * (rank + 1) // world))
    else:
        k = seeds_per_gpu or cfg["seeds_per_gpu"]
        seeds = list(range(rank * k, (rank + 1) * k))
    config = cfg.get("same_as", config)
    base = base_config(config)
    configs = [sweep.apply_cell(base, c) for c in sweep.sweep_cells(sweep_axes(config, seeds))]
    batch = prepare_batch(configs)
    batch.configs = configs
    return batch, seeds


def alg_bytes(batch, counters) -> float:
    """B_alg = 20 N_ticks + 112 N_turns + 128 N_instance_epochs."""
    from paper_2604_16682_b200 import _abi

    ctr = counters.reshape(-1, _abi.ASB_NCOUNTERS)
    ticks = float(ctr[:, _abi.CTR["ticks"]].sum())
    turns = float(ctr[:, _abi.CTR["turns"]].sum())
    inst_epochs = float((batch.scen["n_instances"].astype(np.int64) * batch.scen["n_epochs"]).sum())
    return 20.0 * ticks + 112.0 * turns + 128.0 * inst_epochs


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (SURVEY/BASELINE measured copy bandwidth)"


def ncu_traffic(config: str):
    """dram bytes per launch of the engine from the committed ncu capture of
    the same workload (profiles/ncu_engine_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_engine_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        if d.get("config", "c5") != config:
            return None, None
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU legs


def cpu_run(batch, threads: int = 0):
    from oracle.oracle import run_oracle

    timing = {}
    host, stats = run_oracle(batch, decisions=False, turn_log=False, threads=threads, timing=timing)
    return host, stats, timing["seconds"]


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # pip install --target of /root/reference/pkg (travels)
PYREF_SCEN_PER_WORKER = {"c5": 1, "c3": 3}  # ~5-10 s of reference time per worker; C4 (70 s) is not sampled


def trace_arrays_of(batch, s: int) -> dict:
    """The CSR trace scenario s runs, sliced from the packed pool."""
    tp = batch.traces
    t = int(batch.scen[s]["trace_id"])
    a0, a1 = int(tp.trace_agent_off[t]), int(tp.trace_agent_off[t + 1])
    t0, t1 = int(tp.trace_turn_off[t]), int(tp.trace_turn_off[t + 1])
    return {"arrival": tp.arrival[a0:a1], "turn_off": tp.agent_turn_off[a0:a1 + 1] - t0,
            "prefill": tp.prefill[t0:t1], "decode": tp.decode[t0:t1], "tool": tp.tool[t0:t1]}


def _pyref_one(job):
    """One scenario through the REFERENCE's own run_simulation (baseline/_ref),
    on the same trace arrays and cell config the GPU ran."""
    cell, arrs, ref_dir = job
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import agentsim as ref

    from paper_2604_16682_b200.adapter import convert
    from paper_2604_16682_b200.engine import agent_ticks_closed_form

    arrival, off = arrs["arrival"], arrs["turn_off"]
    pre, dec, tool = arrs["prefill"].tolist(), arrs["decode"].tolist(), arrs["tool"].tolist()
    traces = [ref.AgentTrace(f"a{i:06d}", float(arrival[i]),
                             tuple(ref.TurnRecord(pre[j], dec[j], tool[j]) for j in range(off[i], off[i + 1])))
              for i in range(arrival.size)]
    cfg = convert(cell, ref)
    cfg.workload, cfg.seed, cfg.traces = None, None, traces  # the same trace, generation not timed
    t0 = time.perf_counter()
    res = ref.run_simulation(cfg)
    sec = time.perf_counter() - t0
    e = cfg.controller.epoch_length
    k = 0
    while k * e < cfg.sim_duration:
        k += 1
    arr = np.array([a.arrival_time for a in res.agents], dtype=np.float64)
    comp = np.array([np.nan if a.completion_time is None else a.completion_time for a in res.agents])
    return sec, agent_ticks_closed_form(arr, comp, e, k)


def python_reference(batch, config: str):
    """The reference's own Python path (agentsim.run_simulation from
    baseline/_ref) on a bounded sample of the shard, one process per host
    core, as the reference's sweep runs cells (cli.py:161-188)."""
    per = PYREF_SCEN_PER_WORKER.get(config)
    if per is None or not os.path.isdir(os.path.join(REF_DIR, "agentsim")):
        why = "reference not installed in baseline/_ref" if per is not None else \
            f"{config}: one reference scenario takes minutes; not sampled"
        return {"unavailable": why}
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    workers = max(1, min(cpu_cores(), 64, batch.n // per))
    n = workers * per
    picks = [round(q * batch.n / n) for q in range(n)]  # spread over the shard's cells and seeds
    jobs = [(batch.configs[s], trace_arrays_of(batch, s), REF_DIR) for s in picks]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        out = list(ex.map(_pyref_one, jobs))
    wall = time.perf_counter() - t0
    sec = sum(o[0] for o in out)
    ticks = sum(o[1] for o in out)
    return {"value": ticks / sec * workers, "unit": UNIT, "cores": workers, "kind": "python-reference",
            "per_core": ticks / sec,
            "sample": f"{n} scenarios spread evenly over the shard ({per} per process, {workers} processes, "
                      f"{wall:.1f} s wall): agentsim.run_simulation from baseline/_ref (the unmodified reference), "
                      "value = per-core rate x processes; trace object construction excluded"}


def reference_arm(args, world, rank):
    """`--impl reference`: the CPU restatement of the reference on all host cores."""
    if rank != 0:
        return
    from paper_2604_16682_b200 import _abi, _build

    _build.build_oracle()
    batch, seeds = build_shard(0, args.seeds_per_gpu, args.config)
    cores = cpu_cores()
    for _ in range(args.warmup):
        cpu_run(batch, cores)
    times, ticks = [], 0.0
    for _ in range(args.steps):
        host, _, sec = cpu_run(batch, cores)
        times.append(sec)
        ticks = float(host["counters"].reshape(-1, _abi.ASB_NCOUNTERS)[:, _abi.CTR["ticks"]].sum())
    sec = sum(times) / len(times)
    # the whole job at N GPUs is N shards; the CPU arm times one shard per step
    value = ticks / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": scaling_of(args.config),
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(batch, seeds, world, args.config),
        "arm": f"CPU: serial C restatement of the reference (oracle/des_oracle.c), OpenMP over scenarios, {cores} threads",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"one {args.config.upper()} shard per step: {batch.n} scenarios (seeds {seeds[0]}-{seeds[-1]})"},
        "python_reference": python_reference(batch, CONFIGS[args.config].get("same_as", args.config)),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(batch, seeds, world, config="c5"):
    cfg = CONFIGS[config]
    n_agents = batch.total_agents / max(batch.n, 1)
    tbytes = sum(getattr(batch.traces, k).nbytes for k in ("arrival", "agent_turn_off", "prefill", "decode", "tool"))
    return {
        "workload": cfg["desc"], "name": config,
        "scenarios_per_gpu": batch.n, "seeds_per_gpu": len(seeds), "instances": cfg["instances"],
        "mean_agents_per_scenario": round(n_agents, 1), "sim_duration_s": cfg["sim_duration_s"],
        "epochs": cfg["epochs"],
        "parallelism": f"scenario-sharded x{world}",
        "l2": f"inputs larger than L2: {tbytes / 2**20:.0f} MiB trace pool + workspace per GPU, no flush",
    }


# ----------------------------------------------------------------------------- GPU arm


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch

    from paper_2604_16682_b200 import _abi, _build
    from paper_2604_16682_b200.engine import DeviceBatch
    from paper_2604_16682_b200.parallel import allreduce_stats

    _build.build_cuda()
    # ASB_DIST_BACKEND=gloo: a functional check of the multi-rank path on a
    # box with fewer GPUs than ranks (ranks share devices; timings are not
    # scaling numbers).  The benchmark itself is one rank per GPU over NCCL.
    backend = os.environ.get("ASB_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist
    batch, seeds = build_shard(rank, args.seeds_per_gpu, args.config)
    db = DeviceBatch(batch, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev0=None, ev1=None):
        if ev0 is not None:
            ev0.record(stream)
        torch.ops.agentsim_b200.run_scenarios(db.scen, db.traces, db.tables, db.out_list, db.workspace,
                                              batch.launch_instances, batch.total_agents, batch.total_ring, batch.max_levels)
        if ev1 is not None:
            ev1.record(stream)
        torch.ops.agentsim_b200.scenario_stats(db.scen, db.out_list, db.stats)
        torch.ops.agentsim_b200.reduce_stats(db.stats, db.outputs["counters"], batch.n, db.red)
        if pg is not None:
            allreduce_stats(db.red)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    if pg is not None:
        pg.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        t0.record(stream)
        for k in range(args.steps):
            step(*evs[k])
        t1.record(stream)
        torch.cuda.synchronize(dev)
    if pg is not None:
        pg.barrier()
    total_ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in evs]
    host_ctr = db.outputs["counters"].cpu().numpy()
    red = db.red.cpu().numpy()
    ticks_local = float(host_ctr.reshape(-1, _abi.ASB_NCOUNTERS)[:, _abi.CTR["ticks"]].sum())
    ms_per_step = total_ms / args.steps
    if pg is not None:
        t = torch.tensor([ms_per_step, ticks_local], dtype=torch.float64, device=dev)
        mx = t.clone()
        pg.all_reduce(mx, op=pg.ReduceOp.MAX)
        pg.all_reduce(t)
        ms_max, ticks_all = float(mx[0]), float(t[1])
    else:
        ms_max, ticks_all = ms_per_step, ticks_local
    value = ticks_all / (ms_max / 1e3)

    # roofline of the dominant kernel (the engine) from its own CUDA events
    b_alg = alg_bytes(batch, host_ctr)
    kern_s = (sum(kern_ms) / len(kern_ms)) / 1e3
    achieved = b_alg / kern_s / 1e9
    peak, peak_src = hbm_peak()
    traffic, _ = ncu_traffic(args.config)

    # end-to-end through the public API with host buffers: every step copies
    # its inputs from pinned host memory and reads its results back.  Two
    # device input sets and a copy stream pipeline the steps: step k+1's
    # inputs upload while step k computes (each step still waits for its own
    # upload, and an input set is only overwritten after the step using it)
    e2e = None
    if not args.no_e2e:
        host_in = [torch.from_numpy(np.ascontiguousarray(batch.scen.view(np.uint8))).pin_memory()]
        host_in += [torch.from_numpy(np.ascontiguousarray(getattr(batch.traces, k))).pin_memory()
                    for k in _abi.TRACE_FIELDS]
        host_in += [torch.from_numpy(np.ascontiguousarray(getattr(batch.tables, k))).pin_memory()
                    for k in _abi.TABLE_FIELDS]
        sets = [[db.scen, *db.traces, *db.tables],
                [torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host_in]]
        nt, ntab = len(_abi.TRACE_FIELDS), len(_abi.TABLE_FIELDS)
        h2d = sum(t.numel() * t.element_size() for t in host_in)
        out_stats = torch.empty(db.stats.shape, dtype=db.stats.dtype).pin_memory()
        out_red = torch.empty(db.red.shape, dtype=db.red.dtype).pin_memory()
        d2h = out_stats.numel() + out_red.numel() * 8
        copy_stream = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]

        def upload(k):
            dst = sets[k % 2]
            with torch.cuda.stream(copy_stream):
                if k >= 2:
                    copy_stream.wait_event(used[k % 2])  # step k-2 is done with this set
                for d_t, h_t in zip(dst, host_in):
                    d_t.copy_(h_t, non_blocking=True)
                copied[k % 2].record(copy_stream)

        def step_on(k):
            inp = sets[k % 2]
            scen, traces, tables = inp[0], inp[1:1 + nt], inp[1 + nt:1 + nt + ntab]
            stream.wait_event(copied[k % 2])
            torch.ops.agentsim_b200.run_scenarios(scen, traces, tables, db.out_list, db.workspace,
                                                  batch.launch_instances, batch.total_agents, batch.total_ring, batch.max_levels)
            torch.ops.agentsim_b200.scenario_stats(scen, db.out_list, db.stats)
            used[k % 2].record(stream)
            torch.ops.agentsim_b200.reduce_stats(db.stats, db.outputs["counters"], batch.n, db.red)
            if pg is not None:
                allreduce_stats(db.red)
            out_stats.copy_(db.stats, non_blocking=True)
            out_red.copy_(db.red, non_blocking=True)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if pg is not None:
            pg.barrier()
        e0.record(stream)
        copy_stream.wait_event(e0)
        upload(0)
        for k in range(args.steps):
            if k + 1 < args.steps:
                upload(k + 1)
            step_on(k)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = e0.elapsed_time(e1) / args.steps
        if pg is not None:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_ms = float(t[0])
        e2e = {"value": ticks_all / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "pipelining": "two device input sets: step k+1's upload overlaps step k's compute"}

    cpu = None
    parity = None
    pyref = None
    if rank == 0 and not args.no_cpu_baseline:
        _build.build_oracle()
        cores = cpu_cores()
        host_ref, stats_ref, sec = cpu_run(batch, cores)
        ctr_ref = host_ref["counters"].reshape(-1, _abi.ASB_NCOUNTERS)
        cpu = {"value": float(ctr_ref[:, _abi.CTR["ticks"]].sum()) / sec, "unit": UNIT, "cores": cores,
               "kind": "port",
               "sample": f"the full shard ({batch.n} scenarios, {sec:.1f} s wall on {cores} threads): serial C "
                         "restatement of the reference DES (oracle/des_oracle.c), OpenMP over scenarios"}
        got = {k: t.cpu().numpy() for k, t in db.outputs.items()}
        keys = [k for k in _abi.AGENT_OUT] + [k for k in _abi.INST_OUT]
        same = all(np.array_equal(got[k], host_ref[k], equal_nan=got[k].dtype.kind == "f") for k in keys)
        a = got["counters"].reshape(-1, _abi.ASB_NCOUNTERS)[:, :9]
        same = same and np.array_equal(a, ctr_ref[:, :9])
        parity = f"{'bit-exact' if same else 'MISMATCH'} vs oracle on all {batch.n} scenarios of the timed shard"
        if world > 1:
            parity += " (rank 0's shard)"
            cpu["sample"] = "rank 0's shard: " + cpu["sample"]
        pyref = python_reference(batch, CONFIGS[args.config].get("same_as", args.config))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": scaling_of(args.config),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: the reference's generate_workload stream (same numpy default_rng draws, CSR arrays)",
            "config": config_block(batch, seeds, world, args.config),
            "arm": f"B200 x{world}" + (": NCCL allreduce of the stats vector" if world > 1 else ""),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "asb_engine_kernel", "kernel_ms": kern_s * 1e3,
                         "alg_bytes_per_launch": b_alg, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "python_reference": pyref,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": 4 * args.steps,
            "parity": parity,
            "stats": {k: float(v) for k, v in zip(_abi.RED, red)},
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
