"""Per-phase cycle breakdown of the engine (ASB_PROFILE build) on a C5 shard.

    python tools/profile_phases.py [seeds] [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16682_b200 import _build  # noqa: E402

WALK = os.environ.get("ASB_PROFILE_WALK") == "1"
SWEEP = os.environ.get("ASB_PROFILE_SWEEP") == "1"
SORT = os.environ.get("ASB_PROFILE_SORT") == "1"
SPEC = os.environ.get("ASB_PROFILE_SPEC") == "1"
EPOCH = os.environ.get("ASB_PROFILE_EPOCH") == "1"
APPLY = os.environ.get("ASB_PROFILE_APPLY") == "1"
os.environ["ASB_LIB"] = os.environ.get("ASB_PROF_LIB") or _build.build_cuda(
    profile="walk" if WALK else ("sweep" if SWEEP else ("sort" if SORT else ("spec" if SPEC else ("epoch" if EPOCH else ("apply" if APPLY else True))))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_16682_b200 import _abi  # noqa: E402
from paper_2604_16682_b200.engine import DeviceBatch  # noqa: E402

PHASES = ("tick_sweep+due", "epoch_instances", "arrivals+speculate", "sort", "walk", "apply+serial")
if WALK:
    PHASES = ("w0_deplist", "w1_replay", "w2_checks", "w3_writeback", "w4_scans", "w5_arrivals")
if SORT:  # thread 0's cycles per JOB_SORT step
    PHASES = ("q0_keys", "q1_bitonic", "q2_rank_emit", "q3_barrier", "q4_tie_check", "q5_inst_lists")
    WALK = True
if APPLY:  # cycles per apply step (thread 0 inside the job; lane 0 of the main warp for 4, 5)
    PHASES = ("a0_cursor", "a1_records", "a2_writeback", "a3_loop_exit", "a4_apply_forkjoin", "a5_coupling_serial")
    WALK = True
if EPOCH:  # the main warp's cycles per epoch-event step
    PHASES = ("e0_levels_power_pending", "e1_admit_job", "e2_keys_scans", "e3_retime_start_job", "e4_final_power",
              "e5_unused")
    WALK = True
if SPEC:  # thread 0's cycles per JOB_SPEC step
    PHASES = ("p0_unused", "p1_record_loads", "p2_first_event", "p3_chain", "p4_horizon_key", "p5_unused")
    WALK = True
if SWEEP:  # slots 3, 5 are event counts per epoch, not cycles
    PHASES = ("tick_fork_cycles", "collect_due_cycles", "helper_in_tick_sweep_cycles", "bisections",
              "due_total_cycles", "admit_job_forks")
    WALK = True


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    batch, _ = bench.build_shard(0, seeds if seeds > 0 else None, os.environ.get('ASB_CONFIG', 'c5'))
    db = DeviceBatch(batch, device="cuda:0")
    db.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.run()
    e1.record()
    torch.cuda.synchronize()
    ctr = db.outputs["counters"].cpu().numpy().reshape(-1, _abi.ASB_NCOUNTERS)
    prof = ctr[:, 10:16].astype(np.float64)
    tot = prof.sum(axis=1)
    res = {
        "scenarios": int(batch.n), "step_ms": e0.elapsed_time(e1),
        "mean_cycles_per_scenario": float(tot.mean()), "max_cycles_per_scenario": float(tot.max()),
        "phase_share": {p: float(prof[:, i].sum() / tot.sum()) for i, p in enumerate(PHASES)},
        "phase_cycles_per_epoch": {p: float(prof[:, i].mean() / float(batch.scen["n_epochs"][0]))
                                   for i, p in enumerate(PHASES)},
        "batches_per_scenario": float(ctr[:, _abi.CTR["batches"]].mean()),
        "events_per_scenario": float(ctr[:, _abi.CTR["events"]].mean()),
        "ticks_per_scenario": float(ctr[:, _abi.CTR["ticks"]].mean()),
        "records_per_batch": None if WALK else float(ctr[:, _abi.CTR["retimes"]].sum() / ctr[:, _abi.CTR["batches"]].sum()),
    }
    cells = 8 if batch.n % 8 == 0 else 1
    res["per_cell_mean_max_Mcycles"] = [[round(float(tot[c::cells].mean()) / 1e6, 1), round(float(tot[c::cells].max()) / 1e6, 1)]
                                        for c in range(cells)]
    if os.environ.get("ASB_DUMP_SCEN"):
        tto = batch.traces.trace_turn_off
        tid = batch.scen["trace_id"].astype(np.int64)
        res["per_scenario"] = {"cycles": tot.tolist(), "turns": (tto[tid + 1] - tto[tid]).tolist(),
                               "events": ctr[:, _abi.CTR["events"]].tolist(), "batches": ctr[:, _abi.CTR["batches"]].tolist(),
                               "ticks": ctr[:, _abi.CTR["ticks"]].tolist()}
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
