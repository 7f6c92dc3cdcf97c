"""Wall time of the public batch API on the C5 shard (512 scenarios = 64
seeds x 8 cells, 16 instances x ~10k agents, 3600 s), the way a user calls
it: SimConfig objects with a WorkloadSpec each, run_simulation_batch(...,
columnar=True), then per-scenario results on demand.

    python tools/time_batch_api.py [seeds] [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_16682_b200 as asb  # noqa: E402
from paper_2604_16682_b200.engine import BatchResult, DeviceBatch, build_results, prepare_batch  # noqa: E402


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    from paper_2604_16682_b200 import sweep

    base = bench.base_config("c5")
    cfgs = [sweep.apply_cell(base, c) for c in sweep.sweep_cells(bench.sweep_axes("c5", list(range(seeds))))]
    out = {"scenarios": len(cfgs)}
    t0 = time.perf_counter()
    batch = prepare_batch(cfgs)
    out["prepare_batch_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    db = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=False)
    torch.cuda.synchronize()
    out["upload_alloc_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    db.run()
    torch.cuda.synchronize()
    out["device_run_s"] = time.perf_counter() - t0  # first launch: module load + 1.4 GB of decision rows
    t0 = time.perf_counter()
    db.run()
    torch.cuda.synchronize()
    out["device_rerun_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    host, stats = db.download()
    out["download_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = BatchResult(batch, host, stats, cfgs, None)
    out["batch_result_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for s in range(8):
        res[s]
    out["objects_per_scenario_s"] = (time.perf_counter() - t0) / 8
    # the whole public call, end to end (fresh)
    t0 = time.perf_counter()
    res2 = asb.run_simulation_batch(cfgs, decisions=True, turn_log=False, columnar=True)
    out["run_simulation_batch_columnar_s"] = time.perf_counter() - t0
    ticks = float(res2.counter("ticks").sum())
    out["ticks"] = ticks
    out["e2e_ticks_per_s"] = ticks / out["run_simulation_batch_columnar_s"]
    out["objects_all_scenarios_est_s"] = out["objects_per_scenario_s"] * len(cfgs)
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
