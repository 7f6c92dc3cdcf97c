"""Where and when each scenario of a shard ran (ASB_PROFILE_PLACEMENT build):
per-scenario SM id, start/end (globaltimer ns) and duration, and how the
duration depends on the number of teams co-resident on its SM.

    ASB_LIB=<placement build> python tools/placement.py [config] [out.json]
"""
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_16682_b200 import _abi  # noqa: E402
from paper_2604_16682_b200.engine import DeviceBatch  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "c5"
    batch, _ = bench.build_shard(0, None, config)
    db = DeviceBatch(batch, device="cuda:0")
    db.run()
    db.run()
    torch.cuda.synchronize()
    ctr = db.outputs["counters"].cpu().numpy().reshape(-1, _abi.ASB_NCOUNTERS)
    sm, t0, t1 = ctr[:, 10], ctr[:, 11], ctr[:, 12]
    dur = (t1 - t0) / 1e6
    per_sm = defaultdict(list)
    for s in range(batch.n):
        per_sm[int(sm[s])].append(s)
    res = {"n": int(batch.n), "sms": len(per_sm), "makespan_ms": float((t1.max() - t0.min()) / 1e6),
           "dur_mean_ms": float(dur.mean()), "dur_max_ms": float(dur.max()),
           "by_residents": {}}
    groups = defaultdict(list)
    for smid, ss in per_sm.items():
        for s in ss:
            groups[len(ss)].append(dur[s])
    for k, v in sorted(groups.items()):
        res["by_residents"][k] = {"scenarios": len(v), "mean_ms": float(np.mean(v)), "max_ms": float(np.max(v))}
    ticks = ctr[:, _abi.CTR["ticks"]].astype(np.float64)
    res["corr_dur_ticks"] = float(np.corrcoef(dur, ticks)[0, 1])
    res["start_spread_ms"] = float((t0.max() - t0.min()) / 1e6)
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        turns = ctr[:, _abi.CTR["turns"]].astype(np.float64)
        json.dump({**res, "sm": sm.tolist(), "dur": dur.tolist(), "ticks": ticks.tolist(), "turns": turns.tolist(),
                   "t0_ms": ((t0 - t0.min()) / 1e6).tolist(), "t1_ms": ((t1 - t0.min()) / 1e6).tolist()},
                  open(sys.argv[2], "w"))


if __name__ == "__main__":
    main()
