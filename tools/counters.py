"""Mean engine counters per scenario (and per epoch) for a bench workload.

    python tools/counters.py [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2604_16682_b200 import _abi  # noqa: E402
from paper_2604_16682_b200.engine import DeviceBatch  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "c5"
    batch, _ = bench.build_shard(0, None, config)
    db = DeviceBatch(batch, device="cuda:0")
    db.run()
    ctr = db.outputs["counters"].cpu().numpy().reshape(-1, _abi.ASB_NCOUNTERS).astype(np.float64)
    ep = float(batch.scen["n_epochs"].mean())
    for name, k in sorted(_abi.CTR.items(), key=lambda kv: kv[1]):
        v = ctr[:, k].mean()
        print(f"{name:14s} per scenario {v:14.1f}   per epoch {v / ep:10.2f}")


if __name__ == "__main__":
    main()
