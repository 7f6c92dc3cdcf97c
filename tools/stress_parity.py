"""Randomised parity stress on the GPU: many random configuration batches on
every team shape against the C oracle (bit-exact).  A kernel that fails to
finish is caught by the host watchdog thread (exit code 3).

    python tools/stress_parity.py [n_batches] [configs_per_batch] [first_seed]

Every 4th batch also runs in timeseries mode (rows compared byte for byte);
every 3rd batch widens its scenarios to 17-64 instances (the MAXM=64
kernels, and the JOB_DEPS team job on the multi-warp teams).
"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import dataclasses  # noqa: E402
import random  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from common import array_outputs_equal  # noqa: E402
from oracle.oracle import run_oracle  # noqa: E402
from paper_2604_16682_b200.engine import DeviceBatch, prepare_batch  # noqa: E402
from test_host_engine import random_configs  # noqa: E402


def main():
    n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    per = int(sys.argv[2]) if len(sys.argv) > 2 else 48
    seed0 = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
    state = {"t": time.time(), "what": ""}

    def watchdog():
        while True:
            time.sleep(2)
            if time.time() - state["t"] > 120:
                print("HANG:", state["what"], flush=True)
                os._exit(3)

    threading.Thread(target=watchdog, daemon=True).start()
    fails = 0
    for b in range(n_batches):
        team = ("solo", "quad", "big")[b % 3]
        os.environ["ASB_TEAM"] = team
        seed = seed0 + b
        state["t"], state["what"] = time.time(), f"batch {b} seed {seed} team {team}"
        cfgs = random_configs(seed, per)
        wide = b % 3 == 2
        if wide:
            rng = random.Random(seed)
            cfgs = [dataclasses.replace(c, instance_count=rng.choice([17, 33, 48, 64])) for c in cfgs]
        ts = b % 4 == 3
        batch = prepare_batch(cfgs)
        dev = DeviceBatch(batch, device="cuda:0", decisions=True, turn_log=True, timeseries=ts)
        dev.run()
        torch.cuda.synchronize()
        got, gst = dev.download()
        want, wst = run_oracle(batch, timeseries=ts)
        keys = [k for k in want if k not in ("agent_off", "inst_off", "dec_off", "turn_off", "ts_off", "timeseries")]
        diff = array_outputs_equal(want, got, keys=keys)
        if ts and diff is None:
            for s_ in range(batch.n):
                o, n = int(batch.ts_off[s_]), int(want["ts_count"][s_])
                if got["timeseries"][o: o + n].tobytes() != want["timeseries"][o: o + n].tobytes():
                    diff = f"timeseries rows of scenario {s_}"
                    break
        ok = diff is None and all(np.array_equal(gst[f], wst[f], equal_nan=True) for f in gst.dtype.names)
        fails += not ok
        print(f"batch {b:3d} seed {seed} team {team:4s} scen {batch.n:3d}{' wide' if wide else ''}{' ts' if ts else ''}: "
              f"{'ok' if ok else 'MISMATCH ' + str(diff)[:200]}",
              flush=True)
    print(f"done: {n_batches - fails}/{n_batches} batches bit-exact")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
