"""Wall time of one ``run_simulation`` call on the C2 golden case, with and
without timeseries rows (the serial-loop instantiation vs the batched
engine), next to the reference's own wall time recorded in the fixture.

    python tools/time_timeseries.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2604_16682_b200 as asb  # noqa: E402
from common import config_from_dict, load_golden, traces_from_json  # noqa: E402

g = load_golden("c2.json.gz")
cfg = config_from_dict(asb, g["config"], traces_from_json(asb, g["trace"]))
asb.run_simulation(cfg, timeseries=False)  # warm-up (library load, context)
for ts in (False, True, True):
    t0 = time.perf_counter()
    r = asb.run_simulation(cfg, timeseries=ts)
    dt = time.perf_counter() - t0
    print(f"timeseries={ts} rows={len(r.timeseries)} wall_s={dt:.3f} reference_wall_s={g['ref_wall_s']:.1f}")
