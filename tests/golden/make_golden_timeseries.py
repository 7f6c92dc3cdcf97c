"""Generate the timeseries golden fixtures from the REFERENCE itself (run in
the build container, where /root/reference exists).

    python tests/golden/make_golden_timeseries.py

For every golden case that carries its full trace (tests/golden/*.json.gz:
the known-answer cases, the random configurations, the tie storms, C1, C2)
the reference is run with one of three record intervals (the default 1.0,
0.7, 2.5 in turn) and its ``SimulationResult.timeseries`` (``_mark_row``,
engine.py:403-429) is frozen in the canonical form of
tests/common.canonical_timeseries: every row for series of up to 4,000 rows,
else a SHA-256 digest plus the row count and the first 200 rows.
Output: tests/golden/timeseries/<case>.json.gz.
"""

from __future__ import annotations

import glob
import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from common import (canonical_timeseries, config_from_dict, digest, load_golden, reference_module,  # noqa: E402
                    traces_from_json)

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"

OUT = os.path.join(HERE, "timeseries")
INTERVALS = (None, 0.7, 2.5)
FULL_ROWS = 4000


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sorted(os.path.basename(p) for p in glob.glob(os.path.join(HERE, "*.json.gz")))
    k = 0
    for name in names:
        g = load_golden(name)
        if "trace" not in g:
            continue
        d = dict(g["config"])
        ri = INTERVALS[k % len(INTERVALS)]
        k += 1
        if ri is not None:
            d["record_interval"] = ri
        res = ref.run_simulation(config_from_dict(ref, d, traces_from_json(ref, g["trace"])))
        rows = canonical_timeseries(res)
        payload = {"name": name, "config": d, "n_rows": len(rows), "digest": digest(rows)}
        if len(rows) <= FULL_ROWS:
            payload["rows"] = rows
        else:
            payload["head"] = rows[:200]
        path = os.path.join(OUT, name)
        with gzip.open(path, "wt", encoding="utf-8") as fh:
            json.dump(payload, fh, separators=(",", ":"), allow_nan=True)
        print(f"{name:24s} interval={ri} rows={len(rows):7d} {os.path.getsize(path) / 1024:8.1f} KiB", flush=True)


if __name__ == "__main__":
    main()
