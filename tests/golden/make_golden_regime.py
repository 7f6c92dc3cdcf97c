"""regime_classify goldens from the REFERENCE itself (build container only):
for every timeseries golden case (tests/golden/timeseries/), the reference's
run_simulation with that case's config, then its
metrics.regime_classify(result.usage_series(), capacity, window) for three
(capacity, window) choices: the run's own (capacity_tokens, sim_duration), a
halved capacity, and a window clipped to 60% of the run.

    python tests/golden/make_golden_regime.py

Output: tests/golden/regime/<case>.json.gz — per choice the thrash fraction,
the span count, a digest of the spans and (up to 2,000 spans) the spans.
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

from common import config_from_dict, digest, load_golden, reference_module, traces_from_json  # noqa: E402

ref = reference_module()
assert ref is not None, "the reference is needed to generate golden vectors"

OUT = os.path.join(HERE, "regime")
FULL = 2000


def spans_json(segments):
    return [[iid, [[a, b, bool(f)] for a, b, f in segments[iid]]] for iid in segments]


def choices(cfg):
    cap, T = float(cfg.instance.capacity_tokens), float(cfg.sim_duration)
    return [(cap, T), (cap / 2.0, T), (cap, 0.6 * T)]


def main():
    os.makedirs(OUT, exist_ok=True)
    for path in sorted(glob.glob(os.path.join(HERE, "timeseries", "*.json.gz"))):
        name = os.path.basename(path)
        with gzip.open(path, "rt", encoding="utf-8") as fh:
            t = json.load(fh)
        g = load_golden(name)
        cfg = config_from_dict(ref, t["config"], traces_from_json(ref, g["trace"]))
        res = ref.run_simulation(cfg)
        series = res.usage_series()
        out = {"name": name, "config": t["config"], "cases": []}
        for cap, win in choices(cfg):
            seg, frac = ref.regime_classify(series, cap, win)
            sj = spans_json(seg)
            n = sum(len(v) for v in seg.values())
            case = {"capacity": cap, "window": win, "fraction": frac, "n_spans": n, "digest": digest(sj)}
            if n <= FULL:
                case["spans"] = sj
            out["cases"].append(case)
        with gzip.open(os.path.join(OUT, name), "wt", encoding="utf-8") as fh:
            json.dump(out, fh, separators=(",", ":"), allow_nan=True)
        print(name, [(c["n_spans"], round(c["fraction"], 4)) for c in out["cases"]], flush=True)


if __name__ == "__main__":
    main()
