"""regime_classify (metrics.py:72-109): the host mirror over oracle results
and the device kernel (asb_regime_classify) over the engine's own timeseries
rows, both against the REFERENCE's regime_classify of its own usage series
(tests/golden/make_golden_regime.py), for three (capacity, window) choices
per case.  Exact: spans and the thrash fraction."""

import glob
import gzip
import json
import os

import pytest

import paper_2604_16682_b200 as asb
from common import GOLDEN, config_from_dict, digest, load_golden, results_via, traces_from_json
from oracle.oracle import run_oracle
from paper_2604_16682_b200.engine import DeviceBatch, prepare_batch

REG = os.path.join(GOLDEN, "regime")
CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(REG, "*.json.gz")))


def load(name):
    with gzip.open(os.path.join(REG, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


def config(r):
    g = load_golden(r["name"])
    return config_from_dict(asb, r["config"], traces_from_json(asb, g["trace"]))


def check(case, seg, frac):
    sj = [[iid, [[a, b, bool(f)] for a, b, f in seg[iid]]] for iid in seg]
    assert frac == case["fraction"]
    assert sum(len(v) for v in seg.values()) == case["n_spans"]
    if "spans" in case:
        assert sj == case["spans"]
    assert digest(sj) == case["digest"]


def test_fixtures_present():
    assert len(CASES) >= 30


@pytest.mark.parametrize("name", CASES)
def test_host_mirror_on_oracle_series(name):
    r = load(name)
    (res,), _ = results_via(run_oracle, [config(r)], timeseries=True)
    for case in r["cases"]:
        seg, frac = asb.regime_classify(res.usage_series(), case["capacity"], case["window"])
        check(case, seg, frac)


@pytest.mark.gpu
def test_device_regime_classify_all_cases(cuda_device):
    """Every golden case in one batch: the engine writes the timeseries rows,
    the kernel classifies them on the device."""
    regs = [load(n) for n in CASES]
    batch = prepare_batch([config(r) for r in regs])
    dev = DeviceBatch(batch, device="cuda:0", timeseries=True)
    dev.run()
    for k in range(3):
        caps = [r["cases"][k]["capacity"] for r in regs]
        wins = [r["cases"][k]["window"] for r in regs]
        out = dev.regime_classify(capacity=caps, window=wins)
        for r, (seg, frac) in zip(regs, out):
            check(r["cases"][k], seg, frac)


@pytest.mark.gpu
def test_device_regime_classify_rejects_bad_window(cuda_device):
    r = load(CASES[0])
    dev = DeviceBatch(prepare_batch([config(r)]), device="cuda:0", timeseries=True)
    dev.run()
    with pytest.raises(asb.ConfigurationError, match="window"):
        dev.regime_classify(window=[0.0])
    nots = DeviceBatch(prepare_batch([config(r)]), device="cuda:0")
    with pytest.raises(asb.ConfigurationError, match="timeseries"):
        nots.regime_classify()
