"""Native JSON-lines trace reader (csrc/trace_io.cpp, workload.load_trace_arrays):
same arrays as the reference-semantics loader on every accepted file, and the
same exception (type and message) on every rejected one."""

import ctypes as C

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from paper_2604_16682_b200.errors import TraceFormatError
from paper_2604_16682_b200.packing import trace_arrays_from_objects
from paper_2604_16682_b200.workload import _trace_io, load_trace_arrays


def python_arrays(path):
    return trace_arrays_from_objects(asb.load_trace(path))


def assert_same(a, b):
    for k in ("arrival", "turn_off", "prefill", "decode", "tool"):
        assert a[k].dtype == b[k].dtype, k
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k  # bit-exact, signed zeros included
    assert list(a["agent_ids"]) == list(b["agent_ids"])


def native_rc(path):
    lib = _trace_io()
    h = C.c_void_p()
    na, nt, nb, bad = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    rc = lib.asb_trace_parse(str(path).encode(), C.byref(h), C.byref(na), C.byref(nt), C.byref(nb), C.byref(bad))
    lib.asb_trace_free(h)
    return rc, bad.value


@pytest.mark.parametrize("seed", [0, 7])
def test_roundtrip_generated_trace(tmp_path, seed):
    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=2.0, duration=200.0, seed=seed))
    p = tmp_path / "t.jsonl"
    asb.save_trace(traces, str(p))
    assert native_rc(p) == (0, 0)  # the fast path handles the canonical format
    assert_same(load_trace_arrays(str(p)), python_arrays(str(p)))


def test_accepted_variations(tmp_path):
    p = tmp_path / "v.jsonl"
    p.write_text(
        '\n'
        '  {"turns": [[400, 150, 2.0], [1e2, 3.0, 0]], "x": {"a": [1, {"b": null}]}, "arrival_time": 12, '
        '"agent_id": "a\\"1"}  \n'
        '\n'
        '{"agent_id":"a2","arrival_time":0.1,"turns":[[1,1,-0.0]],"turns":[[5,6,7.25]],"extra":true}\n'
        '{"agent_id": "é", "arrival_time": -0, "turns": [[2147483647, 1, 1e-300]]}\n'
        '{"agent_id": "b", "arrival_time": 0.5E+1, "turns": [[10E0, 2, 0e-5], [3, 1, 1.25e1]]}\n',
        encoding="utf-8")
    assert native_rc(p) == (0, 0)
    assert_same(load_trace_arrays(str(p)), python_arrays(str(p)))


BAD = [
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[0, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": []}', TraceFormatError),
    ('{"agent_id": "", "arrival_time": 1.0, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": -1.0, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, -1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0}', TraceFormatError),
    ('{"agent_id": 3, "arrival_time": 1.0, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, 1.0]]', TraceFormatError),
    ('[1, 2]', TraceFormatError),
    # numbers outside the JSON grammar: json.loads rejects them, so must the fast path
    ('{"agent_id": "a", "arrival_time": 1., "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": .5, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[0400, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, 1e]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, -]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": +1.0, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, 1.0e+]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 00, "turns": [[1, 1, 1.0]]}', TraceFormatError),
    ('{"agent_id": "a", "arrival_time": 1.0, "turns": [[1, 1, 1.0]]}\n'
     '{"agent_id": "a", "arrival_time": 2.0, "turns": [[1, 1, 1.0]]}', TraceFormatError),
]


@pytest.mark.parametrize("text,exc", BAD)
def test_rejected_files_raise_like_the_reference(tmp_path, text, exc):
    p = tmp_path / "b.jsonl"
    p.write_text(text + "\n", encoding="utf-8")
    assert native_rc(p)[0] == 1
    with pytest.raises(exc) as want:
        asb.load_trace(str(p))
    with pytest.raises(exc) as got:
        load_trace_arrays(str(p))
    assert type(got.value) is type(want.value)
    assert str(got.value) == str(want.value)


@pytest.mark.parametrize("text", [
    '{"agent_id": "a", "arrival_time": NaN, "turns": [[1, 1, 1.0]]}',       # json.loads accepts NaN
    '{"agent_id": "a", "arrival_time": 1.0, "turns": [[2.5, 1, 1.0]]}',     # int(2.5) == 2
    '{"agent_id": "a", "arrival_time": 1.0, "turns": [[true, 1, 1.0]]}',    # int(True) == 1
    '{"agent_id": "\\u00e9", "arrival_time": 1.0, "turns": [[1, 1, 1.0]]}',  # unicode escape
])
def test_unusual_but_valid_files_take_the_reference_path(tmp_path, text):
    p = tmp_path / "u.jsonl"
    p.write_text(text + "\n", encoding="utf-8")
    assert native_rc(p)[0] == 1
    a, b = load_trace_arrays(str(p)), python_arrays(str(p))
    for k in ("turn_off", "prefill", "decode", "tool"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["arrival"], b["arrival"], equal_nan=True)


def test_missing_file_raises_like_the_reference(tmp_path):
    p = tmp_path / "missing.jsonl"
    with pytest.raises(FileNotFoundError):
        load_trace_arrays(str(p))


def test_trace_path_configs_pack_identically(tmp_path):
    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=1.0, duration=100.0, seed=3))
    p = tmp_path / "t.jsonl"
    asb.save_trace(traces, str(p))
    from paper_2604_16682_b200.engine import prepare_batch

    a = prepare_batch([asb.SimConfig(trace_path=str(p), instance_count=2)])
    b = prepare_batch([asb.SimConfig(traces=traces, instance_count=2)])
    for k in ("arrival", "agent_turn_off", "prefill", "decode", "tool", "arrival_order"):
        assert np.array_equal(getattr(a.traces, k), getattr(b.traces, k)), k


def test_matches_the_reference_loader_when_importable(tmp_path):
    """Against the reference's own load_trace (only where /root/reference exists)."""
    from common import reference_module

    ref = reference_module()
    if ref is None:
        pytest.skip("reference not importable here")
    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=3.0, duration=300.0, seed=11))
    p = tmp_path / "t.jsonl"
    asb.save_trace(traces, str(p))
    want = ref.load_trace(str(p))
    got = load_trace_arrays(str(p))
    assert got["agent_ids"] == [t.agent_id for t in want]
    assert np.array_equal(got["arrival"], np.array([t.arrival_time for t in want]))
    flat = [r for t in want for r in t.turns]
    assert np.array_equal(got["prefill"], np.array([r.prefill_tokens for r in flat], dtype=np.int32))
    assert np.array_equal(got["decode"], np.array([r.decode_tokens for r in flat], dtype=np.int32))
    assert np.array_equal(got["tool"], np.array([r.tool_time for r in flat]))
