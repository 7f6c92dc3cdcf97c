"""The C-ABI library loads (no GPU needed) and exports every symbol the
header declares; the ctypes/numpy mirrors match the C struct layouts."""

import ctypes
import os
import re

from common import ROOT
from paper_2604_16682_b200 import _abi, _build, _native


def header_functions():
    text = open(os.path.join(ROOT, "include", "agentsim_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|size_t)\s+(asb_\w+)\(", text, flags=re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    _build.build_cuda()
    lib = _native.lib()
    names = header_functions()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match_header():
    lib = _native.lib()
    buf = (ctypes.c_int64 * 8)()
    assert lib.asb_struct_sizes(buf) == 8
    assert list(buf) == _abi.struct_sizes()
    assert lib.asb_abi_version() == 1


def test_workspace_size_is_monotone():
    lib = _native.lib()
    a = lib.asb_workspace_bytes(4, 1000, 16000)
    b = lib.asb_workspace_bytes(4, 2000, 32000)
    assert 0 < a < b


def test_launch_instances_declares_fixed_counts():
    """asb_run_scenarios' max_instances: -m when every scenario has m
    instances (fixed-count kernels), else the maximum (include/agentsim_b200.h)."""
    import dataclasses

    import paper_2604_16682_b200 as asb
    from paper_2604_16682_b200.engine import prepare_batch

    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.2, duration=30.0, seed=1))
    base = asb.SimConfig(traces=traces, instance_count=4, sim_duration=40.0)
    assert prepare_batch([base, base]).launch_instances == -4
    assert prepare_batch([base, dataclasses.replace(base, instance_count=1)]).launch_instances == 4
    assert prepare_batch([dataclasses.replace(base, instance_count=1)]).launch_instances == -1


def test_engine_limits():
    """127 instances and 64 DVFS levels are the engine's limits
    (ASB_MAX_INSTANCES / ASB_MAX_LEVELS); one more raises ConfigurationError
    before any launch, like the reference's own validation errors."""
    import dataclasses

    import pytest

    import paper_2604_16682_b200 as asb
    from paper_2604_16682_b200.engine import prepare_batch

    traces = asb.generate_workload(asb.WorkloadSpec(arrival_rate=0.2, duration=30.0, seed=1))
    t64 = asb.default_frequency_table(mhz=tuple(600.0 + 10.0 * k for k in range(64)))
    ok = asb.SimConfig(traces=traces, instance_count=127, sim_duration=40.0,
                       instance=asb.InstanceConfig(frequency_table=t64))
    b = prepare_batch([ok])
    assert b.max_levels == 64 and b.launch_instances == -127
    with pytest.raises(asb.ConfigurationError):
        prepare_batch([dataclasses.replace(ok, instance_count=128)])
    t65 = asb.default_frequency_table(mhz=tuple(600.0 + 10.0 * k for k in range(65)))
    with pytest.raises(asb.ConfigurationError):
        prepare_batch([dataclasses.replace(ok, instance=asb.InstanceConfig(frequency_table=t65))])
