"""In-tree native builds (nvcc for sm_100a; gcc/g++ for test infrastructure).

* ``paper_2604_16682_b200/_lib/libagentsim_b200.so`` — the product: the C ABI
  of include/agentsim_b200.h over the sm_100a kernels (engine.cu,
  unit_ops.cu).  Built with ``--fmad=false`` because the reference is
  Python, which never contracts multiply-add, and parity is bit-exact.
* ``oracle/build/liboracle.so`` — the serial C oracle (tests/bench CPU legs).
* ``tests/native/build/libhost_engine.so`` — 1-lane CPU build of the engine
  core, a test harness for the batching logic.
"""

from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_16682_b200")
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libagentsim_b200.so")
PROF_LIB_PATH = os.path.join(LIB_DIR, "libagentsim_b200_prof.so")
WPROF_LIB_PATH = os.path.join(LIB_DIR, "libagentsim_b200_wprof.so")
DEBUG_LIB_PATH = os.path.join(LIB_DIR, "libagentsim_b200_debug.so")
TRACE_IO_LIB = os.path.join(LIB_DIR, "libagentsim_trace_io.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "build", "liboracle.so")
HOST_ENGINE_LIB = os.path.join(ROOT, "tests", "native", "build", "libhost_engine.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _tmp(target: str) -> str:
    """Per-process temporary output: concurrent builds (one per rank under
    torchrun) never write the same file; the final rename is atomic."""
    return f"{target}.{os.getpid()}.tmp"


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def build_cuda(force: bool = False, verbose: bool = False, profile: bool | str = False) -> str:
    """The product library; ``profile=True`` builds the phase-timing variant
    (-DASB_PROFILE, counters[10..15]) used only by tools/profile_phases.py."""
    srcs = [os.path.join(CSRC, f) for f in ("engine.cu", "unit_ops.cu")]
    deps = srcs + [os.path.join(CSRC, "engine_core.h"), os.path.join(ROOT, "include", "agentsim_b200.h")]
    target = {"walk": WPROF_LIB_PATH, "debug": DEBUG_LIB_PATH,
              "sweep": os.path.join(LIB_DIR, "libagentsim_b200_sprof.so"),
              "sort": os.path.join(LIB_DIR, "libagentsim_b200_qprof.so"),
              "spec": os.path.join(LIB_DIR, "libagentsim_b200_pprof.so"),
              "epoch": os.path.join(LIB_DIR, "libagentsim_b200_eprof.so"),
              "apply": os.path.join(LIB_DIR, "libagentsim_b200_aprof.so")}.get(profile) if isinstance(profile, str) else (
        PROF_LIB_PATH if profile else LIB_PATH)
    if force or _stale(target, deps):
        os.makedirs(LIB_DIR, exist_ok=True)
        cmd = [_nvcc(), *NVCC_FLAGS, "-shared", "-o", _tmp(target), *srcs]
        if profile == "debug":
            cmd.insert(1, "-DASB_DEBUG_TRACE")
        elif profile:
            cmd.insert(1, "-DASB_PROFILE")
        if profile == "walk":
            cmd.insert(1, "-DASB_PROFILE_WALK")
        if profile == "sweep":
            cmd.insert(1, "-DASB_PROFILE_SWEEP")
        if profile == "sort":
            cmd.insert(1, "-DASB_PROFILE_SORT")
        if profile == "spec":
            cmd.insert(1, "-DASB_PROFILE_SPEC")
        if profile == "epoch":
            cmd.insert(1, "-DASB_PROFILE_EPOCH")
        if profile == "apply":
            cmd.insert(1, "-DASB_PROFILE_APPLY")
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
        os.replace(_tmp(target), target)
    return target


def build_trace_io(force: bool = False) -> str:
    """Host-side native JSON-lines trace reader (csrc/trace_io.cpp)."""
    src = os.path.join(CSRC, "trace_io.cpp")
    if force or _stale(TRACE_IO_LIB, [src]):
        os.makedirs(LIB_DIR, exist_ok=True)
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", _tmp(TRACE_IO_LIB), src])
        os.replace(_tmp(TRACE_IO_LIB), TRACE_IO_LIB)
    return TRACE_IO_LIB


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "des_oracle.c")
    deps = [src, os.path.join(ROOT, "include", "agentsim_b200.h")]
    if force or _stale(ORACLE_LIB, deps):
        os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
        _run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
              "-o", _tmp(ORACLE_LIB), src, "-lm"])
        os.replace(_tmp(ORACLE_LIB), ORACLE_LIB)
    return ORACLE_LIB


def build_host_engine(force: bool = False) -> str:
    src = os.path.join(ROOT, "tests", "native", "host_engine.cpp")
    deps = [src, os.path.join(CSRC, "engine_core.h"), os.path.join(ROOT, "include", "agentsim_b200.h")]
    if force or _stale(HOST_ENGINE_LIB, deps):
        os.makedirs(os.path.dirname(HOST_ENGINE_LIB), exist_ok=True)
        _run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
              "-o", _tmp(HOST_ENGINE_LIB), src])
        os.replace(_tmp(HOST_ENGINE_LIB), HOST_ENGINE_LIB)
    return HOST_ENGINE_LIB


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_trace_io(force)
    build_cuda(force, profile=True)
    build_cuda(force, profile="walk")
    build_oracle(force)
    build_host_engine(force)


if __name__ == "__main__":
    build_all(force=True)
    print("built", LIB_PATH, ORACLE_LIB, HOST_ENGINE_LIB)
