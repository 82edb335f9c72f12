"""Build of the CUDA engine library (nvcc, sm_100a) into paper_2508_03148_b200/lib/.

Each translation unit is compiled to its own object (in parallel, and only when
it or a header changed), then linked into libfrontier_b200.so. Device code
never calls across translation units, so no relocatable device code is needed.
"""

from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libfrontier_b200.so")
OBJ = os.path.join(HERE, "lib", "obj")
SOURCES = ["fs_engine.cu", "fs_engine_learned.cu", "fs_engine_longrow.cu", "fs_engine_dense.cu",
           "fs_engine_comoe.cu",
           "fs_metrics.cu",
           "fs_costs.cu", "fs_capi.cu"]
HEADERS = ["fs_device.cuh", "fs_route.cuh", "fs_engine.h", "fs_forest.cuh", "fs_sim.cuh",
           "fs_dirichlet.cuh", "fs_ziggurat.h", "fs_glibm.h", "fs_glibm_tables.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH, "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # no FMA contraction: fp64 must follow Python's operation order
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, h) for h in HEADERS]
    hs.append(os.path.join(os.path.dirname(HERE), "include", "frontier_b200.h"))
    return hs


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def stale() -> bool:
    deps = [os.path.join(CSRC, f) for f in SOURCES] + _headers()
    return _stale(LIB, deps)


def _compile(src: str, verbose: bool, extra: list[str]) -> str:
    out = _obj(src)
    if not _stale(out, [os.path.join(CSRC, src)] + _headers()) and not extra:
        return out
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", out + ".tmp", os.path.join(CSRC, src)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


HOSTPY_SRC = os.path.join(CSRC, "fs_hostpy.c")


def hostpy_path() -> str:
    import sysconfig
    return os.path.join(HERE, "lib", "_fs_host" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_hostpy(force: bool = False) -> str:
    """The CPython host helper (csrc/fs_hostpy.c; gcc, in-tree next to the engine)."""
    import sysconfig
    target = hostpy_path()
    if not force and not _stale(target, [HOSTPY_SRC]):
        return target
    os.makedirs(os.path.dirname(target), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
                    "-o", target + ".tmp", HOSTPY_SRC], check=True)
    os.replace(target + ".tmp", target)
    return target


def load_hostpy():
    """The _fs_host module, or None when it is not built (pure-Python fallback:
    the same dictionaries, slower)."""
    import importlib.util
    path = hostpy_path()
    if not os.path.exists(path):
        return None
    spec = importlib.util.spec_from_file_location("_fs_host", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: str | None = None) -> str:
    if out is None and not extra:
        build_hostpy(force)
    target = out or LIB
    if not force and not extra and not stale() and os.path.exists(target):
        return target
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, extra or []), SOURCES))
    tmp = target + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, target)
    return target
