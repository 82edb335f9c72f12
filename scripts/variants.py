"""Compile-time variants of the analytic simulation kernel, built here and timed on the GPU.

  python scripts/variants.py build NAME "-DFLAG=1 ..." [NAME "FLAGS" ...]
      compiles fs_engine.cu (or the SRC=file.cu named among the flags) with the flags
      into paper_2508_03148_b200/lib/variants/NAME.so
      (linked with the standard objects of the other translation units)
  python scripts/variants.py timeenv SEEDS "FS_X=1,FS_Y=2" ...
      GPU: the default library under runtime knobs (environment), one process each
  python scripts/variants.py time [seeds] [NAME ...]
      GPU: for the default library and each variant, one process that stages the C5
      sweep and times 3 launches with CUDA events (prints one JSON line each)
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2508_03148_b200", "lib", "variants")


def build(pairs):
    from paper_2508_03148_b200 import native
    native.build()  # standard objects up to date
    os.makedirs(VDIR, exist_ok=True)
    procs = []
    for name, flags in pairs:
        obj = os.path.join(VDIR, name + ".o")
        # a token SRC=file.cu picks the translation unit to vary (default fs_engine.cu)
        src = next((f[4:] for f in flags.split() if f.startswith("SRC=")), "fs_engine.cu")
        fl = [f for f in flags.split() if not f.startswith("SRC=")]
        cmd = [native.nvcc(), *native.NVCC_FLAGS, *fl, "-c", "-o", obj,
               os.path.join(native.CSRC, src)]
        procs.append((name, obj, src, subprocess.Popen(cmd)))
    for name, obj, src, p in procs:
        if p.wait() != 0:
            raise SystemExit(f"variant {name} failed to compile")
        others = [native._obj(s) for s in native.SOURCES if s != src]
        subprocess.run([native.nvcc(), *native.ARCH, "-shared", "-o",
                        os.path.join(VDIR, name + ".so"), obj, *others], check=True)
        print("built", name)


def time_one(seeds: int):
    import torch

    from bench import lower_docs, workload_docs
    from paper_2508_03148_b200.engine import Engine
    docs = workload_docs(0, seeds, 64)
    fams = os.environ.get("FS_FAMILIES")  # e.g. "AB": the dense families of C5 only
    if fams:
        fam_of = ["A"] * 16 + ["B"] * 32 + ["C"] * 16
        docs = [d for i, d in enumerate(docs) if fam_of[i // seeds] in fams]
    low = lower_docs(docs)
    eng = Engine(0)
    eng.stage(low)
    eng.launch()
    torch.cuda.synchronize()
    res = eng.fetch(low, per_request=False)
    ok = bool((res.rows["status"] == 0).all())
    its = int(res.rows["iterations"].sum())
    ms = []
    st = torch.cuda.Stream()
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        eng.launch(st.cuda_stream)
        e.record(st)
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    again = eng.fetch(low, per_request=False)
    same = bool((again.rows["iterations"] == res.rows["iterations"]).all()
                and (again.rows["ttft"] == res.rows["ttft"]).all())
    print(json.dumps({"lib": os.environ.get("FS_ENGINE_LIB", "default"), "ms": ms,
                      "iterations": its, "all_ok": ok, "repeatable": same}), flush=True)


def time_all(seeds: int, names):
    libs = [None] + [os.path.join(VDIR, n + ".so") for n in names]
    for lib in libs:
        env = dict(os.environ)
        if lib:
            env["FS_ENGINE_LIB"] = lib
        subprocess.run([sys.executable, __file__, "_one", str(seeds)], env=env, timeout=600)


def time_envs(seeds: int, envs):
    """Runtime knobs (fs_capi.cu reads FS_* at fs_create): one process per setting."""
    for spec in [""] + list(envs):
        env = dict(os.environ)
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            env[k] = v
        print("env:", spec or "(defaults)", flush=True)
        subprocess.run([sys.executable, __file__, "_one", str(seeds)], env=env, timeout=600)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        a = sys.argv[2:]
        build(list(zip(a[0::2], a[1::2])))
    elif cmd == "time":
        seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 64
        time_all(seeds, sys.argv[3:])
    elif cmd == "timeenv":
        time_envs(int(sys.argv[2]), sys.argv[3:])
    elif cmd == "_one":
        time_one(int(sys.argv[2]))
