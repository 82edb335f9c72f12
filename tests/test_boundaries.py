"""Accept/reject decisions at their boundaries (tests/boundaries.py): the
device's libm restatement (csrc/fs_glibm.h) must decide every near-tie
comparison of numpy's gamma / beta / ziggurat / lognormal code exactly as
glibc does -- the comparisons that, decided the other way, would change how
many Philox words a dirichlet_skew call or a workload stream consumes.

CPU half: fs_glibm.h compiled for the host. GPU half: the same arguments
evaluated on the device through fs_eval, beside CUDA's own libm (which flips
some of these decisions -- the reason the restatement exists).
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from boundaries import families

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODES = {"exp": 1, "log": 2, "log1p": 3, "pow": 4}


def _host_libm():
    from oracle import oracle
    return lambda fn, x, y=None: oracle.libm(fn, x, y)


@pytest.fixture(scope="module")
def fams():
    fs = families(_host_libm())
    assert {f.name for f in fs} == {"gamma_mt", "gamma_small1", "gamma_small2", "beta_johnk",
                                    "zig_exp", "zig_norm", "norm_tail", "lognormal"}
    for f in fs:
        assert f.n > 1000, (f.name, f.n)
        _, d = f.evaluate(_host_libm())
        if d.dtype == bool:  # both sides of the boundary are present
            assert d.any() and not d.all(), f.name
    return fs


def _compare(fams, libm, label):
    host = _host_libm()
    for f in fams:
        want_res, want = f.evaluate(host)
        got_res, got = f.evaluate(libm)
        for k in want_res:
            a, b = np.asarray(want_res[k]), np.asarray(got_res[k])
            bad = a.view(np.int64) != b.view(np.int64)
            assert not bad.any(), (label, f.name, k, int(bad.sum()))
        assert (got == want).all(), (label, f.name)


def test_host_restatement_decides_like_glibc(fams, tmp_path):
    so = tmp_path / "glibm_eval.so"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(so),
                    os.path.join(ROOT, "tests", "glibm", "glibm_eval.c"), "-lm"], check=True)
    lib = ctypes.CDLL(str(so))
    vp = ctypes.c_void_p
    lib.glm_eval.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_int64]

    def glm(fn, x, y=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(x if y is None else y, dtype=np.float64)
        out = np.empty_like(x)
        lib.glm_eval(CODES[fn], x.ctypes.data, y.ctypes.data, out.ctypes.data, len(x))
        return out

    _compare(fams, glm, "host fs_glibm.h")


@pytest.mark.gpu
def test_device_decides_like_glibc(fams):
    from paper_2508_03148_b200.engine import Engine
    eng = Engine(0)

    def dev(prefix):
        def f(fn, x, y=None):
            x = np.asarray(x, dtype=np.float64)
            y = x if y is None else np.asarray(y, dtype=np.float64)
            out, st = eng.eval(prefix + fn, np.stack([x, y], axis=1))
            assert (st == 0).all()
            return out[:, 0].copy()
        return f

    _compare(fams, dev(""), "device fs_glibm.h")
    # CUDA's libm on the same arguments decides some of them the other way
    host = _host_libm()
    flips = {}
    for f in fams:
        _, want = f.evaluate(host)
        _, cud = f.evaluate(dev("cuda_"))
        flips[f.name] = int((cud != want).sum())
    assert sum(flips.values()) > 0, flips
