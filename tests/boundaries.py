"""Decision-boundary arguments for every libm-dependent branch on the device path
(test infrastructure for tests/test_boundaries.py).

numpy's distributions take accept/reject decisions on libm results
(numpy 2.3.5 random/src/distributions/distributions.c, restated in
csrc/fs_dirichlet.cuh and oracle/fs_oracle.c):

  gamma_mt      random_standard_gamma, shape >= 1 (Marsaglia-Tsang):
                log(U) < 0.5*X*X + b*(1 - V + log(V))
  gamma_small1  shape < 1, U <= 1 - shape:    pow(U, 1/shape) <= V
  gamma_small2  shape < 1, U >  1 - shape:    Y = -log((1-U)/shape);
                pow(1 - shape + shape*Y, 1/shape) <= V + Y
  beta_johnk    random_beta, a, b <= 1:       pow(U, 1/a) + pow(V, 1/b) <= 1
  zig_exp       random_standard_exponential wedge:
                (fe[i-1] - fe[i])*u + fe[i] < exp(-x)
  zig_norm      random_standard_normal wedge: ... < exp(-0.5*x*x)
  norm_tail     normal tail (idx 0): yy + yy > xx*xx, xx = -inv_r*log1p(-u1),
                yy = -log1p(-u2)
  lognormal     workload lengths (reference workload.py, numpy lognormal then
                rounding): rint(exp(mu + sigma*z)) at k + 1/2

A uniformly random seed puts a comparison within a few ulp of its boundary
with probability ~1e-15, so searching seeds for such calls is not feasible.
Instead each case here is built AT the boundary: the free uniform (on numpy's
2^-53 grid, or the argument itself) is solved for from the other operands and
its neighbours are taken, and only cases whose two sides lie within 4 ulp of
each other are kept. Every decision is a fixed expression of IEEE operations
(compiled with -fmad=false on the device) over libm results, so the device and
the host decide alike exactly when their libm results agree on these
arguments; the tests check both, and count how many decisions CUDA's own libm
would have flipped.
"""

from __future__ import annotations

import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ZIG_H = os.path.join(ROOT, "paper_2508_03148_b200", "csrc", "fs_ziggurat.h")
GRID = 2.0 ** -53
NOR_INV_R = 0.27366123732975827203338247596


def zig_tables() -> dict[str, np.ndarray]:
    src = open(ZIG_H).read()
    out = {}
    for name, body in re.findall(r"fs_zig_(\w+)\[256\] = \{(.*?)\};", src, re.S):
        vals = np.array([int(v, 16) for v in re.findall(r"0x([0-9a-f]+)ull", body)], np.uint64)
        out[name] = vals if name in ("ke", "ki") else vals.view(np.float64)
    return out


def _grid_neighbours(u_star: np.ndarray, span: int = 4):
    """numpy uniforms (k * 2^-53) around u_star: offsets -span..span."""
    k0 = np.floor(u_star / GRID)
    ks = k0[:, None] + np.arange(-span, span + 1)[None, :]
    return ks * GRID


def _within(a: np.ndarray, b: np.ndarray, ulps: int = 4) -> np.ndarray:
    sp = np.maximum(np.spacing(np.abs(a)), np.spacing(np.abs(b)))
    return np.isfinite(a) & np.isfinite(b) & (np.abs(a - b) <= ulps * sp)


class Family:
    """One decision: `compute(libm)` makes the libm calls the decision reads, in
    the order the distribution makes them (an argument may depend on an earlier
    result) and returns {name: result}; `decide(res)` gives the decisions."""

    def __init__(self, name, compute, decide, n):
        self.name, self.compute, self.decide, self.n = name, compute, decide, n

    def evaluate(self, libm):
        res = self.compute(libm)
        return res, np.asarray(self.decide(res))


def _calls(**calls):
    """compute() for independent calls: name=(fn, x, y)."""
    return lambda libm: {k: libm(fn, x, y) for k, (fn, x, y) in calls.items()}


def families(libm, n: int = 4000, seed: int = 20251017) -> list[Family]:
    """Build the boundary cases. `libm(fn, x, y)` is the host library the
    boundaries are solved with (glibc, as numpy links it)."""
    rng = np.random.default_rng(seed)
    z = zig_tables()
    out = []

    # gamma_mt: shapes >= 1 (dirichlet alpha >= 1 and beta's gamma legs)
    shape = np.concatenate([1.0 + rng.random(n) * 3.0, rng.choice([1.3, 2.0, 5.0, 16.0], n)])
    b = shape - 1.0 / 3.0
    c = 1.0 / np.sqrt(9 * b)
    X = rng.normal(size=2 * n) * 1.5
    V = 1.0 + c * X
    keep = V > 0
    b, X, V = b[keep], X[keep], V[keep]
    V3 = V * V * V
    logV = libm("log", V3)
    rhs = 0.5 * X * X + b * (1.0 - V3 + logV)
    ok = rhs < 0
    b, X, V3, rhs = b[ok], X[ok], V3[ok], rhs[ok]
    U = _grid_neighbours(libm("exp", rhs))
    rep = U.shape[1]
    U, b, X, V3, rhs = (U.ravel(), np.repeat(b, rep), np.repeat(X, rep), np.repeat(V3, rep),
                        np.repeat(rhs, rep))
    good = (U > 0) & (U < 1) & ~(U < 1.0 - 0.0331 * (X * X) * (X * X))  # squeeze failed
    good &= _within(libm("log", U), rhs)
    U, b, X, V3 = U[good], b[good], X[good], V3[good]
    out.append(Family(
        "gamma_mt", _calls(logU=("log", U, U), logV=("log", V3, V3)),
        lambda r, b=b, X=X, V3=V3: r["logU"] < 0.5 * X * X + b * (1.0 - V3 + r["logV"]),
        len(U)))

    # gamma_small1: X = U^(1/shape) <= V, V an exponential variate
    sh = 0.02 + rng.random(n) * 0.97
    Vx = rng.exponential(size=n) * 0.5
    U = _grid_neighbours(libm("pow", Vx, sh))
    rep = U.shape[1]
    U, sh, Vx = U.ravel(), np.repeat(sh, rep), np.repeat(Vx, rep)
    inv = 1.0 / sh
    good = (U > 0) & (U <= 1.0 - sh) & _within(libm("pow", U, inv), Vx)
    U, inv, Vx = U[good], inv[good], Vx[good]
    out.append(Family("gamma_small1", _calls(X=("pow", U, inv)),
                      lambda r, Vx=Vx: r["X"] <= Vx, len(U)))

    # gamma_small2: U > 1 - shape; V placed at the boundary X - Y, +-4 ulp
    sh = 0.05 + rng.random(n) * 0.9
    U = 1.0 - sh + rng.random(n) * sh
    U = np.floor(U / GRID) * GRID
    ok = (U > 1.0 - sh) & (U < 1.0)
    sh, U = sh[ok], U[ok]
    arg = (1 - U) / sh
    Y = -libm("log", arg, arg)
    inv = 1.0 / sh
    Xv = libm("pow", 1.0 - sh + sh * Y, inv)
    Vb = Xv - Y
    offs = np.arange(-4, 5)
    Vs = Vb[:, None] + offs[None, :] * np.spacing(np.abs(Vb))[:, None]
    rep = len(offs)
    Vs = Vs.ravel()
    arg, sh, inv = np.repeat(arg, rep), np.repeat(sh, rep), np.repeat(inv, rep)
    good = Vs >= 0
    Vs, arg, sh, inv = Vs[good], arg[good], sh[good], inv[good]

    def small2(libm, arg=arg, sh=sh, inv=inv):
        logA = libm("log", arg, arg)
        Y = -logA
        return {"Y": Y, "X": libm("pow", 1.0 - sh + sh * Y, inv)}

    out.append(Family("gamma_small2", small2, lambda r, Vs=Vs: r["X"] <= Vs + r["Y"], len(Vs)))

    # beta_johnk: X + Y <= 1 with Y placed on the boundary through V
    a = 0.02 + rng.random(n) * 0.98
    bb = 0.02 + rng.random(n) * 0.98
    Uj = np.floor(rng.random(n) / GRID) * GRID
    Xj = libm("pow", Uj, 1.0 / a)
    ok = (Xj < 1) & (Uj > 0)
    a, bb, Uj, Xj = a[ok], bb[ok], Uj[ok], Xj[ok]
    Vj = _grid_neighbours(libm("pow", 1.0 - Xj, bb))
    rep = Vj.shape[1]
    Vj = Vj.ravel()
    a, bb, Uj, Xj = (np.repeat(a, rep), np.repeat(bb, rep), np.repeat(Uj, rep),
                     np.repeat(Xj, rep))
    good = (Vj > 0) & (Vj < 1) & _within(Xj + libm("pow", Vj, 1.0 / bb), np.ones_like(Vj))
    a, bb, Uj, Vj = a[good], bb[good], Uj[good], Vj[good]
    out.append(Family("beta_johnk", _calls(X=("pow", Uj, 1.0 / a), Y=("pow", Vj, 1.0 / bb)),
                      lambda r: r["X"] + r["Y"] <= 1.0, len(Uj)))

    # ziggurat wedges
    for name, kk, ww, ff, mant, f in (("zig_exp", "ke", "we", "fe", 2 ** 53, lambda x: -x),
                                      ("zig_norm", "ki", "wi", "fi", 2 ** 52,
                                       lambda x: -0.5 * x * x)):
        idx = rng.integers(1, 256, n)
        lo = z[kk][idx].astype(np.float64)
        ri = np.floor(lo + rng.random(n) * (mant - lo))
        x = ri * z[ww][idx]
        arg = f(x)
        e = libm("exp", arg)
        f0, f1 = z[ff][idx - 1], z[ff][idx]
        ustar = (e - f1) / (f0 - f1)
        ok = (ustar > 0) & (ustar < 1)
        # one ulp of exp's result moves u by ulp(e) / (f0 - f1) >> 2^-53
        step = np.maximum(1.0, np.round(np.spacing(e[ok]) / (f0 - f1)[ok] / GRID))
        u = (np.floor(ustar[ok] / GRID)[:, None]
             + step[:, None] * np.arange(-4, 5)[None, :]) * GRID
        rep = u.shape[1]
        u = u.ravel()
        arg, e, f0, f1 = (np.repeat(arg[ok], rep), np.repeat(e[ok], rep), np.repeat(f0[ok], rep),
                          np.repeat(f1[ok], rep))
        lhs = (f0 - f1) * u + f1
        good = (u >= 0) & (u < 1) & _within(lhs, e)
        lhs, arg = lhs[good], arg[good]
        out.append(Family(name, _calls(e=("exp", arg, arg)),
                          lambda r, lhs=lhs: lhs < r["e"], len(lhs)))

    # normal tail: yy + yy > xx*xx
    u1 = np.floor(rng.random(n) / GRID) * GRID
    xx = -NOR_INV_R * libm("log1p", -u1)
    ystar = 0.5 * xx * xx
    u2 = _grid_neighbours(-np.expm1(-ystar))
    rep = u2.shape[1]
    u2 = u2.ravel()
    u1r = np.repeat(u1, rep)
    yy = -libm("log1p", -u2)
    xxr = -NOR_INV_R * libm("log1p", -u1r)
    good = (u2 >= 0) & (u2 < 1) & _within(yy + yy, xxr * xxr)
    u1r, u2 = u1r[good], u2[good]
    out.append(Family(
        "norm_tail", _calls(a=("log1p", -u1r, -u1r), y=("log1p", -u2, -u2)),
        lambda r: (-r["y"]) + (-r["y"]) > (-NOR_INV_R * r["a"]) * (-NOR_INV_R * r["a"]),
        len(u2)))

    # lognormal lengths: rint(exp(t)) at half-integers
    k = rng.integers(1, 20000, n).astype(np.float64) + 0.5
    t = libm("log", k)
    offs = np.arange(-4, 5)
    ts = (t[:, None] + offs[None, :] * np.spacing(t)[:, None]).ravel()
    out.append(Family("lognormal", _calls(e=("exp", ts, ts)),
                      lambda r: np.rint(r["e"]), len(ts)))
    return out
