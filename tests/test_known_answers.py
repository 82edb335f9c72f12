"""Known-answer values the reference's own tests pin,
checked against this repo's host mirror, the C oracle and -- where the value is
on the device path -- the CUDA engine.

Reference tests: test_analytic.py:31-36 (linear FLOP term), test_topology.py:
107-110 (KV bytes/token), 135-138 (ring all-reduce), test_routing_moe.py:28-30
(top_k == E saturation), test_core.py:166-169 (ns rounding half to even).
"""

import numpy as np
import pytest

from paper_2508_03148_b200.topology import ModelConfig, kv_bytes_per_token


def test_linear_flop_term_hand_value():
    from oracle import oracle
    lib = oracle.load()
    peak, bw, ovh = 312e12, 2.0e12, 5.0
    t = lib.fso_linear_us(1024, 4096, 4096, peak, bw, ovh, 2)
    flop_term_us = 2 * 1024 * 4096 * 4096 / 312e12 * 1e6
    assert flop_term_us == pytest.approx(110.1, abs=0.1)
    assert t == pytest.approx(ovh + flop_term_us, rel=1e-6)


def test_kv_bytes_per_token_hand_arithmetic():
    m = ModelConfig(num_layers=28, d_model=3584, d_ff=18944, num_query_heads=28,
                    num_kv_heads=4, head_dim=128, dtype_bytes=2)
    assert kv_bytes_per_token(m) == 57_344
    unit = ModelConfig(num_layers=1, d_model=1, d_ff=1, num_query_heads=1, num_kv_heads=1,
                       head_dim=1, dtype_bytes=2)
    assert kv_bytes_per_token(unit) == 4


def test_collectives_hand_values():
    from oracle import oracle
    lib = oracle.load()
    # 2*alpha + 2*(1 MB * 1/2)/beta = 10 us + 10 us
    assert lib.fso_collective(1, 1e6, 2, 5e-6, 100e9) == pytest.approx(20e-6)
    for kind in (0, 1, 2):
        assert lib.fso_collective(kind, 1e6, 1, 5e-6, 100e9) == 0.0
    assert lib.fso_collective(0, 1e6, 4, 5e-6, 100e9) < lib.fso_collective(1, 1e6, 4, 5e-6, 100e9)


def test_topk_equals_e_saturates_oracle():
    from oracle import oracle
    for policy in ("uniform", "dirichlet_skew"):
        c, st = oracle.route(37, 8, 8, policy, 5)
        assert st == 0 and c == [37] * 8


@pytest.mark.gpu
def test_topk_equals_e_saturates_device(engine):
    for policy in ("uniform", "dirichlet_skew"):
        counts, st = engine.route_tokens([37, 0, 5], [5, 6, 7], 8, 8, policy)
        assert (st == 0).all()
        assert counts.tolist() == [[37] * 8, [0] * 8, [5] * 8]


@pytest.mark.gpu
def test_invalid_topk_and_alpha_on_device(engine):
    _, st = engine.route_tokens([10], [1], 8, 9, "uniform")
    assert st.tolist() == [8]  # FS_ERR_INVALID_TOPK (routing.py:76-77)
    _, st = engine.route_tokens([10], [1], 8, 2, "dirichlet_skew", 0.0)
    assert st.tolist() == [5]  # RoutingError: dirichlet_skew needs alpha > 0


def test_python_sum_of_identical_layers_is_one_rounded_product():
    """execute_batch (csrc/fs_sim.cuh) replaces the L-step Neumaier sum of L
    identical layer totals (cluster.py:345) by fl(L * x). CPython's sum() catches
    every step's rounding error exactly in its compensation (a multiple of ulp(x)
    below 2^53 ulp for L < 2^26), so the two are the same double."""
    import math
    import random
    rng = random.Random(2508)
    xs = [0.1, 1 / 3, 2 / 3, 0.30000000000000004, 123456.789, 5e-324 * 12345]
    xs += [rng.lognormvariate(5, 4) for _ in range(3000)]
    xs += [math.ldexp(rng.random() + 0.5, rng.randint(-60, 60)) for _ in range(3000)]
    for x in xs:
        for L in (1, 2, 3, 7, 32, 61, 80, 127, 128, rng.randint(1, 5000)):
            assert sum([x] * L) == L * x, (x, L)


_TIE_PROBE = r"""
import hashlib, numpy as np
rng = np.random.default_rng(0)
out = []
for trial in range(600):
    E = int(rng.choice([8, 16, 60, 256])); k = int(rng.integers(1, min(E, 17)))
    keys = rng.random(E); order = np.argsort(keys, kind="stable")
    keys[order[k]] = keys[order[k - 1]]          # k-th and (k+1)-th smallest tie exactly
    out.append(tuple(sorted(np.argpartition(keys[None, :], k - 1, axis=1)[0, :k].tolist())))
print(hashlib.sha256(repr(out).encode()).hexdigest())
"""


def test_argpartition_boundary_ties_depend_on_numpy_simd_dispatch():
    """Why an exact tie at the top-k boundary is FS_ERR_ROUTING_TIE rather than an
    answer: routing.py:110 picks the experts with np.argpartition, whose choice
    between two equal keys is not a property of the reference but of numpy's
    SIMD dispatch on the host CPU (the same rows give different experts with the
    AVX2+ kernels and with the baseline ones). A tie has probability ~E^2 2^-54
    per row; the engine reports it instead of guessing one host's answer."""
    import os
    import subprocess
    import sys
    base = dict(os.environ)
    simd = subprocess.run([sys.executable, "-c", _TIE_PROBE], capture_output=True, text=True,
                          env=base)
    off = dict(base, NPY_DISABLE_CPU_FEATURES="AVX2 FMA3 AVX512F AVX512CD AVX512_SKX "
                                             "AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR")
    scalar = subprocess.run([sys.executable, "-c", _TIE_PROBE], capture_output=True, text=True,
                            env=off)
    if simd.returncode or scalar.returncode:
        pytest.skip("numpy SIMD dispatch cannot be switched here")
    if simd.stdout == scalar.stdout:
        pytest.skip("this host's numpy has no SIMD argpartition kernel")
    assert simd.stdout != scalar.stdout
