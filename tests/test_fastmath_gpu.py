"""The fused kernel's branch-free IEEE division and sqrt (pointwise.cuh div_fast/sqrt_fast)
against numpy's correctly rounded a / b and sqrt: bit-identical wherever they do not ask
for the slow path, on random, wide-exponent and edge inputs."""
import ctypes as C

import numpy as np
import pytest

from paper_2211_13295_b200 import hydro

pytestmark = pytest.mark.gpu


def _inputs():
    r = np.random.default_rng(5)
    n = 1 << 20
    a = r.uniform(-4, 4, n) * 2.0 ** r.integers(-60, 60, n)
    b = r.uniform(-4, 4, n) * 2.0 ** r.integers(-60, 60, n)
    wide_a = r.uniform(0.5, 1, 1 << 16) * 2.0 ** r.integers(-1070, 1020, 1 << 16)
    wide_b = r.uniform(0.5, 1, 1 << 16) * 2.0 ** r.integers(-1070, 1020, 1 << 16)
    edge = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308,
                     1.7976931348623157e308, 1e-300, 1e300, 3.0, 7.0, 1.0 / 3.0])
    ea, eb = np.meshgrid(edge, edge)
    a = np.concatenate([a, wide_a, ea.ravel(), np.abs(a[:1000])])
    b = np.concatenate([b, wide_b, eb.ravel(), np.abs(b[:1000])])
    return np.ascontiguousarray(a), np.ascontiguousarray(b)


def test_fast_division_and_sqrt_match_ieee():
    lib = hydro.load_library()
    a, b = _inputs()
    n = a.size
    q, s = np.zeros(n), np.zeros(n)
    qs, ss = np.zeros(n, np.int32), np.zeros(n, np.int32)
    P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    lib.hc_selftest_fastmath.argtypes = [C.c_void_p] * 2 + [C.c_size_t] + [C.c_void_p] * 4
    assert lib.hc_selftest_fastmath(P(a), P(b), n, P(q), P(qs), P(s), P(ss)) == 0
    with np.errstate(all="ignore"):
        want_q = a / b
        want_s = np.sqrt(a)
    okq = qs == 0
    oks = ss == 0
    assert okq.mean() > 0.9 and oks.sum() > 100000
    assert (q[okq].view(np.uint64) == want_q[okq].view(np.uint64)).all()
    assert (s[oks].view(np.uint64) == want_s[oks].view(np.uint64)).all()
