"""Kernel-level checks of the tcgen05 building blocks against an fp64 numpy
reference (inputs pre-truncated to tf32 so the products are exact)."""
import numpy as np
import pytest

L = pytest.importorskip("paper_1910_02270_b200")
from paper_1910_02270_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    try:
        n = L.device_count()
    except L.Error:
        n = 0
    if n < 1:
        pytest.skip("no CUDA device")


def tf32(a):
    return (np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def test_tcgen05_mma_shapes():
    rng = np.random.default_rng(0)
    a1 = tf32(rng.standard_normal((128, 32)))
    b1 = tf32(rng.standard_normal((32, 64)))
    ah = tf32(rng.standard_normal((128, 64)))
    b2 = tf32(rng.standard_normal((64, 32)))
    a3 = tf32(np.sign(rng.standard_normal((128, 32))))
    d1 = np.zeros((128, 64), np.float32)
    d2 = np.zeros((128, 32), np.float32)
    d3 = np.zeros((128, 64), np.float32)
    _lib.check(_lib.lib.ltfb_selftest_tcgen05(a1, b1, ah, b2, a3, d1, d2, d3))
    r1 = a1.astype(np.float64) @ b1.astype(np.float64)
    r2 = ah.astype(np.float64) @ b2.astype(np.float64)
    r3 = a3.astype(np.float64) @ b2.astype(np.float64).T
    for got, ref in ((d1, r1), (d2, r2), (d3, r3)):
        err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        assert err < 1e-5, err


def test_device_adam_bit_exact_against_reference(golden):
    """nn/adam.hpp:87-122 on the device (the K7 Adam kernel; the post
    kernel's owners run the same element routine, device_common.cuh
    adam_elem) against the reference's three-step Adam vectors
    (tests/golden/nn.npz, written by the unmodified reference): p, m and v
    bit-identical after every step; a non-finite gradient changes nothing
    and raises NumericError (adam.hpp:95-102)."""
    import ctypes as C
    g = golden("nn")
    p = g["adam_p0"].astype(np.float32).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    t = C.c_uint64(0)
    for s in (1, 2, 3):
        gr = np.ascontiguousarray(g[f"adam_g{s}"], np.float32)
        _lib.check(_lib.lib.ltfb_adam_step(p, m, v, gr, p.size, C.byref(t), 1e-3, 0.9, 0.999, 1e-8, 0))
        assert t.value == s
        assert np.array_equal(p.view(np.uint32), g[f"adam_p{s}"].view(np.uint32)), s
        assert np.array_equal(m.view(np.uint32), g[f"adam_m{s}"].view(np.uint32)), s
        assert np.array_equal(v.view(np.uint32), g[f"adam_v{s}"].view(np.uint32)), s
    bad = np.ascontiguousarray(g["adam_g1"], np.float32).copy()
    bad[3] = np.inf
    before = (p.copy(), m.copy(), v.copy())
    with pytest.raises(L.NumericError):
        _lib.check(_lib.lib.ltfb_adam_step(p, m, v, bad, p.size, C.byref(t), 1e-3, 0.9, 0.999, 1e-8, 0))
    assert t.value == 3
    for a, b in zip((p, m, v), before):
        assert np.array_equal(a, b)
    # a larger blob (many CTAs, grid-stride loop) against a float64 numpy
    # restatement of the reference loop (same operation order, IEEE double)
    rng = np.random.default_rng(5)
    n = 1 << 20
    p2 = rng.standard_normal(n).astype(np.float32)
    m2 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v2 = (rng.random(n) * 1e-6).astype(np.float32)
    g2 = rng.standard_normal(n).astype(np.float32)
    t2 = C.c_uint64(6)
    ref_p, ref_m, ref_v = p2.copy(), m2.copy(), v2.copy()
    gd = g2.astype(np.float64)
    mi = 0.9 * ref_m.astype(np.float64) + (1.0 - 0.9) * gd
    vi = 0.999 * ref_v.astype(np.float64) + (1.0 - 0.999) * gd * gd
    c1, c2 = 1.0 - 0.9 ** 7, 1.0 - 0.999 ** 7
    ref_p = (ref_p.astype(np.float64) - 1e-3 * (mi / c1) / (np.sqrt(vi / c2) + 1e-8)).astype(np.float32)
    _lib.check(_lib.lib.ltfb_adam_step(p2, m2, v2, g2, n, C.byref(t2), 1e-3, 0.9, 0.999, 1e-8, 0))
    assert np.array_equal(m2, mi.astype(np.float32)) and np.array_equal(v2, vi.astype(np.float32))
    assert np.array_equal(p2, ref_p)
