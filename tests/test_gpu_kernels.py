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
