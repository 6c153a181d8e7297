import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1910_02270_b200 as L
from paper_1910_02270_b200 import _lib
def tf32(a):
    return (np.ascontiguousarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
rng = np.random.default_rng(0)
a1 = tf32(rng.standard_normal((128, 32))); b1 = tf32(rng.standard_normal((32, 64)))
ah = tf32(rng.standard_normal((128, 64))); b2 = tf32(rng.standard_normal((64, 32)))
a3 = tf32(np.sign(rng.standard_normal((128, 32))))
d1 = np.zeros((128, 64), np.float32); d2 = np.zeros((128, 32), np.float32); d3 = np.zeros((128, 64), np.float32)
rc = _lib.lib.ltfb_selftest_tcgen05(a1, b1, ah, b2, a3, d1, d2, d3)
print("rc", rc, _lib.lib.ltfb_last_error())
r1 = a1.astype(np.float64) @ b1; r2 = ah.astype(np.float64) @ b2; r3 = a3.astype(np.float64) @ b2.T
np.set_printoptions(precision=3, suppress=True, linewidth=200)
for name, got, ref in (("d1", d1, r1), ("d2", d2, r2), ("d3", d3, r3)):
    err = np.abs(got - ref)
    print(name, "maxabs got", np.abs(got).max(), "ref", np.abs(ref).max(), "maxerr", err.max(),
          "rows ok", int((err.max(1) < 1e-3 * np.abs(ref).max()).sum()), "cols ok", int((err.max(0) < 1e-3*np.abs(ref).max()).sum()))
    print(" got[0,:8]", got[0, :8]); print(" ref[0,:8]", ref[0, :8])
    print(" got[1,:8]", got[1, :8]); print(" ref[1,:8]", ref[1, :8])
    print(" got[8,:8]", got[8, :8]); print(" ref[8,:8]", ref[8, :8])
