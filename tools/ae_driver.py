#!/usr/bin/env python3
"""Dev driver: autoencoder pre-training steps at paper dims (timing / ncu)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02270_b200 as L  # noqa: E402

dims = L.ModalityDims.paper_scale()
ds = L.synthetic_dataset(dims, 1000, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 3)
p = L.AutoencoderPretrainer(m, ds.y)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
draws = L.ae_batch_rows(1, 1000, 128, n)
for s in range(3):
    p.step(draws[s])
t = time.perf_counter()
for s in range(3, n):
    loss = p.step(draws[s])
print(f"ae step {(time.perf_counter() - t) / (n - 3) * 1e3:.3f} ms (host wall incl. sync), loss {loss:.6f}")
