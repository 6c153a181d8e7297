#!/usr/bin/env python3
"""Dev driver: one desk-dims trainer whose tournament slice is C5-sized
(--tour-rows, rendered on the device); times --evals tournament evaluations
(host wall incl. sync) -- for ncu / timing of the eval kernels at C5 scale."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1910_02270_b200 as L  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tour-rows", type=int, default=225000)
p.add_argument("--evals", type=int, default=5)
a = p.parse_args()
dims = L.ModalityDims()
n = a.tour_rows + 4096
ds = L.SynthDataset(dims, n, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 5)
m.autoencoder_frozen = True
ids = np.arange(n, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=3, prefetch_depth=0, train_ids=ids[a.tour_rows:],
                              tournament_ids=ids[:a.tour_rows]), ds, m)
t.synchronize()
t.eval_tournament()
t0 = time.perf_counter()
for _ in range(a.evals):
    e = t.eval_tournament()
dt = (time.perf_counter() - t0) / a.evals
print(f"eval_tournament {a.tour_rows} rows: {dt * 1e3:.3f} ms per call (host wall, incl. sync)", e)
