#!/usr/bin/env python3
"""Small driver for ncu / compute-sanitizer: one paper-dims trainer on
cuda:0, a few warm-up steps, then --steps timed-free steps (and optionally
one tournament evaluation)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1910_02270_b200 as L  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=8)
p.add_argument("--dims", default="paper")
p.add_argument("--n", type=int, default=1200)
p.add_argument("--wide-kernel", type=int, default=0)
p.add_argument("--eval", action="store_true")
a = p.parse_args()
dims = L.ModalityDims.paper_scale() if a.dims == "paper" else L.ModalityDims()
ds = L.synthetic_dataset(dims, a.n, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 5)
m.autoencoder_frozen = True
ids = np.arange(a.n, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=3, train_ids=ids[64:], tournament_ids=ids[:64],
                              wide_kernel=a.wide_kernel), ds, m)
t.train_steps(a.steps)
if a.eval:
    print(t.eval_tournament())
print("steps", t.step(), "last", t.history().steps[-1])
