"""Streamed step vs launched step (LTFB_NO_STREAM=1), same trainer config:
prints the step records as JSON so a caller can diff the two modes, and the
per-step device time of a long run.

  python tools/stream_check.py [--steps N] [--n SAMPLES]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02270_b200 as L  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=40)
p.add_argument("--n", type=int, default=2000)
p.add_argument("--time-steps", type=int, default=0)
p.add_argument("--dims", default="paper", choices=["paper", "desk"])
a = p.parse_args()
dims = L.ModalityDims.paper_scale() if a.dims == "paper" else L.ModalityDims()
ds = L.SynthDataset(dims, a.n, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 5)
m.autoencoder_frozen = True
ids = np.arange(a.n, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=3, train_ids=ids[100:], tournament_ids=ids[:100]),
              ds, m)
t0 = time.time()
t.train_steps(a.steps)
wall = time.time() - t0
recs = [[s.step, s.epoch, int(s.skipped), s.d_loss, s.g_total, s.g_fwd, s.g_adv, s.g_cyc] for s in t.history().steps]
ev = t.eval_tournament()
out = {"stream": bool(t.stream_mode()), "wide_ctas": t.wide_info()[1], "records": recs,
       "fwd_hash": L.hex64(t.model().fwd_hash()), "disc_hash": L.hex64(t.model().disc_hash()),
       "inv_hash": L.hex64(t.model().inv_hash()), "eval": [ev.forward_mae, ev.inverse_mae, ev.combined],
       "wall_s": wall}
if a.time_steps:
    t.train_steps(10)
    t.synchronize()
    t.timer_start()
    t.train_steps_raw(a.time_steps)
    ms = t.timer_stop()
    out["ms_per_step"] = ms / a.time_steps
print(json.dumps(out))
