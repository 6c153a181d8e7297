"""compute-sanitizer target: one paper-dim training step graph-free pass
(k_row_h, k_wide_tc: TMA gather4 + tcgen05 + mbarrier rings + grid barrier;
k_post_small: 16-CTA cluster, DSMEM, bulk copies), then one tournament
round (k_eval_small, k_eval_tc over two 128-row blocks, k_eval_finalize)
and one AE step. Run as

  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LTFB_NO_GRAPH", "1")
import paper_1910_02270_b200 as L  # noqa: E402

dims = L.ModalityDims.paper_scale()
n, n_tour = 400, 140
ds = L.synthetic_dataset(dims, n, sampling_seed=3, spec_seed=1)
model = L.make_cyclegan(dims, L.SurrogateArch(), 5)
p = L.AutoencoderPretrainer(model, ds.y, batch_size=128)
print("ae step loss", p.step(L.ae_batch_rows(5, n, 128, 1)))
del p
model.autoencoder_frozen = True
ids = np.arange(n, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=2, train_ids=ids[n_tour:],
                              tournament_ids=ids[:n_tour]), ds, model)
assert t.wide_info()[0] == 2 and t.eval_info(0) == 2
t.train_steps(2)
t._set_incoming(model.blobs["fwd"], model.blobs["inv"])
print("round", t._decide())
print("steps", [(s.d_loss, s.g_total) for s in t.history().steps])
