"""Compare generic SIMT vs tcgen05 wide pass step records at desk/paper dims."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1910_02270_b200 as L
dims_name = sys.argv[1] if len(sys.argv) > 1 else "desk"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dims = L.ModalityDims.paper_scale() if dims_name == "paper" else L.ModalityDims()
n = 600
ds = L.synthetic_dataset(dims, n, sampling_seed=1, spec_seed=1, samples_per_file=100)
ids = np.arange(n, dtype=np.uint32)
res = {}
for k in (1, 2, 3):
    m = L.make_cyclegan(dims, L.SurrogateArch(), 3)
    m.autoencoder_frozen = True
    t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=7, train_ids=ids[30:], tournament_ids=ids[:30],
                                  wide_kernel=k), ds, m)
    t0 = time.time()
    t.train_steps(steps)
    rec = np.array([[s.d_loss, s.g_total, s.g_fwd, s.g_adv, s.g_cyc] for s in t.history().steps])
    res[k] = (rec, t.model().blobs["fwd"].copy(), t.wide_info())
    print("kernel", k, t.wide_info(), "time", round(time.time() - t0, 3))
    print(rec)
for k in (2, 3):
    d = np.abs(res[k][0] - res[1][0]) / np.abs(res[1][0])
    w = np.abs(res[k][1] - res[1][1]).max()
    print(f"kernel {k} vs generic: max rel loss diff {d.max():.3e}, max abs fwd weight diff {w:.3e}")
