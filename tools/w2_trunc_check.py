"""k_wide2 experiment: do the tf32 MMAs truncate fp32 operands themselves?
Runs the same paper-dim training with and without the in-place hi writes
(LTFB_W2_FLAGS=1) in two processes and compares the step losses bitwise."""
import json, os, subprocess, sys
code = r'''
import sys, os, json, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1910_02270_b200 as L
dims = L.ModalityDims.paper_scale()
ds = L.synthetic_dataset(dims, 1200, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 5); m.autoencoder_frozen = True
ids = np.arange(1200, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=3, train_ids=ids[64:], tournament_ids=ids[:64]), ds, m)
t.train_steps(12)
print(json.dumps([[s.d_loss, s.g_total, s.g_fwd, s.g_adv, s.g_cyc] for s in t.history().steps]))
'''
res = {}
for f in ("0", "1"):
    env = dict(os.environ, LTFB_W2_FLAGS=f)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True).stdout
    res[f] = json.loads(out.strip().splitlines()[-1])
same = res["0"] == res["1"]
import numpy as np
a, b = np.array(res["0"]), np.array(res["1"])
print(json.dumps({"bit_identical": same, "max_rel": float(np.max(np.abs(a - b) / np.abs(a)))}))
