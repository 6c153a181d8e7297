"""Per-kernel CUDA-event times of the launched step (bench.py's kernel-timing
pass) next to the streamed step's per-step time, in one process."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02270_b200 as L  # noqa: E402
dims = L.ModalityDims.paper_scale()
ds = L.SynthDataset(dims, 8000, sampling_seed=1, spec_seed=1)
m = L.make_cyclegan(dims, L.SurrogateArch(), 5)
m.autoencoder_frozen = True
ids = np.arange(8000, dtype=np.uint32)
t = L.Trainer(L.TrainerConfig(n_shards=1, batch_size=128, seed=3, train_ids=ids[400:], tournament_ids=ids[:400]), ds, m)
out = {"stream": t.stream_mode()}
for label in ("first", "after_stream"):
    t.kernel_timing(True)
    t.train_steps_raw(20)
    out[label] = {n: t.kernel_time(i) for i, n in enumerate(("gather", "small_fwd", "wide", "post", "reduce"))}
    t.kernel_timing(False)
    t.synchronize(); t.timer_start(); t.train_steps_raw(100); out[label + "_stream_ms"] = t.timer_stop() / 100
print(json.dumps(out))
