"""Device vs host synthetic-data throughput (k_synth vs SynthGenerator on
all host cores), paper dims. Prints one JSON line.

usage: python tools/synth_driver.py [--n 100000] [--host-n 4000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02270_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--host-n", type=int, default=4000)
    a = ap.parse_args()
    d = L.ModalityDims.paper_scale()
    total = a.n
    ids = np.random.default_rng(1).permutation(total).astype(np.uint32)
    L.synth_generate_device(d, 256, total, ids=ids[:256])  # warm-up (module load, pool)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, y = L.synth_generate_device(d, a.n, total, ids=ids)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    L.synth_generate_ids(d, ids[:a.host_n], total)
    host_s = time.perf_counter() - t0
    out_bytes = a.n * (d.output_dim() + d.input_dim) * 4
    print(json.dumps({
        "dims": "paper 3x4x64x64", "n_device": a.n,
        "device_samples_per_s": a.n / dev_s, "device_GB_per_s_written": out_bytes / dev_s / 1e9,
        "host_samples_per_s": a.host_n / host_s, "host_threads": os.cpu_count(),
        "device_s_incl_ids_upload": dev_s}))


if __name__ == "__main__":
    main()
