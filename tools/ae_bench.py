"""Times autoencoder pre-training steps (train_ops.hpp:71-81) on one GPU:
the tcgen05 column passes (k_ae_tc.cu) and, for comparison, the SIMT ones
(LTFB_AE_SIMT=1), at paper dims with B = 128 by default. Each step is the
public AutoencoderPretrainer.step() (host sync per step, as the runner).

    python tools/ae_bench.py [--dims paper|desk] [--steps 50] [--rows 128]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_02270_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="paper")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rows", type=int, default=128)
    ap.add_argument("--source", type=int, default=2000)
    args = ap.parse_args()
    dims = L.ModalityDims.paper_scale() if args.dims == "paper" else L.ModalityDims()
    ds = L.synthetic_dataset(dims, args.source, sampling_seed=2, spec_seed=1)
    out = {"dims": args.dims, "output_dim": dims.output_dim(), "rows": args.rows, "steps": args.steps}
    draws = L.ae_batch_rows(11, args.source, args.rows, args.warmup + args.steps)
    for mode in ("tc", "simt"):
        if mode == "simt":
            os.environ["LTFB_AE_SIMT"] = "1"
        else:
            os.environ.pop("LTFB_AE_SIMT", None)
        model = L.make_cyclegan(dims, L.SurrogateArch(), 7)
        p = L.AutoencoderPretrainer(model, ds.y, batch_size=args.rows)
        kind = p.kind(args.rows)
        losses = []
        for s in range(args.warmup):
            losses.append(p.step(draws[s]))
        t0 = time.perf_counter()
        for s in range(args.warmup, args.warmup + args.steps):
            losses.append(p.step(draws[s]))
        dt = (time.perf_counter() - t0) / args.steps
        out[mode] = {"kind": kind, "ms_per_step": dt * 1e3, "first_loss": losses[0], "last_loss": losses[-1]}
        del p
    os.environ.pop("LTFB_AE_SIMT", None)
    out["loss_rel_diff_last"] = abs(out["tc"]["last_loss"] - out["simt"]["last_loss"]) / abs(out["simt"]["last_loss"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
