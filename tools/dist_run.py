#!/usr/bin/env python3
"""Multi-GPU LTFB run: one trainer per GPU (torchrun, NCCL), driven by
runner.run_experiment_rank with the device-to-device NCCL generator exchange.
With --golden PFX (tiny_k2_, desk_k2_, ...) the run replays that reference
experiment (tests/golden/tournament.npz) and rank 0 checks the merged
history against it; prints one JSON line on rank 0, exit 1 on mismatch.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_run.py --golden tiny_k2_
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--golden", default="tiny_k2_")
    p.add_argument("--out", default=None, help="rank 0 writes the run directory here (outputs.py)")
    p.add_argument("--validation-sharding", default="replicate", choices=["replicate", "shard"])
    p.add_argument("--ae-sharding", default="replicate", choices=["replicate", "shard"])
    a = p.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1910_02270_b200 as L
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = [L.Comm.unique_id() if rank == 0 else b"\0" * 128]
    dist.broadcast_object_list(uid, src=0)
    comm = L.NcclRoundComm(L.Comm(uid[0], world, rank, local), dist)

    g = dict(np.load(os.path.join(REPO, "tests", "golden", "tournament.npz")))
    pfx = a.golden
    gen_n, spf, spec_seed, sampling_seed, k, batch, interval, budget, ae_steps, seed, shards = (
        int(v) for v in g[pfx + "cfg"])
    if k != world:
        raise SystemExit(f"{pfx} needs {k} ranks, got {world}")
    dims = L.ModalityDims(*(int(v) for v in g[pfx + "dims"]))
    arch = L.SurrogateArch.tiny() if pfx.startswith("tiny") else L.SurrogateArch()
    ds = L.synthetic_dataset(dims, gen_n, sampling_seed=sampling_seed, spec_seed=spec_seed, samples_per_file=spf)
    cfg = L.RunConfig(dims=dims, arch=arch, mode="ltfb", trainers=k, shards=shards, batch_size=batch,
                      interval=interval, step_budget=budget, ae_steps=ae_steps, seed=seed, gen_n=gen_n,
                      samples_per_file=spf, spec_seed=spec_seed, sampling_seed=sampling_seed,
                      data_dir="data_" + pfx.rstrip("_"),  # = tests/golden/run_<pfx>/config.json
                      validation_sharding=a.validation_sharding, ae_sharding=a.ae_sharding)
    res = L.run_experiment_rank(cfg, ds, comm, device=local)
    ok = True
    if rank == 0:
        h = res.history

        def rel(x, y):
            x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
            return float(np.max(np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1e-12)))

        checks = {
            "steps_order": [(s.trainer, s.step) for s in h.steps] ==
            list(zip(g[pfx + "steps_trainer"].tolist(), g[pfx + "steps_step"].tolist())),
            "g_total_rel": rel([s.g_total for s in h.steps], g[pfx + "steps_g_total"]),
            "kept": [int(r.kept_incoming) for r in h.trainer_rounds] == g[pfx + "tr_kept"].astype(int).tolist(),
            "local_rel": rel([r.local_metric for r in h.trainer_rounds], g[pfx + "tr_local"]),
            "xf_bytes": [x.bytes for x in h.transfers] == g[pfx + "xf_bytes"].astype(int).tolist(),
            "best_trainer": res.best_trainer == int(g[pfx + "best_trainer"][0]),
            "evals_rel": rel([e.combined for e in h.evals], g[pfx + "evals_combined"]),
        }
        checks["pretrain_rel"] = rel([pp[1] for pp in h.pretrain], g[pfx + "pretrain_loss"]) if ae_steps else 0.0
        # end to end with the device AE (tests/test_gpu_parity.py REL_LOSS_DEVICE_AE)
        ok = (checks["steps_order"] and checks["kept"] and checks["xf_bytes"] and checks["best_trainer"]
              and checks["g_total_rel"] < 5e-4 and checks["local_rel"] < 5e-4 and checks["evals_rel"] < 5e-4
              and checks["pretrain_rel"] < 1e-4)
        if a.out:
            L.write_run_outputs(a.out, cfg, h, res.best_model)
        print(json.dumps({"golden": pfx, "ranks": world, "validation": a.validation_sharding,
                          "ae": a.ae_sharding, "ok": bool(ok), "checks": checks,
                          "rounds": len(h.rounds), "exchange": "nccl device-to-device",
                          "pretrain": [pp[1] for pp in h.pretrain], "g_total": [s.g_total for s in h.steps],
                          "local": [r.local_metric for r in h.trainer_rounds],
                          "best_hash": L.hex64(res.best_model.model_hash())}))
    okt = [ok]
    dist.broadcast_object_list(okt, src=0)
    comm.comm.close()
    dist.destroy_process_group()
    sys.exit(0 if okt[0] else 1)


if __name__ == "__main__":
    main()
