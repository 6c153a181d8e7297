#!/usr/bin/env python3
"""BASELINE config C5 at scale: an HBM-resident data store of ~10 M synthetic
JAG samples (desk dims 3 x 4 x 16 x 16, 12.4 KB per sample) sharded across
the GPUs, one LTFB trainer per GPU (torchrun, NCCL). Each rank renders its
partition and tournament slice straight into HBM (k_synth), pre-trains the
autoencoder with batches gathered from all ranks' stores (NCCL all-gather,
no rank holds the union: runner.pretrain_autoencoder_sharded), then trains
with a tournament round every --interval steps. Prints one JSON line on
rank 0: per-GPU store bytes, render / AE / epoch-plan times, samples/s.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/c5_run.py [--total 10000000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--total", type=int, default=10_000_000)
    p.add_argument("--ae-steps", type=int, default=20)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--interval", type=int, default=100)
    p.add_argument("--batch", type=int, default=128)
    a = p.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1910_02270_b200 as L
    from paper_1910_02270_b200.runner import pretrain_autoencoder_sharded, sharded_ae_plan
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [L.Comm.unique_id() if rank == 0 else b"\0" * 128]
        dist.broadcast_object_list(uid, src=0)
        comm = L.NcclRoundComm(L.Comm(uid[0], world, rank, local), dist)

    def max_all(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dims, arch, seed, k = L.ModalityDims(), L.SurrogateArch(), 1, world
    val, tour_parts = None, None
    val, train_parts, tour_parts = L.split_dataset(a.total, k, 0.05, 0.05, seed, k >= 2)
    ds = L.SynthDataset(dims, a.total, sampling_seed=1, spec_seed=1)
    base = L.make_cyclegan(dims, arch, L.mix_seed(seed, 0xAE0))
    model = base.copy()
    L.reinit_gan_nets(model, L.mix_seed(seed, 0x1417, rank))
    model.autoencoder_frozen = True
    cfg = L.TrainerConfig(trainer_id=rank, n_shards=1, batch_size=a.batch, seed=L.mix_seed(seed, 0x57A7E1, rank),
                          prefetch_depth=0, train_ids=train_parts[rank], tournament_ids=tour_parts[rank],
                          device=local)
    t0 = time.perf_counter()
    tr = L.Trainer(cfg, ds, model)  # renders the partition + tournament slice into HBM
    tr.synchronize()
    render_s = max_all(time.perf_counter() - t0)
    out_pad = (dims.output_dim() + 3) // 4 * 4
    store_bytes = int(train_parts[rank].size) * (dims.input_dim + out_pad) * 4
    # AE pre-training over the sharded union: the host plan (which rank holds
    # each draw: a sort of the union ids), then the device steps
    t0 = time.perf_counter()
    plan = sharded_ae_plan(train_parts, a.batch, a.ae_steps + 1, seed)
    plan_s = max_all(time.perf_counter() - t0)
    pretrain_autoencoder_sharded(tr, comm, train_parts, rank, 1, a.batch, seed,
                                 plan=(plan[0][:1], plan[1][:1], plan[2]))  # allocation, first launch
    tr.synchronize()
    t0 = time.perf_counter()
    pre = pretrain_autoencoder_sharded(tr, comm, train_parts, rank, a.ae_steps, a.batch, seed,
                                       plan=(plan[0][1:], plan[1][1:], plan[2]))
    tr.synchronize()
    ae_ms = max_all((time.perf_counter() - t0) * 1e3 / max(1, a.ae_steps))
    # epoch plan of this rank's partition (the host shuffle the trainer runs
    # at every epoch start, epoch_plan.hpp:59-71)
    t0 = time.perf_counter()
    L.epoch_permutation(train_parts[rank], 2, cfg.seed)
    plan_ms = max_all((time.perf_counter() - t0) * 1e3)
    if comm is not None:
        L.warm_peer_links(tr, comm)
    tr.train_steps(5)
    rounds = [0]

    def run(n):
        done = 0
        while done < n:
            chunk = min(a.interval, n - done)
            tr.train_steps_raw(chunk)
            done += chunk
            if k > 1 and chunk == a.interval:
                rounds[0] += 1
                L.distributed_round(tr, comm, k, rounds[0], seed)

    if world > 1:
        dist.barrier()
    tr.synchronize()
    tr.timer_start()
    run(a.steps)
    ms = max_all(tr.timer_stop())
    if rank == 0:
        print(json.dumps({
            "config": "C5: HBM-resident store of %d synthetic desk-dim samples (3x4x16x16, out %d) sharded over %d "
                      "GPU(s), one LTFB trainer per GPU, B=%d, round every %d steps" % (
                          a.total, dims.output_dim(), world, a.batch, a.interval),
            "n_gpus": world, "samples_total": a.total, "partition_rows_per_gpu": int(train_parts[rank].size),
            "store_bytes_per_gpu": store_bytes, "store_gb_per_gpu": store_bytes / 1e9,
            "render_s": render_s, "ae_plan_s": plan_s, "ae_steps": a.ae_steps, "ae_ms_per_step": ae_ms,
            "ae_source": "batches gathered from every rank's store (NCCL all-gather), union never replicated",
            "ae_first_losses": [x[1] for x in pre[:3]],
            "epoch_plan_ms": plan_ms, "steps": a.steps, "rounds": rounds[0],
            "ms_per_step": ms / a.steps, "samples_per_s": k * a.batch * a.steps / (ms / 1e3),
            "stream_mode": bool(tr.stream_mode())}))
    if comm is not None:
        comm.comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
