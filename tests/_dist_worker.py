"""One rank of the 2-process gloo test (tests/test_dist_gloo.py).

Drives paper_1910_02270_b200.runner.distributed_round -- the per-rank
tournament logic of the multi-GPU path -- over torch.distributed (gloo) with
an oracle-backed CPU trainer in place of the GPU trainer (test
infrastructure only: the product trainer is the CUDA one). Replays the
reference's tiny_k2 experiment (tests/golden/tournament.npz): split, AE
pre-training, per-trainer reinit, 3 chunks of 10 steps with a round after
each, and writes this rank's records to OUT_DIR/rank<r>.npz.
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch.distributed as dist  # noqa: E402

import paper_1910_02270_b200 as L  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


class OracleTrainer:
    """The trainer surface distributed_round uses, over the C oracle."""

    def __init__(self, gan, ds, part, batch, seed, tour_ids, tid):
        self.tr = O.Trainer(gan, ds.x, ds.y, part, batch, seed)
        self.tx, self.ty = ds.rows(tour_ids)
        self.tid = tid
        self.records = []
        self.inc = None

    def step(self):
        return self.tr.step

    def train_steps(self, n):
        rec, sk, ep, aborted = self.tr.steps(n)
        assert not aborted
        self.records.append(rec)

    def fwd_floats(self):
        return self.tr.gan.blob(O.FWD).size

    def generator_blob(self):
        g = self.tr.gan
        return np.concatenate([g.blob(O.FWD), g.blob(O.INV)]).astype(np.float32)

    def set_validation(self, ids, ds):
        self.vx, self.vy = ds.rows(ids)

    def evaluate_payload(self, f, iv, w_f=1.0, w_i=1.0):
        cand = self.tr.gan.clone()
        cand.blob(O.FWD)[:] = f
        cand.blob(O.INV)[:] = iv
        return L.EvalMetric(*cand.evaluate(self.vx, self.vy, w_f, w_i))

    def _set_incoming(self, f, iv):
        self.inc = (np.array(f, np.float32), np.array(iv, np.float32))

    def model(self):
        g = self.tr.gan

        class _M:
            def disc_hash(_self):
                return L.fnv1a64(g.blob(O.DISC))
        return _M()

    def _decide(self):
        g = self.tr.gan
        loc = g.evaluate(self.tx, self.ty)
        cand = g.clone()
        cand.blob(O.FWD)[:] = self.inc[0]
        cand.blob(O.INV)[:] = self.inc[1]
        inc = cand.evaluate(self.tx, self.ty)
        adopted = L.incoming_wins(float(loc[2]), float(inc[2]))
        if adopted:  # trainer.hpp:117-127: copy, zero the moments, keep t
            for net, blob in ((O.FWD, self.inc[0]), (O.INV, self.inc[1])):
                g.blob(net)[:] = blob
                g.moment(net, 0)[:] = 0
                g.moment(net, 1)[:] = 0
        return L.EvalMetric(*loc), L.EvalMetric(*inc), adopted


def main():
    out_dir = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    g = dict(np.load(os.path.join(REPO, "tests", "golden", "tournament.npz")))
    pfx = "tiny_k2_"
    gen_n, spf, spec_seed, sampling_seed, k, batch, interval, budget, ae_steps, seed, shards = (
        int(v) for v in g[pfx + "cfg"])
    assert k == world
    dims = L.ModalityDims(*(int(v) for v in g[pfx + "dims"]))
    ds = L.synthetic_dataset(dims, gen_n, sampling_seed=sampling_seed, spec_seed=spec_seed,
                             samples_per_file=spf)
    val, train, tour = L.split_dataset(gen_n, k, 0.05, 0.05, seed, k >= 2)
    # AE pre-training on the sorted union (runner.hpp:249-279), oracle math
    base = O.Gan(list(dims.as_tuple()), O.Arch.tiny(), L.mix_seed(seed, 0xAE0))
    union = np.sort(np.concatenate(train))
    _, ay = ds.rows(union)
    draws = L.ae_batch_rows(seed, union.size, min(batch, union.size), ae_steps)
    pre = []
    for s in range(ae_steps):
        loss, eg, dg = base.ae_backward(ay[draws[s]])
        assert base.adam(O.ENC, eg) and base.adam(O.DEC, dg)
        pre.append(loss)
    gan = base.clone()
    gan.reinit_gan_nets(L.mix_seed(seed, 0x1417, rank))
    t = OracleTrainer(gan, ds, train[rank], batch, L.mix_seed(seed, 0x57A7E1, rank), tour[rank], rank)
    comm = L.TorchRoundComm(dist)
    done, rnd, recs, xfers, rounds = 0, 0, [], [], []
    while done < budget:
        chunk = min(interval, budget - done)
        t.train_steps(chunk)
        done += chunk
        if chunk == interval:
            rnd += 1
            rr, rec, xf = L.distributed_round(t, comm, k, rnd, seed)
            rounds.append(rr)
            recs.append(rec)
            xfers += xf
    # sharded validation (runner.sharded_validation): this rank's shard of the
    # validation slice, every model evaluated on it, metrics combined over
    # ranks -- against both models evaluated on the whole slice here
    shard = np.array_split(val, k)[rank]
    t.set_validation(shard, ds)
    sharded = L.runner.sharded_validation(t, comm, k, shard.size, 1.0, 1.0)
    t.set_validation(val, ds)
    blobs = comm.all_gather(t.generator_blob())
    nf = t.fwd_floats()
    full = [t.evaluate_payload(b[:nf], b[nf:]) for b in blobs]
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             val_sharded=np.array([[m.forward_mae, m.inverse_mae, m.combined] for m in sharded]),
             val_full=np.array([[m.forward_mae, m.inverse_mae, m.combined] for m in full]),
             split_train=np.concatenate(train), split_val=val, pretrain=np.array(pre),
             ae_enc=base.blob(O.ENC), ae_dec=base.blob(O.DEC),
             steps=np.concatenate(t.records),
             tr_round=np.array([r.round for r in recs]), tr_peer=np.array([r.peer for r in recs]),
             tr_local=np.array([r.local_metric for r in recs]),
             tr_incoming=np.array([r.incoming_metric for r in recs]),
             tr_kept=np.array([r.kept_incoming for r in recs]),
             xf_bytes=np.array([x.bytes for x in xfers]), xf_to=np.array([x.to_trainer for x in xfers]),
             pairs=np.array([rr.pairs[0] for rr in rounds]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
