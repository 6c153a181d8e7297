"""Experiment orchestration over the B200 trainers (tournament/runner.hpp).

run_experiment() mirrors run_experiment (runner.hpp:232-420) in one process:
split the dataset (runner.hpp:134-169), pre-train the autoencoder on the
device (runner.hpp:249-279), build one trainer per partition with its own
generator / discriminator init (runner.hpp:283-317), then alternate training
chunks with tournament rounds, evaluating every trainer on the shared
validation slice after every chunk (runner.hpp:321-373), and pick the best
trainer (runner.hpp:380-398).

run_experiment_rank() is the same loop with ONE trainer per process (one
process per GPU, launched by torchrun): the split, the AE pre-training and
the pairings are pure functions of the run seed, so every rank computes them
itself (no communication); only the round moves data, the 15 KB generator
payload between the two partners of a pair (RoundComm.exchange), and the
per-rank records are gathered on rank 0 at the end.

RoundComm implementations:
  NcclRoundComm  device-to-device ncclSend/ncclRecv of the generator blob
                 (ltfb_trainer_exchange; the product path on GPUs);
  TorchRoundComm torch.distributed send/recv of the host blob (gloo on CPU:
                 the multi-process tests of this host logic).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import os
import sys
import time

import numpy as np

from .api import (BundleDataset, IoError, write_synth_bundles, CycleGan, Dataset, EvalRecord, HistorySegment, RoundRecord, Trainer, TrainerConfig,
                  TrainerRoundRecord, TransferRecord, ConfigError, ContractError, hex64, fnv1a64,
                  make_cyclegan, mix_seed, pair_trainers, param_count, pretrain_autoencoder,
                  reinit_gan_nets, split_dataset, tournament_round, EvalMetric, ae_batch_rows)


@dataclass
class RunConfig:
    """tournament/runner.hpp:47-78 (dataset generation and on-disk bundles
    are the caller's: the B200 path takes an in-memory Dataset)."""
    dims: object = None
    arch: object = None
    mode: str = "single"  # single | ltfb | k-independent
    trainers: int = 1
    shards: int = 1
    batch_size: int = 128
    interval: int = 100
    step_budget: int = 1000
    ae_steps: int = 2000
    seed: int = 1
    validation_fraction: float = 0.05
    tournament_fraction: float = 0.05
    lr_jitter: float = 0.0
    numeric_abort_threshold: int = 10
    w_f: float = 1.0
    w_i: float = 1.0
    # dataset / store fields of the reference RunConfig (runner.hpp:49-55,
    # 66-75): recorded in config.json and the config hash; the B200 path
    # takes the Dataset object itself and keeps the store HBM-resident
    data_dir: str = ""
    generate: bool = True
    gen_n: int = 16000
    samples_per_file: int = 500
    sampling_seed: int = 1
    spec_seed: int = 1
    noise_level: float = 0.0
    data_store: str = "preload"
    threads: int = 1
    store_budget_mb: int = 0
    prefetch_depth: int = 1
    # B200 placement (not part of the reference config or its hash)
    devices: tuple | None = None  # trainer t runs on devices[t % len(devices)]
    wide_kernel: int = 0
    # run_experiment_rank: "replicate" (every rank holds the whole validation
    # slice) or "shard" (rank r holds 1/k of it; all k models are evaluated on
    # every shard and the metrics combined)
    validation_sharding: str = "replicate"
    # run_experiment_rank: "replicate" (every rank pre-trains the AE on a host
    # copy of the whole union of the training partitions) or "shard" (each
    # AE batch is assembled from the ranks' HBM stores by an NCCL all-gather:
    # no rank holds the union; BASELINE config C5). Same draws, same result.
    ae_sharding: str = "replicate"


def sharded_ae_plan(parts, batch_size: int, steps: int, seed: int):
    """runner.hpp:251-277 with the union of the training partitions sharded
    over the ranks' stores: for the draws the replicated pre-training makes
    (Rng(mix_seed({seed, 0xae1})).below over the sorted union), each batch
    row's owning rank and its slot in that rank's store (the position in the
    rank's partition). Returns (owner [steps x b], slot [steps x b], b)."""
    ids = np.concatenate([np.asarray(p, np.uint32) for p in parts])
    rk = np.concatenate([np.full(len(p), r, np.int32) for r, p in enumerate(parts)])
    sl = np.concatenate([np.arange(len(p), dtype=np.uint32) for p in parts])
    order = np.argsort(ids, kind="stable")  # the sorted union
    b = min(batch_size, ids.size)
    draws = ae_batch_rows(seed, ids.size, b, steps) if steps else np.zeros((0, b), np.uint32)
    return rk[order][draws], sl[order][draws], b


def sharded_ae_indices(owner_row: np.ndarray, k: int, b: int) -> np.ndarray:
    """Source row of every batch row after the all-gather: rank r's rows sit
    at [r b, r b + count_r) in batch order."""
    idx = np.empty(owner_row.size, np.uint32)
    for r in range(k):
        pos = np.nonzero(owner_row == r)[0]
        idx[pos] = r * b + np.arange(pos.size, dtype=np.uint32)
    return idx


def pretrain_autoencoder_sharded(trainer, comm, parts, rank: int, steps: int, batch_size: int, seed: int,
                                 plan=None) -> list:
    """AE pre-training (train_ops.hpp:71-81, runner.hpp:249-279) on this
    rank's Trainer: per step every rank gathers the batch rows its store
    holds into its block of the AE source, an in-place NCCL all-gather
    assembles the batch on every rank, and every rank runs the same AE step
    (replicated, deterministic: identical enc / dec everywhere)."""
    k = len(parts)
    owner, slot, b = plan if plan is not None else sharded_ae_plan(parts, batch_size, steps, seed)
    trainer.ae_alloc_source(k * b)
    out = []
    for s in range(steps):
        mine = np.nonzero(owner[s] == rank)[0]
        trainer.ae_fill_from_store(slot[s][mine], rank * b)
        if k > 1:
            comm.ae_allgather(trainer, b)
        out.append((s + 1, trainer.ae_step(sharded_ae_indices(owner[s], k, b))))
    return out


@dataclass
class RunHistory:
    mode: str = "single"
    n_trainers: int = 1
    pretrain: list = field(default_factory=list)       # (step, loss)
    steps: list = field(default_factory=list)
    evals: list = field(default_factory=list)
    epochs: list = field(default_factory=list)
    rounds: list = field(default_factory=list)
    trainer_rounds: list = field(default_factory=list)
    transfers: list = field(default_factory=list)
    best_trainer: int = -1
    best_metric: EvalMetric | None = None
    config_hash: str = ""
    summaries: list = field(default_factory=list)


@dataclass
class TrainerSummary:
    """train/history.hpp TrainerSummary (one summary.csv row)."""
    trainer: int = 0
    steps: int = 0
    epochs_completed: int = 0
    final_d_loss: float = 0.0
    final_g_total: float = 0.0
    final_g_fwd: float = 0.0
    final_g_adv: float = 0.0
    final_g_cyc: float = 0.0
    final_val_forward_mae: float = 0.0
    final_val_inverse_mae: float = 0.0
    final_val_combined: float = 0.0
    rounds: int = 0
    incoming_adopted: int = 0
    files_opened: int = 0
    bytes_read: int = 0
    samples_shuffled: int = 0
    skipped_steps: int = 0
    is_best: bool = False


def trainer_summary(tid: int, steps: int, seg: HistorySegment, trainer_rounds, best_trainer: int) -> TrainerSummary:
    """runner.hpp:400-432: every field recomputed from the trainer's records
    (store counters = the sums of its epoch records' deltas)."""
    s = TrainerSummary(trainer=tid, steps=int(steps))
    for r in seg.steps:
        if not r.skipped:
            s.final_d_loss, s.final_g_total, s.final_g_fwd = r.d_loss, r.g_total, r.g_fwd
            s.final_g_adv, s.final_g_cyc = r.g_adv, r.g_cyc
    for e in seg.epochs:
        if e.epoch > 0 and not e.partial:
            s.epochs_completed += 1
        s.files_opened += e.files_opened
        s.bytes_read += e.bytes_read
        s.samples_shuffled += e.samples_shuffled
    for e in seg.evals:
        if e.slice == "validation":
            s.final_val_forward_mae, s.final_val_inverse_mae, s.final_val_combined = \
                e.forward_mae, e.inverse_mae, e.combined
    for r in trainer_rounds:
        if r.trainer == tid:
            s.rounds += 1
            s.incoming_adopted += 1 if r.kept_incoming else 0
    s.skipped_steps = int(seg.skipped_steps)
    s.is_best = tid == best_trainer
    return s


@dataclass
class RunResult:
    history: RunHistory
    best_trainer: int = -1
    best_metric: EvalMetric | None = None
    best_model: CycleGan | None = None


def validate_run_config(cfg: RunConfig):
    """runner.hpp:91-110."""
    bad = []
    if cfg.trainers < 1:
        bad.append("trainers must be >= 1")
    if cfg.shards < 1:
        bad.append("shards must be >= 1")
    if cfg.batch_size < 1:
        bad.append("batch_size must be >= 1")
    if cfg.interval < 1:
        bad.append("interval must be >= 1")
    if not (0 <= cfg.validation_fraction < 1):
        bad.append("validation_fraction must be in [0,1)")
    if not (0 <= cfg.tournament_fraction < 1):
        bad.append("tournament_fraction must be in [0,1)")
    if cfg.numeric_abort_threshold < 0:
        bad.append("numeric_abort_threshold must be >= 0")
    if cfg.mode not in ("single", "ltfb", "k-independent", "k_independent"):
        bad.append("unknown run mode: " + str(cfg.mode))
    if cfg.lr_jitter != 0.0:
        bad.append("lr_jitter is not supported on the B200 path")
    if cfg.data_store != "preload":
        # store.hpp:62-271: the B200 store is the HBM-resident preload store;
        # the file-streaming modes are out of scope, so refuse
        # rather than silently running preload semantics
        bad.append(f"data_store '{cfg.data_store}' is not supported on the B200 path (preload only)")
    if cfg.store_budget_mb != 0:
        bad.append("store_budget_mb is not supported on the B200 path (the partition is HBM-resident)")
    if bad:
        raise ConfigError("invalid run config: " + "; ".join(bad) + "; ")


def _base_model(cfg: RunConfig, dataset: Dataset, train_parts, autoencoder=None) -> tuple:
    """runner.hpp:247-279: AE pre-training on the sorted union of the
    training partitions, then frozen. `autoencoder` (a CycleGan whose enc /
    dec blobs are used as the pre-trained AE; no pre-training runs, the
    history's pretrain records stay empty) is the reference-state injection
    the parity tests use to compare the GAN phase on its own."""
    base = make_cyclegan(cfg.dims, cfg.arch, mix_seed(cfg.seed, 0xAE0))
    if autoencoder is not None:
        for n in ("enc", "dec"):
            if autoencoder.blobs[n].size != base.blobs[n].size:
                raise ContractError("run_experiment: injected autoencoder has incompatible shapes")
            base.blobs[n][:] = autoencoder.blobs[n]
        base.autoencoder_frozen = True
        return base, []
    union = np.sort(np.concatenate([np.asarray(p, np.uint32) for p in train_parts]))
    _, ay = dataset.rows(union)
    dev = (cfg.devices or (0,))[0]
    pre = pretrain_autoencoder(base, ay, cfg.ae_steps, cfg.batch_size, cfg.seed, device=dev) if cfg.ae_steps else []
    base.autoencoder_frozen = True
    return base, pre


def _trainer_for(cfg: RunConfig, dataset: Dataset, base: CycleGan, split, t: int) -> Trainer:
    """runner.hpp:283-317."""
    model = base.copy()
    reinit_gan_nets(model, mix_seed(cfg.seed, 0x1417, t))
    devs = cfg.devices or (0,)
    tc = TrainerConfig(trainer_id=t, n_shards=cfg.shards, batch_size=cfg.batch_size,
                       seed=mix_seed(cfg.seed, 0x57A7E1, t), numeric_abort_threshold=cfg.numeric_abort_threshold,
                       w_f=cfg.w_f, w_i=cfg.w_i, train_ids=split[1][t], tournament_ids=split[2][t],
                       device=devs[t % len(devs)], wide_kernel=cfg.wide_kernel, prefetch_depth=0)
    return Trainer(tc, dataset, model)


def _eval_record(t: Trainer, step: int) -> EvalRecord:
    m = t.evaluate_validation(t.cfg.w_f, t.cfg.w_i)
    return EvalRecord(t.cfg.trainer_id, step, "validation", m.forward_mae, m.inverse_mae, m.combined)


def _merge(history: RunHistory, segments):
    """runner.hpp:171-199."""
    for seg in segments:
        history.steps += seg.steps
        history.evals += seg.evals
        history.epochs += seg.epochs
    history.steps.sort(key=lambda r: (r.step, r.trainer))
    history.evals.sort(key=lambda r: (r.step, r.trainer))
    history.epochs.sort(key=lambda r: (r.epoch, r.trainer))


def ensure_dataset(cfg: RunConfig) -> BundleDataset:
    """runner.hpp:203-230: the LBDS bundles under cfg.data_dir, generated
    there first (generate_dataset + write_bundles) when the directory holds
    none and cfg.generate is set."""
    import os
    have = os.path.isdir(cfg.data_dir) and any(f.endswith(".lbds") for f in os.listdir(cfg.data_dir))
    if not have:
        if not cfg.generate:
            raise IoError(f"no dataset found under {cfg.data_dir} and generation is disabled")
        write_synth_bundles(cfg.data_dir, cfg.dims, cfg.gen_n, cfg.sampling_seed, cfg.spec_seed, cfg.noise_level,
                            cfg.samples_per_file)
    return BundleDataset(cfg.data_dir)


def _check_dims(cfg: RunConfig, dataset: Dataset):
    if cfg.dims is not None and dataset.dims != cfg.dims:
        raise ConfigError("configured dims do not match the dataset on disk")


def run_experiment(cfg: RunConfig, dataset: Dataset | None = None, autoencoder=None) -> RunResult:
    """runner.hpp:232-420 in one process (k trainers on cfg.devices).
    Without a dataset, ensure_dataset(cfg) provides the bundles;
    `autoencoder` replaces AE pre-training (see _base_model)."""
    validate_run_config(cfg)
    if dataset is None:
        dataset = ensure_dataset(cfg)
    _check_dims(cfg, dataset)
    k = 1 if cfg.mode == "single" else cfg.trainers
    rounds_enabled = cfg.mode == "ltfb" and k >= 2
    split = split_dataset(dataset.total, k, cfg.validation_fraction, cfg.tournament_fraction, cfg.seed, k >= 2)
    history = RunHistory(mode=cfg.mode.replace("_", "-"), n_trainers=k)
    base, history.pretrain = _base_model(cfg, dataset, split[1], autoencoder)
    trainers = [_trainer_for(cfg, dataset, base, split, t) for t in range(k)]
    have_val = split[0].size > 0
    if have_val:
        for t in trainers:
            t.set_validation(split[0])

    def evaluate_all(at):
        if have_val:
            for t in trainers:
                t.history().evals.append(_eval_record(t, at))

    evaluate_all(0)
    done, round_index = 0, 0
    while done < cfg.step_budget:
        chunk = min(cfg.interval, cfg.step_budget - done)
        for t in trainers:
            t.train_steps(chunk)
        done += chunk
        evaluate_all(done)
        if rounds_enabled and chunk == cfg.interval:
            round_index += 1
            matching = pair_trainers(k, round_index, mix_seed(cfg.seed, 0x9A18))
            r = tournament_round(trainers, matching, round_index)
            history.rounds.append(r.round)
            history.trainer_rounds += r.trainer_records
            history.transfers += r.transfers
    for t in trainers:
        t.flush_epoch_record()
    _merge(history, [t.history() for t in trainers])
    res = RunResult(history)
    if have_val:
        best = float("inf")
        for t in trainers:
            m = t.evaluate_validation(cfg.w_f, cfg.w_i)
            if m.combined < best:
                best, res.best_trainer, res.best_metric = m.combined, t.cfg.trainer_id, m
    else:
        res.best_trainer = 0
    res.best_model = trainers[max(res.best_trainer, 0)].model().copy()
    history.best_trainer, history.best_metric = res.best_trainer, res.best_metric
    history.summaries = [trainer_summary(t.cfg.trainer_id, t.step(), t.history(), history.trainer_rounds,
                                         res.best_trainer) for t in trainers]
    from .outputs import config_hash
    history.config_hash = config_hash(cfg)
    return res


# ------------------------------------------------------------ multi-rank --
class NcclRoundComm:
    """The product exchange: device-to-device ncclSend/ncclRecv of the
    generator blob into the peer's incoming buffer (ltfb_trainer_exchange),
    plus torch.distributed for the small host-side collectives."""

    def __init__(self, comm, dist):
        self.comm, self.dist = comm, dist
        self.rank, self.world = comm.rank, comm.nranks

    def exchange(self, trainer, peer: int):
        trainer.exchange(self.comm, peer)

    def ae_allgather(self, trainer, rows_per_rank: int):
        trainer.ae_allgather(self.comm, rows_per_rank)

    def all_gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


class TorchRoundComm:
    """Generator exchange over torch.distributed point-to-point (gloo on
    CPU). The trainer receives the peer's blob as its incoming candidate."""

    def __init__(self, dist):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def exchange(self, trainer, peer: int):
        import torch
        blob = np.ascontiguousarray(trainer.generator_blob(), np.float32)
        send = torch.from_numpy(blob.copy())
        recv = torch.empty_like(send)
        ops = [self.dist.P2POp(self.dist.isend, send, peer), self.dist.P2POp(self.dist.irecv, recv, peer)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        nf = trainer.fwd_floats()
        got = recv.numpy()
        trainer._set_incoming(got[:nf], got[nf:])

    def all_gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


def warm_peer_links(trainer, comm):
    """Exchanges a payload once with every other rank (circle-method
    schedule: k - 1 rounds of disjoint pairs, a bye for odd k) so that the
    point-to-point connections NCCL sets up lazily on first use exist
    before the first tournament round. Decides nothing; the incoming buffer
    is overwritten by the next real exchange."""
    k, me = comm.world, comm.rank
    n = k + (k & 1)  # even number of slots; slot k is the bye when k is odd
    for r in range(n - 1):
        if me == n - 1:
            peer = r
        elif me == r:
            peer = n - 1
        else:
            peer = (2 * r - me) % (n - 1)
        if peer < k and peer != me:
            comm.exchange(trainer, peer)
    # the round's step-synchronisation all-gather goes through the process
    # group, whose collectives are also set up lazily (~10 ms on first use)
    comm.all_gather(None)
    if hasattr(trainer, "synchronize"):
        trainer.synchronize()


def distributed_round(trainer, comm, k: int, round_index: int, seed: int):
    """tournament/ltfb.hpp:96-164 seen from one rank (rank == trainer id):
    the pairing is recomputed locally (identical on every rank), the pair
    swaps generator payloads, and each side evaluates local vs incoming on
    its own tournament slice and adopts on the device if the incoming one
    wins. Returns (RoundRecord, TrainerRoundRecord | None, [TransferRecord])."""
    _tt = [time.perf_counter()] if os.environ.get("LTFB_ROUND_TIMING") else None
    steps = comm.all_gather(trainer.step())
    if _tt is not None:
        _tt.append(time.perf_counter())
    if len(set(steps)) != 1:
        raise ContractError("tournament_round: trainers are not step-synchronized")
    step = steps[0]
    matching = pair_trainers(k, round_index, mix_seed(seed, 0x9A18))
    rr = RoundRecord(round_index, step, list(matching.pairs), matching.bye)
    me, peer = comm.rank, None
    for a, b in matching.pairs:
        if a == b:
            raise ContractError("tournament_round: trainer paired with itself")
        if a == me:
            peer = b
        elif b == me:
            peer = a
    if peer is None:  # the bye of an odd k
        return rr, None, []
    blob = trainer.generator_blob()
    nf = trainer.fwd_floats()
    f, iv = blob[:nf], blob[nf:]
    transfers = [TransferRecord(round_index, me, peer, "fwd", f.nbytes, hex64(fnv1a64(f))),
                 TransferRecord(round_index, me, peer, "inv", iv.nbytes, hex64(fnv1a64(iv)))]
    if _tt is not None:
        _tt.append(time.perf_counter())
    comm.exchange(trainer, peer)
    if _tt is not None:
        _tt.append(time.perf_counter())
    nh = getattr(trainer, "net_hash", None)  # (a trainer without it: the full model copy)
    disc_hash = hex64(nh("disc") if nh else trainer.model().disc_hash())
    if _tt is not None:
        _tt.append(time.perf_counter())
    loc, inc, adopted = trainer._decide()
    if _tt is not None:  # LTFB_ROUND_TIMING: host wall per phase (dev aid)
        _tt.append(time.perf_counter())
        d = [round((b - a) * 1e3, 3) for a, b in zip(_tt, _tt[1:])]
        print(f"[round {round_index} rank {me}] ms: step all_gather {d[0]}, payload+hashes {d[1]}, "
              f"exchange {d[2]}, disc hash {d[3]}, decide {d[4]}", file=sys.stderr)
    rec = TrainerRoundRecord(round_index, step, me, peer, loc.combined, inc.combined, adopted, disc_hash)
    return rr, rec, transfers


def sharded_validation(trainer, comm, k: int, shard_rows: int, w_f: float, w_i: float) -> list:
    """evaluate_all / best-of-k (runner.hpp:321-337, 380-398) with the
    validation slice sharded over the k ranks: all-gather the k generator
    payloads (15 KB each), evaluate every model on this rank's shard, then
    all-gather the per-shard MAEs and combine them in rank order weighted by
    shard rows (sum_q mae_q n_q / n, the reference's means over the whole
    slice up to double summation order). Returns the k EvalMetrics, the
    same list on every rank."""
    blobs = comm.all_gather(np.ascontiguousarray(trainer.generator_blob(), np.float32))
    nf = trainer.fwd_floats()
    local = []
    for b in blobs:
        if shard_rows:
            m = trainer.evaluate_payload(b[:nf], b[nf:], w_f, w_i)
            local.append((m.forward_mae, m.inverse_mae))
        else:
            local.append((0.0, 0.0))
    parts = comm.all_gather((local, int(shard_rows)))
    n = sum(p[1] for p in parts)
    if n == 0:
        raise ContractError("evaluate: empty data slice")
    out = []
    for r in range(k):
        f = i = 0.0
        for q in range(len(parts)):
            if parts[q][1]:
                f += parts[q][0][r][0] * parts[q][1]
                i += parts[q][0][r][1] * parts[q][1]
        f, i = f / n, i / n
        out.append(EvalMetric(f, i, w_f * f + w_i * i))
    return out


def run_experiment_rank(cfg: RunConfig, dataset: Dataset | None, comm, device: int = 0) -> RunResult | None:
    """One rank of a k = world-size LTFB run (one trainer per GPU). Returns
    the merged RunResult on rank 0 (None elsewhere)."""
    validate_run_config(cfg)
    if dataset is None:
        dataset = ensure_dataset(cfg)  # every rank generates / scans the same bundles
    _check_dims(cfg, dataset)
    k = comm.world
    if cfg.mode != "single" and cfg.trainers != k:
        raise ConfigError("run_experiment_rank: trainers must equal the world size")
    k = 1 if cfg.mode == "single" else k
    rounds_enabled = cfg.mode == "ltfb" and k >= 2
    split = split_dataset(dataset.total, k, cfg.validation_fraction, cfg.tournament_fraction, cfg.seed, k >= 2)
    history = RunHistory(mode=cfg.mode.replace("_", "-"), n_trainers=k)
    rcfg = RunConfig(**{**cfg.__dict__, "devices": (device,)})
    if cfg.ae_sharding not in ("replicate", "shard"):
        raise ConfigError("ae_sharding must be 'replicate' or 'shard'")
    if cfg.ae_sharding == "shard":
        # the trainer's store first (its rows are the AE's source), then the
        # AE pre-training on the trainer itself: reinit_gan_nets touches only
        # fwd / inv / disc and the AE only enc / dec, so the order is free
        base = make_cyclegan(cfg.dims, cfg.arch, mix_seed(cfg.seed, 0xAE0))
        base.autoencoder_frozen = True
        t = _trainer_for(rcfg, dataset, base, split, comm.rank)
        history.pretrain = pretrain_autoencoder_sharded(t, comm, split[1], comm.rank, cfg.ae_steps,
                                                        cfg.batch_size, cfg.seed) if cfg.ae_steps else []
    else:
        base, history.pretrain = _base_model(rcfg, dataset, split[1])  # replicated, deterministic
        t = _trainer_for(rcfg, dataset, base, split, comm.rank)
    if rounds_enabled:
        warm_peer_links(t, comm)
    have_val = split[0].size > 0
    shard = cfg.validation_sharding == "shard" and k > 1
    if cfg.validation_sharding not in ("replicate", "shard"):
        raise ConfigError("validation_sharding must be 'replicate' or 'shard'")
    my_val = np.array_split(split[0], k)[comm.rank] if shard else split[0]

    def eval_record(at):
        if not shard:
            return _eval_record(t, at)
        m = sharded_validation(t, comm, k, my_val.size, cfg.w_f, cfg.w_i)[comm.rank]
        return EvalRecord(t.cfg.trainer_id, at, "validation", m.forward_mae, m.inverse_mae, m.combined)

    if have_val:
        if my_val.size:
            t.set_validation(my_val)
        t.history().evals.append(eval_record(0))
    done, round_index, my_rounds, my_xfers, rounds = 0, 0, [], [], []
    while done < cfg.step_budget:
        chunk = min(cfg.interval, cfg.step_budget - done)
        t.train_steps(chunk)
        done += chunk
        if have_val:
            t.history().evals.append(eval_record(done))
        if rounds_enabled and chunk == cfg.interval:
            round_index += 1
            rr, rec, xf = distributed_round(t, comm, k, round_index, cfg.seed)
            rounds.append(rr)
            if rec is not None:
                my_rounds.append(rec)
            my_xfers += xf
    t.flush_epoch_record()
    if have_val and shard:
        final = sharded_validation(t, comm, k, my_val.size, cfg.w_f, cfg.w_i)[comm.rank]
    else:
        final = t.evaluate_validation(cfg.w_f, cfg.w_i) if have_val else None
    parts = comm.all_gather((t.history(), my_rounds, my_xfers, final, t.step()))
    # best-of-k on the shared validation slice (runner.hpp:380-398): every
    # rank sees the same metrics, only the winner ships its model
    best_rank, best = 0, float("inf")
    if have_val:
        for r, p in enumerate(parts):
            if p[3].combined < best:
                best, best_rank = p[3].combined, r
    models = comm.all_gather(t.model().copy() if comm.rank == best_rank else None)
    if comm.rank != 0:
        return None
    _merge(history, [p[0] for p in parts])
    history.rounds = rounds
    history.trainer_rounds = sorted([r for p in parts for r in p[1]], key=lambda r: (r.round, r.trainer))
    # transfers in the reference's order: per pair (a <- b, then b <- a)
    by = {(x.round, x.from_trainer, x.payload): x for p in parts for x in p[2]}
    for rr in rounds:
        for a, b in rr.pairs:
            for to, frm in ((a, b), (b, a)):
                history.transfers += [by[(rr.round, frm, "fwd")], by[(rr.round, frm, "inv")]]
    res = RunResult(history, best_rank, parts[best_rank][3] if have_val else None, models[best_rank])
    history.best_trainer, history.best_metric = res.best_trainer, res.best_metric
    history.summaries = [trainer_summary(r, p[4], p[0], history.trainer_rounds, best_rank)
                         for r, p in enumerate(parts)]
    from .outputs import config_hash
    history.config_hash = config_hash(cfg)
    return res
