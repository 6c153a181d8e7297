"""Python mirror of the reference's trainer / model / tournament API.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/ltfb), so parity tests read like the
reference's own tests; every numeric operation runs in libltfb_gpu.so on the
GPU (through include/ltfb_gpu.h). Host work is limited to what the
reference itself does on the host and must stay bit-exact: seeded integer
decisions (partitions, pairings, epoch permutations), parameter init and the
synthetic data source -- all through the library's C ABI as well.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import (CapacityError, ConfigError, ContractError, DimensionError, Error, IoError,
                   NumericError, StoreCorruptError, check, lib, ptr)

NET_NAMES = ("enc", "dec", "fwd", "inv", "disc")
_ACTS = {"identity": 0, "relu": 1, "leaky_relu": 2, "tanh": 3, "sigmoid": 4}


# ------------------------------------------------------------- host algos --
def mix_seed(*words: int) -> int:
    """core/rng.hpp:23-30."""
    return int(lib.ltfb_mix_seed(np.array(words, dtype=np.uint64), len(words)))


def fnv1a64(buf) -> int:
    """core/hash.hpp:15-22 over raw bytes."""
    b = np.ascontiguousarray(buf)
    return int(lib.ltfb_fnv1a64(b.ctypes.data_as(C.c_void_p), b.nbytes))


def hex64(v: int) -> str:
    return f"{v:016x}"


@dataclass
class Matching:
    pairs: list = field(default_factory=list)
    bye: int = -1


def pair_trainers(k: int, round_: int, seed: int) -> Matching:
    """tournament/ltfb.hpp:52-66."""
    pairs = np.zeros(max(2, k), np.int32)
    bye, n = C.c_int32(-1), C.c_int32(0)
    check(lib.ltfb_pair_trainers(k, round_, seed, pairs, C.byref(bye), C.byref(n)))
    return Matching([(int(pairs[2 * i]), int(pairs[2 * i + 1])) for i in range(n.value)], int(bye.value))


def partition_dataset(ids: Sequence[int], k: int, seed: int) -> list:
    """tournament/ltfb.hpp:24-43."""
    a = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.empty_like(a)
    sizes = np.empty(max(k, 1), np.uint32)
    check(lib.ltfb_partition_dataset(a, a.size, k, seed, out, sizes))
    parts, at = [], 0
    for s in sizes[:k]:
        parts.append(out[at:at + s].copy())
        at += int(s)
    return parts


def split_dataset(total: int, k: int, validation_fraction: float, tournament_fraction: float,
                  seed: int, need_tournament: bool):
    """runner.hpp:134-169 -> (validation, [train per trainer], [tournament per trainer])."""
    n = max(total, 1)
    val, tr, to = np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint32)
    trs, tos = np.empty(k, np.uint32), np.empty(k, np.uint32)
    nv = C.c_uint64(0)
    check(lib.ltfb_split_dataset(total, k, validation_fraction, tournament_fraction, seed,
                                 int(need_tournament), val, C.byref(nv), tr, trs, to, tos))
    train, tour, a, b = [], [], 0, 0
    for t in range(k):
        train.append(tr[a:a + trs[t]].copy())
        tour.append(to[b:b + tos[t]].copy())
        a += int(trs[t])
        b += int(tos[t])
    return val[:nv.value].copy(), train, tour


def epoch_permutation(partition, epoch: int, seed: int) -> np.ndarray:
    """data/epoch_plan.hpp:69-71."""
    p = np.ascontiguousarray(partition, dtype=np.uint32)
    out = np.empty_like(p)
    check(lib.ltfb_epoch_permutation(p, p.size, epoch, seed, out))
    return out


def incoming_wins(local: float, incoming: float) -> bool:
    """tournament/ltfb.hpp:82-88 (the device decision kernel applies the same rule)."""
    return bool(lib.ltfb_incoming_wins(local, incoming))


def device_count() -> int:
    n = C.c_int(0)
    check(lib.ltfb_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------- shapes --
@dataclass
class ModalityDims:
    """surrogate/dims.hpp:15-53."""
    input_dim: int = 5
    latent_dim: int = 20
    scalar_dim: int = 15
    image_views: int = 3
    image_channels: int = 4
    image_h: int = 16
    image_w: int = 16

    def image_elems(self) -> int:
        return self.image_views * self.image_channels * self.image_h * self.image_w

    def output_dim(self) -> int:
        return self.scalar_dim + self.image_elems()

    def record_floats(self) -> int:
        return self.input_dim + self.output_dim()

    @staticmethod
    def paper_scale() -> "ModalityDims":
        return ModalityDims(image_h=64, image_w=64)

    def as_tuple(self):
        return (self.input_dim, self.latent_dim, self.scalar_dim, self.image_views,
                self.image_channels, self.image_h, self.image_w)

    def c(self) -> _lib.Dims:
        return _lib.Dims(*self.as_tuple())


@dataclass
class SurrogateArch:
    """surrogate/model.hpp:18-30."""
    enc_hidden: tuple = (64,)
    dec_hidden: tuple = (64,)
    fwd_hidden: tuple = (32, 32)
    inv_hidden: tuple = (32, 32)
    disc_hidden: tuple = (32, 32)
    hidden_act: str = "leaky_relu"
    hidden_slope: float = 0.2
    lambda_adv: float = 0.01
    lambda_cyc: float = 1.0
    lr: float = 0.001
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @staticmethod
    def tiny(width: int = 8) -> "SurrogateArch":
        return SurrogateArch(enc_hidden=(width,), dec_hidden=(width,), fwd_hidden=(width,),
                             inv_hidden=(width,), disc_hidden=(width,))

    def c(self) -> _lib.Arch:
        a = _lib.Arch()
        lib.ltfb_arch_defaults(C.byref(a))
        for name in ("enc", "dec", "fwd", "inv", "disc"):
            h = tuple(getattr(self, name + "_hidden"))
            if len(h) > 8:
                raise ContractError("more than 8 hidden layers")
            arr = getattr(a, name + "_hidden")
            for i in range(8):
                arr[i] = h[i] if i < len(h) else 0
            setattr(a, f"n_{name}_hidden", len(h))
        if self.hidden_act not in _ACTS:
            raise ConfigError("unknown activation name: " + self.hidden_act)
        a.hidden_act = _ACTS[self.hidden_act]
        a.hidden_slope = self.hidden_slope
        a.lambda_adv, a.lambda_cyc = self.lambda_adv, self.lambda_cyc
        a.lr, a.beta1, a.beta2, a.eps = self.lr, self.beta1, self.beta2, self.eps
        return a


def layer_widths(dims: ModalityDims, arch: SurrogateArch, net: int) -> list:
    o, lat, i = dims.output_dim(), dims.latent_dim, dims.input_dim
    h = [arch.enc_hidden, arch.dec_hidden, arch.fwd_hidden, arch.inv_hidden, arch.disc_hidden][net]
    ends = [(o, lat), (lat, o), (i, lat), (lat, i), (lat, 1)][net]
    return [ends[0], *h, ends[1]]


def param_count(dims: ModalityDims, arch: SurrogateArch, net: int) -> int:
    w = layer_widths(dims, arch, net)
    return sum(w[l] * w[l + 1] + w[l + 1] for l in range(len(w) - 1))


# ---------------------------------------------------------------- model --
@dataclass
class AdamState:
    """nn/adam.hpp:25-47."""
    m: np.ndarray
    v: np.ndarray
    t: int = 0

    def reset_moments(self):
        self.m[:] = 0
        self.v[:] = 0


class CycleGan:
    """Host value type of surrogate::CycleGan<float> (model.hpp:36-73).

    Each network is one float32 blob in manifest order; on the training
    path the authoritative copy lives in HBM and Trainer.model() returns a
    refreshed mirror."""

    def __init__(self, dims: ModalityDims, arch: SurrogateArch):
        self.dims, self.arch = dims, arch
        self.blobs = {n: np.zeros(param_count(dims, arch, i), np.float32) for i, n in enumerate(NET_NAMES)}
        self.opt = {n: AdamState(np.zeros_like(b), np.zeros_like(b)) for n, b in self.blobs.items()}
        self.lambda_adv = np.float32(arch.lambda_adv)
        self.lambda_cyc = np.float32(arch.lambda_cyc)
        self.autoencoder_frozen = False
        self.init_seeds = {n: 0 for n in NET_NAMES}  # MlpSpec::init_seed per net (checkpoints)

    def __getattr__(self, name):
        if name in NET_NAMES:
            return self.blobs[name]
        raise AttributeError(name)

    def copy(self) -> "CycleGan":
        m = CycleGan(self.dims, self.arch)
        m.blobs = {k: v.copy() for k, v in self.blobs.items()}
        m.opt = {k: AdamState(o.m.copy(), o.v.copy(), o.t) for k, o in self.opt.items()}
        m.autoencoder_frozen = self.autoencoder_frozen
        m.init_seeds = dict(self.init_seeds)
        return m

    def hash_of(self, net: str) -> int:
        return fnv1a64(self.blobs[net])

    def enc_hash(self):
        return self.hash_of("enc")

    def dec_hash(self):
        return self.hash_of("dec")

    def fwd_hash(self):
        return self.hash_of("fwd")

    def inv_hash(self):
        return self.hash_of("inv")

    def disc_hash(self):
        return self.hash_of("disc")

    def model_hash(self) -> int:
        """model.hpp:48-58: FNV chained over every blob in net order."""
        return fnv1a64(np.concatenate([self.blobs[n] for n in NET_NAMES]))


def make_cyclegan(dims: ModalityDims, arch: SurrogateArch, seed: int) -> CycleGan:
    """model.hpp:96-132 (init on the host: a bit-exact Rng sequence)."""
    m = CycleGan(dims, arch)
    dc, ac = dims.c(), arch.c()
    for i, n in enumerate(NET_NAMES):
        check(lib.ltfb_init_params(C.byref(dc), C.byref(ac), seed, i, m.blobs[n], m.blobs[n].size))
        m.init_seeds[n] = mix_seed(seed, i + 1)
    return m


def reinit_gan_nets(m: CycleGan, seed: int):
    """model.hpp:137-147."""
    dc, ac = m.dims.c(), m.arch.c()
    for i in (2, 3, 4):
        n = NET_NAMES[i]
        check(lib.ltfb_init_params(C.byref(dc), C.byref(ac), seed, i, m.blobs[n], m.blobs[n].size))
        m.opt[n] = AdamState(np.zeros_like(m.blobs[n]), np.zeros_like(m.blobs[n]), 0)
        m.init_seeds[n] = mix_seed(seed, i + 1)


@dataclass
class EvalMetric:
    forward_mae: float = 0.0
    inverse_mae: float = 0.0
    combined: float = 0.0


# ------------------------------------------------------------------ data --
class Dataset:
    """In-memory dataset: rows indexed by global sample id, plus the file
    layout (samples_per_file) the reference's bundle store would have --
    used for the preload-owner and epoch-0 file accounting
    (store.hpp:100-135)."""

    def __init__(self, dims: ModalityDims, x: np.ndarray, y: np.ndarray, samples_per_file: int = 500):
        self.dims = dims
        self.x = np.ascontiguousarray(x, np.float32)
        self.y = np.ascontiguousarray(y, np.float32)
        self.samples_per_file = int(samples_per_file)
        self.total = self.x.shape[0]

    def file_of(self, ids: np.ndarray) -> np.ndarray:
        return np.asarray(ids, np.int64) // self.samples_per_file

    def stride_bytes(self) -> int:
        return self.dims.record_floats() * 4

    def rows(self, ids):
        ids = np.asarray(ids, np.int64)
        return self.x[ids], self.y[ids]


def synth_generate(dims: ModalityDims, n: int, sampling_seed: int = 1, spec_seed: int = 1,
                   noise_level: float = 0.0, first: int = 0, total: int | None = None,
                   threads: int | None = None):
    """generate_dataset (synth/generator.hpp:195-206), rows [first, first+n)."""
    total = n if total is None else total
    x = np.empty((n, dims.input_dim), np.float32)
    y = np.empty((n, dims.output_dim()), np.float32)
    dc = dims.c()
    threads = threads or max(1, os.cpu_count() or 1)
    check(lib.ltfb_synth_generate(C.byref(dc), spec_seed, noise_level, first, n, total,
                                  sampling_seed, x, y, threads))
    return x, y


def synth_generate_ids(dims: ModalityDims, ids, total: int, sampling_seed: int = 1,
                       spec_seed: int = 1, noise_level: float = 0.0, threads: int | None = None):
    """Samples with global ids `ids` of a `total`-point sweep (host, threads)."""
    ids = np.ascontiguousarray(ids, np.uint32)
    x = np.empty((ids.size, dims.input_dim), np.float32)
    y = np.empty((ids.size, dims.output_dim()), np.float32)
    dc = dims.c()
    threads = threads or max(1, os.cpu_count() or 1)
    check(lib.ltfb_synth_generate_ids(C.byref(dc), spec_seed, noise_level, ids, ids.size, total,
                                      sampling_seed, x, y, threads))
    return x, y


class SparseDataset(Dataset):
    """Only the rows a trainer needs (its partition and tournament slice) of
    a large synthetic dataset; ids stay global."""

    def __init__(self, dims: ModalityDims, ids, x, y, total: int, samples_per_file: int = 500):
        super().__init__(dims, x, y, samples_per_file)
        self.ids = np.ascontiguousarray(ids, np.uint32)
        self.total = int(total)
        self._pos = {int(i): k for k, i in enumerate(self.ids)}

    def rows(self, ids):
        ids = np.asarray(ids)
        sel = np.fromiter((self._pos[int(i)] for i in ids), np.int64, count=ids.size)
        return self.x[sel], self.y[sel]


class BundleDataset(Dataset):
    """The reference's on-disk dataset: LBDS bundle files under a directory
    (data/bundle.hpp:134-224, DatasetIndex::scan_dir). Rows are read from
    the files on demand; a Trainer preloads its partition into HBM once
    (store.hpp:100-135), dealing files to shards round-robin."""

    def __init__(self, path):
        self.path = os.fspath(path)
        self._h = C.c_void_p()
        check(lib.ltfb_dataset_open(self.path.encode(), C.byref(self._h)))
        dc, total, nf = _lib.Dims(), C.c_uint64(0), C.c_uint64(0)
        check(lib.ltfb_dataset_info(self._h, C.byref(dc), C.byref(total), C.byref(nf)))
        self.dims = ModalityDims(dc.input_dim, dc.latent_dim, dc.scalar_dim, dc.image_views, dc.image_channels,
                                 dc.image_h, dc.image_w)
        self.total, self.n_files = int(total.value), int(nf.value)
        self.files_opened = 0  # cumulative, like the store counters

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.ltfb_dataset_destroy(h)
            self._h = None

    def file_of(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.empty(ids.size, np.uint32)
        check(lib.ltfb_dataset_file_of(self._h, ids, ids.size, out))
        return out.astype(np.int64)

    def rows(self, ids):
        ids = np.ascontiguousarray(ids, np.uint32)
        x = np.empty((ids.size, self.dims.input_dim), np.float32)
        y = np.empty((ids.size, self.dims.output_dim()), np.float32)
        opened = C.c_uint64(0)
        check(lib.ltfb_dataset_read(self._h, ids, ids.size, x, y, C.byref(opened)))
        self.files_opened += opened.value
        return x, y


def write_synth_bundles(path, dims: ModalityDims, n: int, sampling_seed: int = 1, spec_seed: int = 1,
                        noise_level: float = 0.0, samples_per_file: int = 500, threads: int | None = None):
    """generate_dataset(n) + write_bundles (runner.hpp:216-227) into path."""
    dc = dims.c()
    check(lib.ltfb_write_synth_bundles(os.fspath(path).encode(), C.byref(dc), spec_seed, noise_level, n,
                                       sampling_seed, samples_per_file, threads or max(1, os.cpu_count() or 1)))


class SynthDataset(Dataset):
    """A `total`-point synthetic sweep (generate_dataset, generator.hpp:195-206)
    that is never materialised on the host: a Trainer renders its partition
    and tournament slice straight into HBM with the device generator
    (k_synth.cu). `rows()` (small host-side reads: validation, e2e inputs)
    runs the host generator."""

    device_generated = True

    def __init__(self, dims: ModalityDims, total: int, sampling_seed: int = 1, spec_seed: int = 1,
                 noise_level: float = 0.0, samples_per_file: int = 500):
        if noise_level != 0.0:
            raise ContractError("SynthDataset: the device generator needs noise_level 0")
        self.dims = dims
        self.total = int(total)
        self.sampling_seed, self.spec_seed, self.noise_level = int(sampling_seed), int(spec_seed), noise_level
        self.samples_per_file = int(samples_per_file)

    def rows(self, ids):
        return synth_generate_ids(self.dims, ids, self.total, self.sampling_seed, self.spec_seed,
                                  self.noise_level)


def synth_generate_device(dims: ModalityDims, n: int, total: int | None = None, ids=None, first: int = 0,
                          sampling_seed: int = 1, spec_seed: int = 1, device: int = 0):
    """synth_generate(_ids) rendered on GPU `device`; returns torch tensors
    (x [n, 5], y [n, output_dim]) on that device."""
    import torch
    total = n if total is None else int(total)
    dev = torch.device("cuda", device)
    x = torch.empty((n, dims.input_dim), dtype=torch.float32, device=dev)
    y = torch.empty((n, dims.output_dim()), dtype=torch.float32, device=dev)
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(ids, np.uint32)
        if ids.size != n:
            raise ContractError("synth_generate_device: ids length must equal n")
        idp = ids.ctypes.data
    dc = dims.c()
    check(lib.ltfb_synth_generate_device(C.byref(dc), spec_seed, 0.0, idp, first, n, total, sampling_seed,
                                         x.data_ptr(), y.data_ptr(), dims.output_dim(), device))
    return x, y


def synthetic_dataset(dims: ModalityDims, n: int, sampling_seed: int = 1, spec_seed: int = 1,
                      noise_level: float = 0.0, samples_per_file: int = 500) -> Dataset:
    x, y = synth_generate(dims, n, sampling_seed, spec_seed, noise_level)
    return Dataset(dims, x, y, samples_per_file)


# --------------------------------------------------------------- history --
@dataclass
class StepRecord:
    trainer: int = 0
    step: int = 0
    epoch: int = 0
    d_loss: float = 0.0
    g_total: float = 0.0
    g_fwd: float = 0.0
    g_adv: float = 0.0
    g_cyc: float = 0.0
    skipped: bool = False


@dataclass
class EvalRecord:
    trainer: int = 0
    step: int = 0
    slice: str = ""
    forward_mae: float = 0.0
    inverse_mae: float = 0.0
    combined: float = 0.0


@dataclass
class EpochRecord:
    trainer: int = 0
    epoch: int = 0
    steps: int = 0
    files_opened: int = 0
    bytes_read: int = 0
    samples_shuffled: int = 0
    seconds: float = 0.0
    partial: bool = False


@dataclass
class RoundRecord:
    round: int = 0
    step: int = 0
    pairs: list = field(default_factory=list)
    bye: int = -1


@dataclass
class TrainerRoundRecord:
    round: int = 0
    step: int = 0
    trainer: int = 0
    peer: int = -1
    local_metric: float = 0.0
    incoming_metric: float = 0.0
    kept_incoming: bool = False
    disc_hash: str = ""


@dataclass
class TransferRecord:
    round: int = 0
    from_trainer: int = 0
    to_trainer: int = 0
    payload: str = ""
    bytes: int = 0
    blob_hash: str = ""


@dataclass
class HistorySegment:
    steps: list = field(default_factory=list)
    evals: list = field(default_factory=list)
    epochs: list = field(default_factory=list)
    skipped_steps: int = 0


@dataclass
class RoundResult:
    round: RoundRecord
    trainer_records: list
    transfers: list


# --------------------------------------------------------------- trainer --
@dataclass
class TrainerConfig:
    """train/trainer.hpp:26-39 (+ device placement and wide-kernel choice)."""
    trainer_id: int = 0
    n_shards: int = 4
    batch_size: int = 128
    store_mode: str = "preload"
    store_budget_bytes: int | None = None
    seed: int = 0
    numeric_abort_threshold: int = 10
    prefetch_depth: int = 1
    w_f: float = 1.0
    w_i: float = 1.0
    train_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    tournament_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    device: int = 0
    wide_kernel: int = 0       # 0 auto, 1 generic SIMT, 2 tcgen05 3xTF32, 3 tcgen05 TF32
    post_kernel: int = 0       # 0 auto, 1 generic, 2 smem fast path, 3 compile-time shapes
    lr: tuple | None = None    # per-net lr override (fwd, inv, disc)


class Trainer:
    """train::Trainer (trainer.hpp:41-308) with its state in HBM."""

    def __init__(self, cfg: TrainerConfig, dataset: Dataset, model: CycleGan):
        if cfg.n_shards < 1:
            raise ContractError("Trainer: n_shards must be >= 1")
        if cfg.batch_size < 1:
            raise ContractError("Trainer: batch_size must be >= 1")
        if not model.autoencoder_frozen:
            raise ContractError("Trainer: model autoencoder must be frozen")
        if cfg.store_mode != "preload":
            raise ContractError("Trainer: the B200 data store is HBM-resident (preload mode only); "
                                f"store mode '{cfg.store_mode}' is out of scope")
        self.cfg = cfg
        self.dataset = dataset
        self._dims, self._arch = model.dims, model.arch
        cc = _lib.TrainerConfigC()
        cc.trainer_id, cc.device, cc.n_shards = cfg.trainer_id, cfg.device, cfg.n_shards
        cc.numeric_abort_threshold = cfg.numeric_abort_threshold
        cc.batch_size, cc.seed = cfg.batch_size, cfg.seed
        cc.w_f, cc.w_i = cfg.w_f, cfg.w_i
        if cfg.lr is not None:
            cc.lr_fwd, cc.lr_inv, cc.lr_disc = cfg.lr
        cc.wide_kernel = cfg.wide_kernel
        cc.post_kernel = cfg.post_kernel
        self._h = C.c_void_p()
        dc, ac = model.dims.c(), model.arch.c()
        check(lib.ltfb_trainer_create(C.byref(dc), C.byref(ac), C.byref(cc), C.byref(self._h)))
        for i, n in enumerate(NET_NAMES):
            b = np.ascontiguousarray(model.blobs[n], np.float32)
            check(lib.ltfb_trainer_set_params(self._h, i, b, b.size))
            o = model.opt[n]
            check(lib.ltfb_trainer_set_adam(self._h, i, ptr(np.ascontiguousarray(o.m, np.float32)),
                                            ptr(np.ascontiguousarray(o.v, np.float32)), o.t))
        self._lr = model.opt  # keep hyper-parameter provenance
        self._segment = HistorySegment()
        self._mirror = model.copy()
        self._dirty = False
        # preload (store.hpp:100-135): files dealt round-robin to shards
        ids = np.ascontiguousarray(cfg.train_ids, np.uint32)
        if ids.size == 0:
            raise ContractError("plan_epoch: empty partition")
        if len(np.unique(ids)) != ids.size:
            raise ContractError("DataStore: duplicate sample ids in partition")
        if ids.max() >= dataset.total:
            raise ContractError("DataStore: partition id outside dataset")
        stride = dataset.stride_bytes()
        required = ids.size * stride
        if cfg.store_budget_bytes is not None and required > cfg.store_budget_bytes:
            raise CapacityError(f"preload requires {required} bytes but the store budget is "
                                f"{cfg.store_budget_bytes} bytes")
        t0 = time.perf_counter()
        files = dataset.file_of(ids)
        used = np.unique(files)  # file order
        loader = {int(f): i % cfg.n_shards for i, f in enumerate(used)}
        owner = np.array([loader[int(f)] for f in files], np.int32)
        gen = getattr(dataset, "device_generated", False)
        if gen:
            check(lib.ltfb_trainer_generate_store(self._h, ids, ids.size, ptr(owner), dataset.spec_seed,
                                                  dataset.noise_level, dataset.sampling_seed, dataset.total))
        else:
            x, y = dataset.rows(ids)
            check(lib.ltfb_trainer_load_store(self._h, ids, ids.size, np.ascontiguousarray(x),
                                              np.ascontiguousarray(y), ptr(owner)))
        preload_s = time.perf_counter() - t0
        self._segment.epochs.append(EpochRecord(cfg.trainer_id, 0, 0, len(used), required, 0, preload_s))
        tids = np.ascontiguousarray(cfg.tournament_ids, np.uint32)
        self._has_tour = tids.size > 0
        if self._has_tour:
            if gen:
                check(lib.ltfb_trainer_generate_slice(self._h, 0, tids, tids.size, dataset.spec_seed,
                                                      dataset.noise_level, dataset.sampling_seed,
                                                      dataset.total))
            else:
                tx, ty = dataset.rows(tids)
                check(lib.ltfb_trainer_set_slice(self._h, 0, np.ascontiguousarray(tx),
                                                 np.ascontiguousarray(ty), tids.size))
        self._val_key = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.ltfb_trainer_destroy(h)
            self._h = None

    # -- reference accessors
    def id(self) -> int:
        return self.cfg.trainer_id

    def step(self) -> int:
        v = C.c_uint64(0)
        check(lib.ltfb_trainer_step(self._h, C.byref(v)))
        return v.value

    def config(self) -> TrainerConfig:
        return self.cfg

    def history(self) -> HistorySegment:
        return self._segment

    def model(self) -> CycleGan:
        if self._dirty:
            for i, n in enumerate(NET_NAMES):
                b = self._mirror.blobs[n]
                check(lib.ltfb_trainer_get_params(self._h, i, b, b.size))
                o = self._mirror.opt[n]
                t = C.c_uint64(0)
                check(lib.ltfb_trainer_get_adam(self._h, i, ptr(o.m), ptr(o.v), C.byref(t)))
                o.t = t.value
            self._dirty = False
        return self._mirror

    def net_hash(self, net: str) -> int:
        """FNV-1a of one network's parameters (model.hpp:48-58 per net), read
        from HBM without refreshing the whole host mirror (a round needs only
        the disc hash; model() would copy every blob and Adam state)."""
        i = NET_NAMES.index(net)
        b = np.empty_like(self._mirror.blobs[net])
        check(lib.ltfb_trainer_get_params(self._h, i, b, b.size))
        return fnv1a64(b)

    def replica_hashes(self) -> list:
        h = self.model().model_hash()
        return [h] * self.cfg.n_shards

    def _drain_epochs(self):
        buf = (_lib.EpochRecordC * 4096)()
        n = C.c_uint64(0)
        check(lib.ltfb_trainer_take_epochs(self._h, buf, 4096, C.byref(n)))
        for i in range(n.value):
            e = buf[i]
            self._segment.epochs.append(EpochRecord(self.cfg.trainer_id, e.epoch, e.steps, 0, 0,
                                                    e.samples_shuffled, e.seconds, bool(e.partial)))

    def train_steps(self, n: int):
        """trainer.hpp:102-104; NumericError after the skip threshold."""
        if n == 0:
            return
        recs = (_lib.StepRecordC * n)()
        got = C.c_uint64(0)
        rc = lib.ltfb_trainer_train_steps(self._h, n, recs, C.byref(got))
        self._dirty = True
        for i in range(got.value):
            r = recs[i]
            self._segment.steps.append(StepRecord(self.cfg.trainer_id, r.step, r.epoch, r.d_loss, r.g_total,
                                                  r.g_fwd, r.g_adv, r.g_cyc, bool(r.skipped)))
            if r.skipped:
                self._segment.skipped_steps += 1
        self._drain_epochs()
        check(rc)

    def synchronize(self):
        check(lib.ltfb_trainer_synchronize(self._h))

    def prepare_graphs(self):
        """Capture the step graphs ahead of a timed region (no execution)."""
        check(lib.ltfb_trainer_prepare_graphs(self._h))

    # -- measurement hooks (bench.py)
    def timer_start(self):
        check(lib.ltfb_trainer_timer_start(self._h))

    def timer_stop(self) -> float:
        ms = C.c_double(0)
        check(lib.ltfb_trainer_timer_stop(self._h, C.byref(ms)))
        return ms.value

    def kernel_timing(self, on: bool):
        check(lib.ltfb_trainer_kernel_timing(self._h, int(on)))

    def kernel_time(self, which: int):
        ms, n = C.c_double(0), C.c_uint64(0)
        check(lib.ltfb_trainer_kernel_time(self._h, which, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def wide_info(self):
        k, c = C.c_int32(0), C.c_int32(0)
        check(lib.ltfb_trainer_wide_info(self._h, C.byref(k), C.byref(c)))
        return k.value, c.value

    def wide_tile(self) -> int:
        """Column-tile width of the tcgen05 wide pass (64: k_wide2; 32: the
        round-2a kernels; 0: generic SIMT)."""
        c = C.c_int32(0)
        check(lib.ltfb_trainer_wide_tile(self._h, C.byref(c)))
        return c.value

    def stream_mode(self) -> bool:
        """True when store-path steps run as the streamed step (persistent
        two-phase wide pass beside a persistent post cluster per run)."""
        k = C.c_int32(0)
        check(lib.ltfb_trainer_stream_info(self._h, C.byref(k)))
        return bool(k.value)

    def stream_profile(self, steps: int = 64) -> dict:
        """Runs `steps` streamed steps with per-stage %globaltimer stamps and
        returns the stage averages in µs; {} when not streamed."""
        if not self.stream_mode():
            return {}
        check(lib.ltfb_trainer_stream_profile(self._h, 1, None, 0))
        self.train_steps_raw(steps)
        out = (C.c_double * 8)()
        check(lib.ltfb_trainer_stream_profile(self._h, 0, out, 8))
        keys = ("step_us", "wide_phase1_us", "h_to_phase2_reduced_us", "phase2_tiles_us",
                "phase2_barrier_reduction_us", "d_step_overlapped_us", "post_chain_after_dec_us", "steps")
        return {k: float(v) for k, v in zip(keys, out)}

    def eval_info(self, which: int = 0) -> int:
        """2 when slice `which` (0 tournament, 1 validation) is evaluated by
        the tcgen05 k_eval_tc, 1 for the SIMT k_eval_wide."""
        k = C.c_int32(0)
        check(lib.ltfb_trainer_eval_info(self._h, which, C.byref(k)))
        return k.value

    def ae_info(self, rows: int = 128) -> int:
        """2 when ae_step over `rows` batch rows runs the tcgen05 column
        passes (k_ae_tc.cu), 1 for the SIMT ones (k_ae.cu)."""
        k = C.c_int32(0)
        check(lib.ltfb_trainer_ae_info(self._h, rows, C.byref(k)))
        return k.value

    def launch_count(self) -> int:
        n = C.c_uint64(0)
        check(lib.ltfb_trainer_launch_count(self._h, C.byref(n)))
        return n.value

    def train_steps_host(self, n: int, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        """e2e path: n steps whose minibatches x [n,B,in], y [n,B,out] are in
        host memory and are copied H2D inside the call."""
        recs = (_lib.StepRecordC * n)()
        got = C.c_uint64(0)
        check(lib.ltfb_trainer_train_steps_host(self._h, n, ptr(x), ptr(y), recs, C.byref(got)))
        self._dirty = True
        return np.ctypeslib.as_array(recs)

    def fwd_floats(self) -> int:
        """Length of the fwd part of the generator payload fwd||inv."""
        return param_count(self._dims, self._arch, 2)

    # -- distributed AE pre-training (runner.pretrain_autoencoder_sharded)
    def ae_alloc_source(self, rows: int):
        check(lib.ltfb_trainer_ae_alloc_source(self._h, rows))

    def ae_fill_from_store(self, slots: np.ndarray, dst_row: int):
        s = np.ascontiguousarray(slots, np.uint32)
        check(lib.ltfb_trainer_ae_fill_from_store(self._h, s, s.size, dst_row))

    def ae_allgather(self, comm: "Comm", rows_per_rank: int):
        check(lib.ltfb_trainer_ae_allgather(self._h, comm._h, rows_per_rank))

    def ae_step(self, idx: np.ndarray) -> float:
        i = np.ascontiguousarray(idx, np.uint32)
        loss = C.c_double(0.0)
        check(lib.ltfb_trainer_ae_step(self._h, i, i.size, C.byref(loss)))
        self._dirty = True
        return loss.value

    def exchange(self, comm: "Comm", peer: int):
        check(lib.ltfb_trainer_exchange(self._h, comm._h, peer))

    def decide_incoming(self):
        return self._decide()

    def train_steps_raw(self, n: int) -> np.ndarray:
        """Benchmark entry: runs n steps and returns the records as an array."""
        recs = (_lib.StepRecordC * n)()
        got = C.c_uint64(0)
        check(lib.ltfb_trainer_train_steps(self._h, n, recs, C.byref(got)))
        self._dirty = True
        return np.ctypeslib.as_array(recs)

    def flush_epoch_record(self):
        check(lib.ltfb_trainer_flush_epoch(self._h))
        self._drain_epochs()

    def _metric(self, m) -> EvalMetric:
        return EvalMetric(m.forward_mae, m.inverse_mae, m.combined)

    def eval_tournament(self, candidate: CycleGan | None = None) -> EvalMetric:
        """trainer.hpp:106-112."""
        if not self._has_tour:
            raise ContractError("Trainer: no tournament slice configured")
        return self._evaluate(0, candidate, self.cfg.w_f, self.cfg.w_i)

    def set_validation(self, ids: np.ndarray):
        ids = np.ascontiguousarray(ids, np.uint32)
        d = self.dataset
        if getattr(d, "device_generated", False):
            check(lib.ltfb_trainer_generate_slice(self._h, 1, ids, ids.size, d.spec_seed, d.noise_level,
                                                  d.sampling_seed, d.total))
        else:
            x, y = d.rows(ids)
            check(lib.ltfb_trainer_set_slice(self._h, 1, np.ascontiguousarray(x), np.ascontiguousarray(y),
                                             ids.size))
        self._val_key = ids.size

    def evaluate_payload(self, fwd: np.ndarray, inv: np.ndarray, w_f: float = 1.0, w_i: float = 1.0,
                         which: int = 1) -> EvalMetric:
        """evaluate (train_ops.hpp:191-205) of a generator payload (fwd, inv
        blobs; the frozen enc / dec are this trainer's) on the validation
        (which=1) or tournament (0) slice: the sharded-validation primitive."""
        if which == 1 and not self._val_key:
            raise ContractError("evaluate: empty data slice")
        out = _lib.EvalMetricC()
        f = np.ascontiguousarray(fwd, np.float32)
        iv = np.ascontiguousarray(inv, np.float32)
        check(lib.ltfb_trainer_evaluate(self._h, which, ptr(f), ptr(iv), w_f, w_i, C.byref(out)))
        return self._metric(out)

    def evaluate_validation(self, w_f: float = 1.0, w_i: float = 1.0, candidate=None) -> EvalMetric:
        if not self._val_key:
            raise ContractError("evaluate: empty data slice")
        return self._evaluate(1, candidate, w_f, w_i)

    def _evaluate(self, which, candidate, w_f, w_i) -> EvalMetric:
        out = _lib.EvalMetricC()
        if candidate is None or candidate is self._mirror:
            check(lib.ltfb_trainer_evaluate(self._h, which, None, None, w_f, w_i, C.byref(out)))
        else:
            if candidate.dec_hash() != self.model().dec_hash():
                raise ContractError("eval_tournament: candidate decoder differs from the trainer's "
                                    "frozen decoder")
            f = np.ascontiguousarray(candidate.blobs["fwd"], np.float32)
            iv = np.ascontiguousarray(candidate.blobs["inv"], np.float32)
            check(lib.ltfb_trainer_evaluate(self._h, which, ptr(f), ptr(iv), w_f, w_i, C.byref(out)))
        return self._metric(out)

    def adopt_generators(self, fwd: np.ndarray, inv: np.ndarray):
        """trainer.hpp:117-127."""
        f = np.ascontiguousarray(fwd, np.float32)
        iv = np.ascontiguousarray(inv, np.float32)
        if f.size != param_count(self._dims, self._arch, 2) or iv.size != param_count(self._dims, self._arch, 3):
            raise ContractError("adopt_generators: incompatible parameter shapes")
        check(lib.ltfb_trainer_adopt(self._h, f, iv))
        self._dirty = True

    def generator_blob(self) -> np.ndarray:
        n = C.c_uint64(0)
        check(lib.ltfb_trainer_generator_floats(self._h, C.byref(n)))
        out = np.empty(n.value, np.float32)
        check(lib.ltfb_trainer_get_generator(self._h, out, out.size))
        return out

    # -- tournament internals
    def _capture_from(self, src: "Trainer"):
        check(lib.ltfb_trainer_copy_incoming(self._h, src._h))

    def _set_incoming(self, fwd, inv):
        check(lib.ltfb_trainer_set_incoming(self._h, np.ascontiguousarray(fwd, np.float32),
                                            np.ascontiguousarray(inv, np.float32)))

    def _decide(self):
        loc, inc = _lib.EvalMetricC(), _lib.EvalMetricC()
        adopted = C.c_int32(0)
        check(lib.ltfb_trainer_tournament_decide(self._h, C.byref(loc), C.byref(inc), C.byref(adopted)))
        self._dirty = True
        return self._metric(loc), self._metric(inc), bool(adopted.value)


def ae_batch_rows(seed: int, rows: int, batch: int, steps: int) -> np.ndarray:
    """runner.hpp:257-266: the AE batch draws, [steps x batch] source rows."""
    out = np.empty(batch * steps, np.uint32)
    check(lib.ltfb_ae_batch_rows(seed, rows, batch, steps, out))
    return out.reshape(steps, batch)


class AutoencoderPretrainer:
    """surrogate::autoencoder_step (train_ops.hpp:71-81) on one GPU.

    Holds the model's five blobs and the enc/dec Adam states in HBM and the
    AE source slab (the sorted union of the training ids' y rows,
    runner.hpp:251-256); step(rows) runs one reconstruction step on those
    source rows. pull(model) copies enc/dec and their optimizer state back."""

    def __init__(self, model: CycleGan, y_source: np.ndarray, device: int = 0, batch_size: int = 128):
        if model.autoencoder_frozen:
            raise ContractError("autoencoder_step: autoencoder is frozen")
        y = np.ascontiguousarray(y_source, np.float32)
        if y.ndim != 2 or y.shape[1] != model.dims.output_dim():
            raise DimensionError("autoencoder source must be [rows x output_dim]")
        cc = _lib.TrainerConfigC()
        cc.trainer_id, cc.device, cc.n_shards = 0, device, 1
        cc.numeric_abort_threshold = 10
        cc.batch_size, cc.seed = batch_size, 0
        cc.w_f, cc.w_i = 1.0, 1.0
        self._h = C.c_void_p()
        dc, ac = model.dims.c(), model.arch.c()
        check(lib.ltfb_trainer_create(C.byref(dc), C.byref(ac), C.byref(cc), C.byref(self._h)))
        for i, n in enumerate(NET_NAMES):
            b = np.ascontiguousarray(model.blobs[n], np.float32)
            check(lib.ltfb_trainer_set_params(self._h, i, b, b.size))
            o = model.opt[n]
            check(lib.ltfb_trainer_set_adam(self._h, i, ptr(np.ascontiguousarray(o.m, np.float32)),
                                            ptr(np.ascontiguousarray(o.v, np.float32)), o.t))
        check(lib.ltfb_trainer_load_ae_source(self._h, y, y.shape[0]))
        self.rows = y.shape[0]

    def step(self, rows: np.ndarray) -> float:
        idx = np.ascontiguousarray(rows, np.uint32)
        loss = C.c_double(0.0)
        check(lib.ltfb_trainer_ae_step(self._h, idx, idx.size, C.byref(loss)))
        return loss.value

    def kind(self, rows: int = 128) -> int:
        """2: step() over `rows` rows runs the tcgen05 column passes
        (k_ae_tc.cu); 1: the SIMT ones (k_ae.cu)."""
        k = C.c_int32(0)
        check(lib.ltfb_trainer_ae_info(self._h, rows, C.byref(k)))
        return k.value

    def pull(self, model: CycleGan):
        for i, n in ((0, "enc"), (1, "dec")):
            b = model.blobs[n]
            check(lib.ltfb_trainer_get_params(self._h, i, b, b.size))
            o = model.opt[n]
            t = C.c_uint64(0)
            check(lib.ltfb_trainer_get_adam(self._h, i, ptr(o.m), ptr(o.v), C.byref(t)))
            o.t = t.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.ltfb_trainer_destroy(h)
            self._h = None


def pretrain_autoencoder(model: CycleGan, y_source: np.ndarray, steps: int, batch_size: int, seed: int,
                         device: int = 0) -> list:
    """runner.hpp:249-279: `steps` AE steps on batches of min(batch_size,
    rows) source rows drawn with replacement by Rng(mix_seed({seed, 0xae1}));
    returns the pretrain history [(step, loss)] and leaves the model's
    enc/dec (and their Adam states) trained. The caller freezes it."""
    rows = int(np.asarray(y_source).shape[0])
    b = min(batch_size, rows)
    draws = ae_batch_rows(seed, rows, b, steps) if steps else np.zeros((0, b), np.uint32)
    p = AutoencoderPretrainer(model, y_source, device, max(b, 1))
    hist = [(s + 1, p.step(draws[s])) for s in range(steps)]
    p.pull(model)
    return hist


class Comm:
    """NCCL communicator of the multi-GPU run (one rank per GPU/trainer)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        self._h = C.c_void_p()
        check(lib.ltfb_comm_create(uid, nranks, rank, device, C.byref(self._h)))
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.ltfb_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self._h and self._h.value:
            check(lib.ltfb_comm_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tournament_round(trainers: list, matching: Matching, round_index: int) -> RoundResult:
    """tournament/ltfb.hpp:96-164. Payloads of every pair are captured
    (device-to-device) before any trainer decides, so both sides judge the
    pre-round generators; each decision runs in a device kernel."""
    steps = {t.step() for t in trainers}
    if len(steps) != 1:
        raise ContractError("tournament_round: trainers are not step-synchronized")
    step = steps.pop()
    rr = RoundRecord(round_index, step, list(matching.pairs), matching.bye)
    transfers, exchanges = [], []
    for a, b in matching.pairs:
        if a == b:
            raise ContractError("tournament_round: trainer paired with itself")
        for to, frm in ((a, b), (b, a)):
            src = trainers[frm]
            blob = src.generator_blob()
            nf = param_count(src._dims, src._arch, 2)
            f, iv = blob[:nf], blob[nf:]
            transfers.append(TransferRecord(round_index, frm, to, "fwd", f.nbytes, hex64(fnv1a64(f))))
            transfers.append(TransferRecord(round_index, frm, to, "inv", iv.nbytes, hex64(fnv1a64(iv))))
            exchanges.append((to, frm))
    for to, frm in exchanges:
        trainers[to]._capture_from(trainers[frm])
    records = []
    for to, frm in exchanges:
        t = trainers[to]
        disc_hash = hex64(t.net_hash("disc"))
        loc, inc, adopted = t._decide()
        records.append(TrainerRoundRecord(round_index, step, to, frm, loc.combined, inc.combined,
                                          adopted, disc_hash))
    records.sort(key=lambda r: r.trainer)
    return RoundResult(rr, records, transfers)
