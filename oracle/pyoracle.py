"""TEST INFRASTRUCTURE (oracle) — ctypes binding for oracle/ltfb_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module; the product package never does.  The shared object is built by
``make -C oracle oracle`` (also run from __graft_entry__.build()); if it is
missing it is compiled on first import (gcc is present on the GPU box too).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "liboracle.so")

ENC, DEC, FWD, INV, DISC = range(5)
NET_NAMES = ("enc", "dec", "fwd", "inv", "disc")


def _load():
    src = os.path.join(HERE, "ltfb_oracle.c")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "_build/liboracle.so"])
    return C.CDLL(SO)


_L = _load()
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class _Rng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_mix = _sig("lo_mix_seed", C.c_uint64, u64p, C.c_int)
_rng_init = _sig("lo_rng_init", None, C.POINTER(_Rng), C.c_uint64)
_rng_next = _sig("lo_rng_next", C.c_uint64, C.POINTER(_Rng))
_rng_uniform = _sig("lo_rng_uniform", C.c_double, C.POINTER(_Rng))
_rng_below = _sig("lo_rng_below", C.c_uint64, C.POINTER(_Rng), C.c_uint64)
_rng_normal = _sig("lo_rng_normal", C.c_double, C.POINTER(_Rng))
_shuffle_u32 = _sig("lo_shuffle_u32", None, C.POINTER(_Rng), u32p, C.c_size_t)
_fnv = _sig("lo_fnv1a64", C.c_uint64, C.c_void_p, C.c_size_t, C.c_uint64)
_partition = _sig("lo_partition", C.c_int, u32p, C.c_size_t, C.c_int, C.c_uint64, u32p, u32p)
_pair = _sig("lo_pair_trainers", C.c_int, C.c_int, C.c_int, C.c_uint64, i32p, C.POINTER(C.c_int32))
_split = _sig("lo_split_dataset", C.c_int, C.c_size_t, C.c_int, C.c_double, C.c_double,
              C.c_uint64, C.c_int, u32p, C.POINTER(C.c_size_t), u32p, u32p, u32p, u32p)
_wins = _sig("lo_incoming_wins", C.c_int, C.c_double, C.c_double)
_plan = _sig("lo_plan_perm", None, u32p, C.c_size_t, C.c_uint32, C.c_uint64, u32p)
_synth_create = _sig("lo_synth_create", C.c_void_p, u32p, C.c_uint64, C.c_double)
_synth_destroy = _sig("lo_synth_destroy", None, C.c_void_p)
_synth_sample = _sig("lo_synth_sample", C.c_int, C.c_void_p, f64p, f32p, f32p)
_grid_side = _sig("lo_grid_side", C.c_uint32, C.c_uint64)
_sweep = _sig("lo_sweep_point", None, C.c_uint64, C.c_uint32, C.c_uint64, f64p)
_synth_gen = _sig("lo_synth_generate", C.c_int, C.c_void_p, C.c_uint64, C.c_uint64,
                  C.c_uint64, C.c_uint64, f32p, f32p)
_mlp_count = _sig("lo_mlp_param_count", C.c_size_t, u32p, C.c_int)
_mlp_init = _sig("lo_mlp_init", None, u32p, C.c_int, C.c_uint64, f32p)
_mlp_fwd = _sig("lo_mlp_forward", None, u32p, i32p, f64p, C.c_int, f32p, f32p, C.c_size_t, f32p)
_mlp_bwd = _sig("lo_mlp_backward", None, u32p, i32p, f64p, C.c_int, f32p, f32p, C.c_size_t,
                f32p, f32p, f32p)
_mae = _sig("lo_mae", C.c_double, f32p, f32p, C.c_size_t, f32p)
_bce = _sig("lo_bce", C.c_double, f32p, f32p, C.c_size_t, f32p)
_sigmoid = _sig("lo_stable_sigmoid", C.c_float, C.c_float)
_adam = _sig("lo_adam_step", C.c_int, f32p, f32p, f32p, f32p, C.c_size_t, C.POINTER(C.c_uint64),
             C.c_double, C.c_double, C.c_double, C.c_double)
_gan_create = _sig("lo_gan_create", C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                   u32p, C.c_int, u32p, C.c_int, u32p, C.c_int, u32p, C.c_int, u32p, C.c_int,
                   C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                   C.c_double)
_gan_clone = _sig("lo_gan_clone", C.c_void_p, C.c_void_p)
_gan_destroy = _sig("lo_gan_destroy", None, C.c_void_p)
_gan_init = _sig("lo_gan_init", None, C.c_void_p, C.c_uint64)
_gan_reinit = _sig("lo_gan_reinit_gan_nets", None, C.c_void_p, C.c_uint64)
_gan_blob = _sig("lo_gan_blob", C.POINTER(C.c_float), C.c_void_p, C.c_int, C.POINTER(C.c_size_t))
_gan_moment = _sig("lo_gan_moment", C.POINTER(C.c_float), C.c_void_p, C.c_int, C.c_int)
_gan_t = _sig("lo_gan_t", C.POINTER(C.c_uint64), C.c_void_p, C.c_int)
_gan_adam = _sig("lo_gan_adam", C.c_int, C.c_void_p, C.c_int, f32p)
_disc_bwd = _sig("lo_disc_backward", C.c_double, C.c_void_p, f32p, f32p, C.c_size_t, f32p)
_gen_bwd = _sig("lo_gen_backward", None, C.c_void_p, f32p, f32p, C.c_size_t, f32p, f32p, f64p)
_ae_bwd = _sig("lo_ae_backward", C.c_double, C.c_void_p, f32p, C.c_size_t, f32p, f32p)
_evaluate = _sig("lo_evaluate", None, C.c_void_p, f32p, f32p, C.c_size_t, C.c_double,
                 C.c_double, f64p)
_tr_create = _sig("lo_trainer_create", C.c_void_p, C.c_void_p, f32p, f32p, u32p, C.c_size_t,
                  C.c_size_t, C.c_uint64, C.c_int)
_tr_destroy = _sig("lo_trainer_destroy", None, C.c_void_p)
_tr_steps = _sig("lo_trainer_steps", C.c_size_t, C.c_void_p, C.c_size_t, f64p, u8p, u32p)
_tr_gan = _sig("lo_trainer_gan", C.c_void_p, C.c_void_p)
_tr_step = _sig("lo_trainer_step", C.c_uint64, C.c_void_p)


def mix_seed(*parts: int) -> int:
    return int(_mix(np.array(parts, dtype=np.uint64), len(parts)))


class Rng:
    """core/rng.hpp:35-97"""

    def __init__(self, seed: int):
        self._s = _Rng()
        _rng_init(C.byref(self._s), seed)

    def next(self) -> int:
        return int(_rng_next(C.byref(self._s)))

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lo + (hi - lo) * float(_rng_uniform(C.byref(self._s)))

    def below(self, n: int) -> int:
        return int(_rng_below(C.byref(self._s), n))

    def normal(self) -> float:
        return float(_rng_normal(C.byref(self._s)))

    def shuffle_u32(self, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.uint32).copy()
        _shuffle_u32(C.byref(self._s), v, v.size)
        return v


def fnv1a64(buf: bytes | np.ndarray, h: int = 0xCBF29CE484222325) -> int:
    b = bytes(buf) if not isinstance(buf, np.ndarray) else np.ascontiguousarray(buf).tobytes()
    return int(_fnv(C.c_char_p(b), len(b), h))


def partition_dataset(ids, k: int, seed: int):
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.empty_like(ids)
    sizes = np.empty(max(k, 1), dtype=np.uint32)
    if _partition(ids, ids.size, k, seed, out, sizes) != 0:
        raise ValueError("partition_dataset: bad k")
    parts, off = [], 0
    for s in sizes:
        parts.append(out[off:off + s].copy())
        off += s
    return parts


def pair_trainers(k: int, round_: int, seed: int):
    pairs = np.zeros(max(k, 2), dtype=np.int32)
    bye = C.c_int32(-1)
    n = _pair(k, round_, seed, pairs, C.byref(bye))
    return [(int(pairs[2 * i]), int(pairs[2 * i + 1])) for i in range(n)], int(bye.value)


def split_dataset(total: int, k: int, vf: float, tf: float, seed: int, need_tournament: bool):
    val = np.zeros(max(total, 1), dtype=np.uint32)
    nval = C.c_size_t(0)
    tr = np.zeros(max(total, 1), dtype=np.uint32)
    tour = np.zeros(max(total, 1), dtype=np.uint32)
    trs = np.zeros(k, dtype=np.uint32)
    tos = np.zeros(k, dtype=np.uint32)
    if _split(total, k, vf, tf, seed, int(need_tournament), val, C.byref(nval), tr, trs, tour, tos):
        raise ValueError("split_dataset failed")
    train, tourn, a, b = [], [], 0, 0
    for t in range(k):
        train.append(tr[a:a + trs[t]].copy())
        tourn.append(tour[b:b + tos[t]].copy())
        a += trs[t]
        b += tos[t]
    return val[:nval.value].copy(), train, tourn


def incoming_wins(local: float, incoming: float) -> bool:
    return bool(_wins(local, incoming))


def plan_perm(partition, epoch: int, seed: int) -> np.ndarray:
    p = np.ascontiguousarray(partition, dtype=np.uint32)
    out = np.empty_like(p)
    _plan(p, p.size, epoch, seed, out)
    return out


def dims_output(d7) -> int:
    return int(d7[2] + d7[3] * d7[4] * d7[5] * d7[6])


class Synth:
    """synth/generator.hpp:51-206"""

    def __init__(self, dims7, spec_seed: int, noise: float = 0.0):
        self.dims = np.array(dims7, dtype=np.uint32)
        self.out_dim = dims_output(self.dims)
        self._p = _synth_create(self.dims, spec_seed, noise)
        if not self._p:
            raise ValueError("synth: input_dim must be 5")

    def __del__(self):
        if getattr(self, "_p", None):
            _synth_destroy(self._p)
            self._p = None

    def sample(self, p5):
        p = np.ascontiguousarray(p5, dtype=np.float64)
        x = np.empty(5, np.float32)
        y = np.empty(self.out_dim, np.float32)
        if _synth_sample(self._p, p, x, y):
            raise ValueError("parameters must lie in [0,1]")
        return x, y

    def generate(self, n: int, sampling_seed: int, first: int = 0, total: int | None = None):
        total = n if total is None else total
        x = np.empty((n, 5), np.float32)
        y = np.empty((n, self.out_dim), np.float32)
        if _synth_gen(self._p, first, n, total, sampling_seed, x, y):
            raise ValueError("generate failed")
        return x, y


def grid_side(n: int) -> int:
    return int(_grid_side(n))


def sweep_point(i: int, g: int, seed: int) -> np.ndarray:
    p = np.empty(5, np.float64)
    _sweep(i, g, seed, p)
    return p


def _mlp_args(widths, acts, slopes):
    w = np.ascontiguousarray(widths, dtype=np.uint32)
    a = np.ascontiguousarray(acts, dtype=np.int32)
    s = np.ascontiguousarray(slopes, dtype=np.float64)
    return w, a, s, len(w) - 1


def mlp_param_count(widths) -> int:
    w = np.ascontiguousarray(widths, dtype=np.uint32)
    return int(_mlp_count(w, len(w) - 1))


def mlp_init(widths, seed: int) -> np.ndarray:
    w = np.ascontiguousarray(widths, dtype=np.uint32)
    blob = np.empty(mlp_param_count(w), np.float32)
    _mlp_init(w, len(w) - 1, seed, blob)
    return blob


def mlp_forward(widths, acts, slopes, blob, x):
    w, a, s, L = _mlp_args(widths, acts, slopes)
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows = x.size // int(w[0])
    out = np.empty((rows, int(w[-1])), np.float32)
    _mlp_fwd(w, a, s, L, np.ascontiguousarray(blob, np.float32), x, rows, out)
    return out


def mlp_backward(widths, acts, slopes, blob, x, grad_out):
    w, a, s, L = _mlp_args(widths, acts, slopes)
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows = x.size // int(w[0])
    pg = np.empty(mlp_param_count(w), np.float32)
    gi = np.empty((rows, int(w[0])), np.float32)
    _mlp_bwd(w, a, s, L, np.ascontiguousarray(blob, np.float32), x, rows,
             np.ascontiguousarray(grad_out, np.float32), pg, gi)
    return pg, gi


def mae(pred, target):
    p = np.ascontiguousarray(pred, np.float32).ravel()
    t = np.ascontiguousarray(target, np.float32).ravel()
    g = np.empty_like(p)
    return float(_mae(p, t, p.size, g)), g


def bce(probs, labels):
    p = np.ascontiguousarray(probs, np.float32).ravel()
    y = np.ascontiguousarray(labels, np.float32).ravel()
    g = np.empty_like(p)
    return float(_bce(p, y, p.size, g)), g


def stable_sigmoid(z: float) -> float:
    return float(_sigmoid(z))


def adam_step(params, grads, m, v, t: int, lr=0.001, b1=0.9, b2=0.999, eps=1e-8):
    """In-place on float32 arrays; returns the new t (unchanged on failure)."""
    tt = C.c_uint64(t)
    rc = _adam(params, np.ascontiguousarray(grads, np.float32), m, v, params.size, C.byref(tt),
               lr, b1, b2, eps)
    return int(tt.value), rc == 0


class Arch:
    """surrogate/model.hpp:18-30 defaults."""

    def __init__(self, enc=(64,), dec=(64,), fwd=(32, 32), inv=(32, 32), disc=(32, 32),
                 slope=0.2, lambda_adv=0.01, lambda_cyc=1.0, lr=0.001, beta1=0.9,
                 beta2=0.999, eps=1e-8):
        self.enc, self.dec, self.fwd, self.inv, self.disc = (tuple(h) for h in (enc, dec, fwd, inv, disc))
        self.slope, self.lambda_adv, self.lambda_cyc = slope, lambda_adv, lambda_cyc
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps

    @staticmethod
    def tiny():
        return Arch(enc=(8,), dec=(8,), fwd=(8,), inv=(8,), disc=(8,))


class Gan:
    """surrogate::CycleGan<float> restated (model.hpp:36-147)."""

    def __init__(self, dims7, arch: Arch, seed: int | None = None, _ptr=None):
        self.dims = np.array(dims7, dtype=np.uint32)
        self.in_dim, self.latent, self.out_dim = int(self.dims[0]), int(self.dims[1]), dims_output(self.dims)
        self.arch = arch
        if _ptr is not None:
            self._p = _ptr
        else:
            h = [np.array(x if len(x) else [0], dtype=np.uint32) for x in
                 (arch.enc, arch.dec, arch.fwd, arch.inv, arch.disc)]
            self._p = _gan_create(self.in_dim, self.latent, self.out_dim,
                                  h[0], len(arch.enc), h[1], len(arch.dec), h[2], len(arch.fwd),
                                  h[3], len(arch.inv), h[4], len(arch.disc), arch.slope,
                                  arch.lambda_adv, arch.lambda_cyc, arch.lr, arch.beta1,
                                  arch.beta2, arch.eps)
            if seed is not None:
                _gan_init(self._p, seed)
        self._owned = _ptr is None

    def __del__(self):
        if getattr(self, "_owned", False) and self._p:
            _gan_destroy(self._p)
            self._p = None

    def clone(self) -> "Gan":
        g = Gan(self.dims, self.arch, _ptr=_gan_clone(self._p))
        g._owned = True
        return g

    def reinit_gan_nets(self, seed: int):
        _gan_reinit(self._p, seed)

    def blob(self, net: int) -> np.ndarray:
        """A live float32 view of the network blob (writable)."""
        n = C.c_size_t(0)
        ptr = _gan_blob(self._p, net, C.byref(n))
        return np.ctypeslib.as_array(ptr, shape=(n.value,))

    def moment(self, net: int, which: int) -> np.ndarray:
        n = self.blob(net).size
        return np.ctypeslib.as_array(_gan_moment(self._p, net, which), shape=(n,))

    def t(self, net: int) -> int:
        return int(_gan_t(self._p, net).contents.value)

    def adam(self, net: int, grads) -> bool:
        return _gan_adam(self._p, net, np.ascontiguousarray(grads, np.float32)) == 0

    def disc_backward(self, x, y):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        g = np.empty(self.blob(DISC).size, np.float32)
        return float(_disc_bwd(self._p, x, y, x.shape[0], g)), g

    def gen_backward(self, x, y):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        fg = np.empty(self.blob(FWD).size, np.float32)
        ig = np.empty(self.blob(INV).size, np.float32)
        losses = np.empty(4, np.float64)
        _gen_bwd(self._p, x, y, x.shape[0], fg, ig, losses)
        return losses, fg, ig

    def ae_backward(self, y):
        y = np.ascontiguousarray(y, np.float32)
        eg = np.empty(self.blob(ENC).size, np.float32)
        dg = np.empty(self.blob(DEC).size, np.float32)
        return float(_ae_bwd(self._p, y, y.shape[0], eg, dg)), eg, dg

    def evaluate(self, x, y, w_f=1.0, w_i=1.0):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        out = np.empty(3, np.float64)
        _evaluate(self._p, x, y, x.shape[0], w_f, w_i, out)
        return out


class Trainer:
    """train::Trainer restated for one shard (trainer.hpp:139-290)."""

    def __init__(self, gan: Gan, ds_x, ds_y, partition, batch: int, seed: int,
                 abort_threshold: int = 10):
        self._x = np.ascontiguousarray(ds_x, np.float32)
        self._y = np.ascontiguousarray(ds_y, np.float32)
        self._part = np.ascontiguousarray(partition, np.uint32)
        self._p = _tr_create(gan._p, self._x, self._y, self._part, self._part.size, batch, seed,
                             abort_threshold)
        self.gan = Gan(gan.dims, gan.arch, _ptr=_tr_gan(self._p))

    def __del__(self):
        if getattr(self, "_p", None):
            _tr_destroy(self._p)
            self._p = None

    def steps(self, n: int):
        rec = np.zeros((n, 5), np.float64)
        sk = np.zeros(n, np.uint8)
        ep = np.zeros(n, np.uint32)
        done = int(_tr_steps(self._p, n, rec, sk, ep))
        return rec[:done], sk[:done], ep[:done], done < n

    @property
    def step(self) -> int:
        return int(_tr_step(self._p))
