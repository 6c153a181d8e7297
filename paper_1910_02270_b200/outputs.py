"""Run directory outputs, byte-compatible with the reference's
(bench/output.hpp:14-176, bench/config.hpp:23-214).

A run directory holds
  config.json    the resolved RunConfig + its hash (config.hpp:23-75, 207-212)
  events.jsonl   every history record, one compact JSON object per line
  summary.csv    per-trainer final figures (deterministic fields only)
  timings.csv    per-epoch wall clock and counters
  best_model.bin the selected model (surrogate/checkpoint.hpp:99-160)

The reference serialises with nlohmann::json 3.11.3 (keys sorted, compact
separators, doubles as Grisu2 round-trip digits in its own fixed / exponent
layout, arrays of scalars kept on one line when pretty-printed) and
"%.17g" in the CSV files; `dumps` below reproduces those layouts so the
reference's tooling (and a byte comparison) reads B200 runs directly.
Pinned against run directories written by the unmodified reference
(tests/golden/run_*; tests/test_outputs.py).
"""
from __future__ import annotations

import json
import math
import os
import struct

import numpy as np

from .api import (NET_NAMES, ConfigError, CycleGan, IoError, ModalityDims, SurrogateArch, fnv1a64, hex64,
                  param_count)

# --------------------------------------------------------------- json ----


# nlohmann::json prints doubles with Grisu2 (Loitsch, "Printing Floating-
# Point Numbers Quickly and Accurately with Integers", PLDI 2010, in the
# dtoa_impl layout of json 3.11.3): round-trip digits that are usually but
# not always the shortest / closest (about 0.3 % of doubles differ from a
# shortest-digits printer such as Python's repr), so the digits are
# generated with the same algorithm here. 64-bit "diy" floats (f, e).
_M64 = (1 << 64) - 1
_ALPHA, _GAMMA = -60, -32


def _diy_mul(xf, xe, yf, ye):
    return ((((xf * yf) >> 32) + (1 << 31)) >> 32) & _M64, xe + ye + 64


def _normalize(f, e):
    sh = 64 - f.bit_length()
    return (f << sh) & _M64, e - sh


def _cached_power(k):
    """10^k as a 64-bit significand rounded to nearest, f * 2^e."""
    from fractions import Fraction
    v = Fraction(10) ** k
    e = (v.numerator.bit_length() - v.denominator.bit_length()) - 64
    while Fraction(2) ** (e + 64) <= v:
        e += 1
    while Fraction(2) ** (e + 63) > v:
        e -= 1
    f = v / Fraction(2) ** e
    fi = int(f)
    if f - fi >= Fraction(1, 2):
        fi += 1
    if fi >> 64:
        fi >>= 1
        e += 1
    return fi, e


_POW_CACHE = {}


def _cached_power_for(e):
    f = _ALPHA - e - 1
    q = abs(f * 78913) >> 18  # C++ integer division truncates towards zero
    k = (q if f >= 0 else -q) + (1 if f > 0 else 0)
    index = (300 + k + 7) // 8
    dk = -300 + 8 * index
    if dk not in _POW_CACHE:
        _POW_CACHE[dk] = _cached_power(dk)
    cf, ce = _POW_CACHE[dk]
    return cf, ce, dk


def _grisu2_digits(v: float):
    """(digits, decimal_exponent): value = digits x 10^decimal_exponent."""
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    if E == 0:
        vf, ve = F, 1 - 1075
    else:
        vf, ve = F + (1 << 52), E - 1075
    closer = F == 0 and E > 1
    mpf, mpe = 2 * vf + 1, ve - 1
    if closer:
        mmf, mme = 4 * vf - 1, ve - 2
    else:
        mmf, mme = 2 * vf - 1, ve - 1
    wpf, wpe = _normalize(mpf, mpe)
    wmf, wme = (mmf << (mme - wpe)) & _M64, wpe
    wf, we = _normalize(vf, ve)
    cf, ce, ck = _cached_power_for(wpe)
    w_f, w_e = _diy_mul(wf, we, cf, ce)
    lo_f, _ = _diy_mul(wmf, wme, cf, ce)
    hi_f, hi_e = _diy_mul(wpf, wpe, cf, ce)
    Mm, Mp = lo_f + 1, hi_f - 1
    dec_exp = -ck
    # digit generation (grisu2_digit_gen)
    delta = (Mp - Mm) & _M64
    dist = (Mp - w_f) & _M64
    sh = -hi_e
    one_f = 1 << sh
    p1 = Mp >> sh
    p2 = Mp & (one_f - 1)
    n = len(str(p1)) if p1 else 1
    pow10 = 10 ** (n - 1)
    buf = []

    def rnd(dist, delta, rest, ten_k):
        while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
            buf[-1] -= 1
            rest += ten_k

    while n > 0:
        d, p1 = divmod(p1, pow10)
        buf.append(d)
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            dec_exp += n
            rnd(dist, delta, rest, pow10 << sh)
            return "".join(map(str, buf)), dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 = (p2 * 10) & _M64
        buf.append(p2 >> sh)
        p2 &= one_f - 1
        m += 1
        delta = (delta * 10) & _M64
        dist = (dist * 10) & _M64
        if p2 <= delta:
            break
    dec_exp -= m
    rnd(dist, delta, p2, one_f)
    return "".join(map(str, buf)), dec_exp


def _fmt_double(v: float) -> str:
    """nlohmann::detail::to_chars: Grisu2 digits d1..dk with the decimal
    point at n; fixed for -4 < n <= 15, else d.ddde+XX."""
    if math.isnan(v) or math.isinf(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    digits, dec_exp = _grisu2_digits(abs(v))
    k = len(digits)
    n = k + dec_exp
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    body = digits if k == 1 else digits[0] + "." + digits[1:]
    return sign + body + "e" + ("-" if e < 0 else "+") + (f"{abs(e):02d}")


def _fmt_string(s: str) -> str:
    out = ['"']
    for ch in s:
        c = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif c < 0x20:
            out.append(f"\\u{c:04x}")
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _scalar(v) -> str:
    if v is None:
        return "null"
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _fmt_double(float(v))
    if isinstance(v, str):
        return _fmt_string(v)
    raise TypeError(f"cannot serialise {type(v).__name__}")


def dumps(v, indent: int | None = None, _level: int = 0) -> str:
    """nlohmann::json::dump(indent) of a value built from dict / list /
    str / int / float / bool / None (objects are key-sorted)."""
    if isinstance(v, dict):
        keys = sorted(v)
        if not keys:
            return "{}"
        if indent is None:
            return "{" + ",".join(_fmt_string(k) + ":" + dumps(v[k]) for k in keys) + "}"
        pad, pad1 = " " * (indent * _level), " " * (indent * (_level + 1))
        return "{\n" + ",\n".join(pad1 + _fmt_string(k) + ": " + dumps(v[k], indent, _level + 1)
                                  for k in keys) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        flat = not any(isinstance(e, (dict, list, tuple)) for e in v)
        if indent is None or flat:
            return "[" + ",".join(dumps(e) for e in v) + "]"
        pad, pad1 = " " * (indent * _level), " " * (indent * (_level + 1))
        return "[\n" + ",\n".join(pad1 + dumps(e, indent, _level + 1) for e in v) + "\n" + pad + "]"
    return _scalar(v)


def fmt_double(v: float) -> str:
    """output.hpp:25-29: "%.17g"."""
    return "%.17g" % v


# ------------------------------------------------------------- config ----
_ACT_NAMES = ("identity", "relu", "leaky_relu", "tanh", "sigmoid")
_ACT_KIND = {n: i for i, n in enumerate(_ACT_NAMES)}


def config_to_json(cfg) -> dict:
    """config.hpp:23-75 (to_json of a RunConfig)."""
    d, a = cfg.dims or ModalityDims(), cfg.arch or SurrogateArch()
    mode = cfg.mode.replace("_", "-")
    return {
        "data_dir": cfg.data_dir, "generate": bool(cfg.generate), "gen_n": int(cfg.gen_n),
        "samples_per_file": int(cfg.samples_per_file), "sampling_seed": int(cfg.sampling_seed),
        "spec_seed": int(cfg.spec_seed), "noise_level": float(cfg.noise_level),
        "input_dim": d.input_dim, "latent_dim": d.latent_dim, "scalar_dim": d.scalar_dim,
        "image_views": d.image_views, "image_channels": d.image_channels, "image_h": d.image_h,
        "image_w": d.image_w,
        "enc_hidden": list(a.enc_hidden), "dec_hidden": list(a.dec_hidden), "fwd_hidden": list(a.fwd_hidden),
        "inv_hidden": list(a.inv_hidden), "disc_hidden": list(a.disc_hidden),
        "hidden_act": a.hidden_act, "leaky_slope": float(a.hidden_slope),
        "lambda_adv": float(a.lambda_adv), "lambda_cyc": float(a.lambda_cyc),
        "lr": float(a.lr), "beta1": float(a.beta1), "beta2": float(a.beta2), "adam_eps": float(a.eps),
        "mode": mode, "trainers": int(cfg.trainers), "shards": int(cfg.shards),
        "batch_size": int(cfg.batch_size), "interval": int(cfg.interval), "step_budget": int(cfg.step_budget),
        "ae_steps": int(cfg.ae_steps), "data_store": cfg.data_store, "threads": int(cfg.threads),
        "seed": int(cfg.seed), "validation_fraction": float(cfg.validation_fraction),
        "tournament_fraction": float(cfg.tournament_fraction), "lr_jitter": float(cfg.lr_jitter),
        "store_budget_mb": int(cfg.store_budget_mb), "numeric_abort_threshold": int(cfg.numeric_abort_threshold),
        "prefetch_depth": int(cfg.prefetch_depth), "w_forward": float(cfg.w_f), "w_inverse": float(cfg.w_i),
    }


_KNOWN = ("data_dir", "generate", "gen_n", "samples_per_file", "sampling_seed", "spec_seed", "noise_level",
          "input_dim", "latent_dim", "scalar_dim", "image_views", "image_channels", "image_h", "image_w",
          "enc_hidden", "dec_hidden", "fwd_hidden", "inv_hidden", "disc_hidden", "hidden_act", "leaky_slope",
          "lambda_adv", "lambda_cyc", "lr", "beta1", "beta2", "adam_eps", "mode", "trainers", "shards",
          "batch_size", "interval", "step_budget", "ae_steps", "data_store", "threads", "seed",
          "validation_fraction", "tournament_fraction", "lr_jitter", "store_budget_mb",
          "numeric_abort_threshold", "prefetch_depth", "w_forward", "w_inverse")


def config_from_json(j: dict):
    """config.hpp:77-202: strict parse; every bad or unknown key is
    collected and reported in one ConfigError."""
    from .runner import RunConfig
    if not isinstance(j, dict):
        raise ConfigError("config root must be a JSON object")
    cfg = RunConfig()
    dims = ModalityDims()
    arch = SurrogateArch()
    errors = []

    def uint(v):
        if isinstance(v, bool) or not isinstance(v, int) or v < 0:
            raise TypeError("type must be number")
        return v

    def sint(v):
        if isinstance(v, bool) or not isinstance(v, int):
            raise TypeError("type must be number")
        return v

    def num(v):
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise TypeError("type must be number")
        return float(v)

    def boolean(v):
        if not isinstance(v, bool):
            raise TypeError("type must be boolean")
        return v

    def string(v):
        if not isinstance(v, str):
            raise TypeError("type must be string")
        return v

    def widths(v):
        if not isinstance(v, list):
            raise TypeError("type must be array")
        return tuple(uint(e) for e in v)

    def act(v):
        if string(v) not in _ACT_KIND:
            raise ConfigError("unknown activation name: " + v)
        return v

    def mode(v):
        if string(v) not in ("single", "ltfb", "k-independent", "k_independent"):
            raise ConfigError("unknown run mode: " + v)
        return v.replace("_", "-")

    def store(v):
        if string(v) not in ("preload", "dynamic"):
            raise ConfigError("unknown data store mode: " + v)
        return v

    setters = {
        "data_dir": (cfg, "data_dir", string), "generate": (cfg, "generate", boolean),
        "gen_n": (cfg, "gen_n", uint), "samples_per_file": (cfg, "samples_per_file", uint),
        "sampling_seed": (cfg, "sampling_seed", uint), "spec_seed": (cfg, "spec_seed", uint),
        "noise_level": (cfg, "noise_level", num),
        "input_dim": (dims, "input_dim", uint), "latent_dim": (dims, "latent_dim", uint),
        "scalar_dim": (dims, "scalar_dim", uint), "image_views": (dims, "image_views", uint),
        "image_channels": (dims, "image_channels", uint), "image_h": (dims, "image_h", uint),
        "image_w": (dims, "image_w", uint),
        "enc_hidden": (arch, "enc_hidden", widths), "dec_hidden": (arch, "dec_hidden", widths),
        "fwd_hidden": (arch, "fwd_hidden", widths), "inv_hidden": (arch, "inv_hidden", widths),
        "disc_hidden": (arch, "disc_hidden", widths), "hidden_act": (arch, "hidden_act", act),
        "leaky_slope": (arch, "hidden_slope", num), "lambda_adv": (arch, "lambda_adv", num),
        "lambda_cyc": (arch, "lambda_cyc", num), "lr": (arch, "lr", num), "beta1": (arch, "beta1", num),
        "beta2": (arch, "beta2", num), "adam_eps": (arch, "eps", num),
        "mode": (cfg, "mode", mode), "trainers": (cfg, "trainers", sint), "shards": (cfg, "shards", sint),
        "batch_size": (cfg, "batch_size", uint), "interval": (cfg, "interval", uint),
        "step_budget": (cfg, "step_budget", uint), "ae_steps": (cfg, "ae_steps", uint),
        "data_store": (cfg, "data_store", store), "threads": (cfg, "threads", sint), "seed": (cfg, "seed", uint),
        "validation_fraction": (cfg, "validation_fraction", num),
        "tournament_fraction": (cfg, "tournament_fraction", num), "lr_jitter": (cfg, "lr_jitter", num),
        "store_budget_mb": (cfg, "store_budget_mb", uint),
        "numeric_abort_threshold": (cfg, "numeric_abort_threshold", sint),
        "prefetch_depth": (cfg, "prefetch_depth", sint), "w_forward": (cfg, "w_f", num),
        "w_inverse": (cfg, "w_i", num),
    }
    for key in _KNOWN:
        if key in j:
            obj, attr, conv = setters[key]
            try:
                setattr(obj, attr, conv(j[key]))
            except (TypeError, ValueError, ConfigError) as e:
                errors.append(f"{key} ({e})")
    for key in j:
        if key not in _KNOWN:
            errors.append(f"{key} (unknown key)")
    if errors:
        raise ConfigError("invalid config keys:" + "".join(" " + e + ";" for e in errors))
    cfg.dims, cfg.arch = dims, arch
    return cfg


def config_hash(cfg) -> str:
    """config.hpp:207-212: FNV-1a of the compact dump without `threads`."""
    j = config_to_json(cfg)
    del j["threads"]
    return hex64(fnv1a64(dumps(j).encode()))


# ------------------------------------------------------------- events ----
def events_jsonl(h) -> str:
    """output.hpp:31-110."""
    lines = [dumps({"type": "run_start", "config_hash": h.config_hash, "mode": h.mode,
                    "trainers": h.n_trainers})]
    for step, loss in h.pretrain:
        lines.append(dumps({"type": "pretrain", "step": int(step), "loss": float(loss)}))
    for r in h.steps:
        lines.append(dumps({"type": "step", "trainer": r.trainer, "step": r.step, "epoch": r.epoch,
                            "d_loss": r.d_loss, "g_total": r.g_total, "g_fwd": r.g_fwd, "g_adv": r.g_adv,
                            "g_cyc": r.g_cyc, "skipped": bool(r.skipped)}))
    for r in h.evals:
        lines.append(dumps({"type": "eval", "trainer": r.trainer, "step": r.step, "slice": r.slice,
                            "forward_mae": r.forward_mae, "inverse_mae": r.inverse_mae,
                            "combined": r.combined}))
    for r in h.epochs:
        lines.append(dumps({"type": "epoch", "trainer": r.trainer, "epoch": r.epoch, "steps": r.steps,
                            "files_opened": r.files_opened, "bytes_read": r.bytes_read,
                            "samples_shuffled": r.samples_shuffled, "seconds": r.seconds,
                            "partial": bool(r.partial)}))
    for r in h.rounds:
        lines.append(dumps({"type": "round", "round": r.round, "step": r.step,
                            "pairs": [[int(a), int(b)] for a, b in r.pairs], "bye": r.bye}))
    for r in h.trainer_rounds:
        lines.append(dumps({"type": "trainer_round", "round": r.round, "step": r.step, "trainer": r.trainer,
                            "peer": r.peer, "local_metric": r.local_metric, "incoming_metric": r.incoming_metric,
                            "winner": "incoming" if r.kept_incoming else "local", "disc_hash": r.disc_hash}))
    for r in h.transfers:
        lines.append(dumps({"type": "transfer", "round": r.round, "from": r.from_trainer, "to": r.to_trainer,
                            "payload": r.payload, "bytes": r.bytes, "blob_hash": r.blob_hash}))
    bm = h.best_metric
    lines.append(dumps({"type": "run_end", "best_trainer": h.best_trainer,
                        "best_forward_mae": bm.forward_mae if bm else 0.0,
                        "best_inverse_mae": bm.inverse_mae if bm else 0.0,
                        "best_combined": bm.combined if bm else 0.0}))
    return "".join(line + "\n" for line in lines)


_SUMMARY_HEADER = ("config_hash,mode,n_trainers,trainer,steps,epochs_completed,"
                   "final_d_loss,final_g_total,final_g_fwd,final_g_adv,final_g_cyc,"
                   "final_val_forward_mae,final_val_inverse_mae,final_val_combined,"
                   "rounds,incoming_adopted,files_opened,bytes_read,samples_shuffled,"
                   "skipped_steps,is_best\n")


def summary_csv(h) -> str:
    """output.hpp:112-141."""
    out = [_SUMMARY_HEADER]
    for s in h.summaries:
        f = fmt_double
        out.append(",".join([
            h.config_hash, h.mode, str(h.n_trainers), str(s.trainer), str(s.steps), str(s.epochs_completed),
            f(s.final_d_loss), f(s.final_g_total), f(s.final_g_fwd), f(s.final_g_adv), f(s.final_g_cyc),
            f(s.final_val_forward_mae), f(s.final_val_inverse_mae), f(s.final_val_combined),
            str(s.rounds), str(s.incoming_adopted), str(s.files_opened), str(s.bytes_read),
            str(s.samples_shuffled), str(s.skipped_steps), "1" if s.is_best else "0"]) + "\n")
    return "".join(out)


def timings_csv(h) -> str:
    """output.hpp:143-155."""
    out = ["trainer,epoch,steps,seconds,files_opened,bytes_read,samples_shuffled,partial\n"]
    for e in h.epochs:
        out.append(f"{e.trainer},{e.epoch},{e.steps},{fmt_double(e.seconds)},{e.files_opened},"
                   f"{e.bytes_read},{e.samples_shuffled},{1 if e.partial else 0}\n")
    return "".join(out)


# --------------------------------------------------------- checkpoint ----
_MAGIC = b"LBCK"
_VERSION = 1


def _net_widths(dims: ModalityDims, arch: SurrogateArch, net: str):
    ins = {"enc": dims.output_dim(), "dec": dims.latent_dim, "fwd": dims.input_dim, "inv": dims.latent_dim,
           "disc": dims.latent_dim}
    outs = {"enc": dims.latent_dim, "dec": dims.output_dim(), "fwd": dims.latent_dim, "inv": dims.input_dim,
            "disc": 1}
    return [ins[net]] + list(getattr(arch, net + "_hidden")) + [outs[net]]


def save_model(path, model: CycleGan):
    """checkpoint.hpp:99-122 (write to path.tmp, then rename)."""
    d, a = model.dims, model.arch
    buf = bytearray(_MAGIC)
    buf += struct.pack("<I", _VERSION)
    buf += struct.pack("<7I", *d.as_tuple())
    buf += struct.pack("<d", float(np.float32(model.lambda_adv)))
    buf += struct.pack("<d", float(np.float32(model.lambda_cyc)))
    hidden = _ACT_KIND[a.hidden_act]
    for net in NET_NAMES:
        w = _net_widths(d, a, net)
        buf += struct.pack("<I", len(w))
        buf += struct.pack(f"<{len(w)}I", *w)
        for layer in range(len(w) - 1):
            last = layer + 2 >= len(w)
            buf += struct.pack("<Id", 0 if last else hidden, 0.01 if last else float(a.hidden_slope))
        buf += struct.pack("<Q", int(model.init_seeds[net]))
        blob = np.ascontiguousarray(model.blobs[net], "<f4")
        buf += struct.pack("<Q", blob.size)
        buf += blob.tobytes()
    tmp = str(path) + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(buf)
        os.replace(tmp, path)
    except OSError as e:
        raise IoError(f"cannot write checkpoint {path}: {e}") from e


def load_model(path) -> CycleGan:
    """checkpoint.hpp:124-160."""
    ctx = str(path)
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError("cannot open checkpoint " + ctx) from e
    pos = 0

    def take(fmt):
        nonlocal pos
        n = struct.calcsize(fmt)
        if pos + n > len(raw):
            raise IoError("truncated read while parsing " + ctx)
        v = struct.unpack_from(fmt, raw, pos)
        pos += n
        return v

    if raw[:4] != _MAGIC:
        raise IoError("bad checkpoint magic in " + ctx)
    pos = 4
    if take("<I")[0] != _VERSION:
        raise IoError("unsupported checkpoint version in " + ctx)
    dims = ModalityDims(*take("<7I"))
    lam_adv, lam_cyc = take("<2d")
    specs, blobs, seeds = {}, {}, {}
    for net in NET_NAMES:
        (nw,) = take("<I")
        if nw < 2 or nw > 1024:
            raise IoError("corrupt checkpoint (layer count) in " + ctx)
        widths = list(take(f"<{nw}I"))
        acts = [take("<Id") for _ in range(nw - 1)]
        (seeds[net],) = take("<Q")
        (count,) = take("<Q")
        total = sum(widths[i] * widths[i + 1] + widths[i + 1] for i in range(nw - 1))
        if count != total:
            raise IoError("checkpoint blob length does not match manifest in " + ctx)
        if pos + 4 * count > len(raw):
            raise IoError("truncated read while parsing " + ctx)
        blobs[net] = np.frombuffer(raw, "<f4", count, pos).astype(np.float32)
        pos += 4 * count
        specs[net] = (widths, acts)
    hid = specs["fwd"][1][0] if len(specs["fwd"][1]) > 1 else (_ACT_KIND["leaky_relu"], 0.2)
    arch = SurrogateArch(enc_hidden=tuple(specs["enc"][0][1:-1]), dec_hidden=tuple(specs["dec"][0][1:-1]),
                         fwd_hidden=tuple(specs["fwd"][0][1:-1]), inv_hidden=tuple(specs["inv"][0][1:-1]),
                         disc_hidden=tuple(specs["disc"][0][1:-1]), hidden_act=_ACT_NAMES[hid[0]],
                         hidden_slope=hid[1], lambda_adv=lam_adv, lambda_cyc=lam_cyc)
    m = CycleGan(dims, arch)
    for net in NET_NAMES:
        if blobs[net].size != param_count(dims, arch, NET_NAMES.index(net)):
            raise IoError("checkpoint blob length does not match manifest in " + ctx)
        m.blobs[net] = blobs[net]
        m.opt[net].m = np.zeros_like(blobs[net])
        m.opt[net].v = np.zeros_like(blobs[net])
    m.init_seeds = dict(seeds)
    m.lambda_adv, m.lambda_cyc = np.float32(lam_adv), np.float32(lam_cyc)
    return m


# ------------------------------------------------------------ run dir ----
def write_run_outputs(out_dir, cfg, history, best_model: CycleGan | None = None):
    """output.hpp:159-176."""
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError as e:
        raise IoError(f"cannot create output directory {out_dir}") from e
    cj = config_to_json(cfg)
    cj["config_hash"] = history.config_hash
    files = {"config.json": dumps(cj, 2) + "\n", "events.jsonl": events_jsonl(history),
             "summary.csv": summary_csv(history), "timings.csv": timings_csv(history)}
    for name, text in files.items():
        p = os.path.join(out_dir, name)
        try:
            with open(p, "wb") as f:
                f.write(text.encode())
        except OSError as e:
            raise IoError(f"cannot open {p} for writing") from e
    if best_model is not None:
        save_model(os.path.join(out_dir, "best_model.bin"), best_model)


def parse_events(text: str) -> list[dict]:
    """events.jsonl -> list of records (floats round-trip exactly)."""
    return [json.loads(line) for line in text.splitlines() if line]
