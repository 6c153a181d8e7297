#!/usr/bin/env python3
"""bench.py — LTFB tournament training of the JAG/ICF surrogate on B200.

Metric (BASELINE.json): samples/s per box (whole job, all GPUs) and the
tournament-round time, one trainer per GPU.

Workload (configs[2]/[3]): paper dims (3 views x 4 ch x 64x64 + 15 scalars,
output_dim 49167), default SurrogateArch, B = 128, one LTFB trainer per
GPU, per-trainer partition of a synthetic JAG-shaped dataset resident in
HBM (weak scaling), tournament rounds every --interval steps at N > 1
(pairwise NCCL exchange + device-side decision). A step = one
discriminator + one generator update on every trainer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 is launched with torchrun (one rank per GPU). Prints one JSON line on
rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
# profiles/traffic.json keys carry this tag: a DRAM-traffic figure measured on
# another version of the step kernels is not reported (bump on kernel changes)
KERNEL_VERSION = "r02i"


def ae_bench(L, dims, ds, ids, B, arch, source=1024, warmup=5, steps=40):
    """Times AE pre-training steps at the bench's dims over a resident AE
    source of `source` rows (random batches of B rows per step). Roofline:
    HBM bytes of one step -- the batch's y rows, the two wide weight matrices
    read by the column passes, Adam's p/m/v read+write and the gradient read
    over both networks -- over the measured step time; flops: the five wide
    products (y We0, h Wd, h^T G, G Wd^T, y^T gz0) in fp32-equivalent terms."""
    import numpy as np
    src_ids = ids[: min(source, ids.size)]
    _, y = ds.rows(src_ids)
    y = np.ascontiguousarray(y, dtype=np.float32)
    model = L.make_cyclegan(dims, arch, 7)
    p = L.AutoencoderPretrainer(model, y, batch_size=B)
    kind = p.kind(B)
    draws = L.ae_batch_rows(11, y.shape[0], B, warmup + steps)
    for s_ in range(warmup):
        p.step(draws[s_])
    t0 = time.perf_counter()
    for s_ in range(warmup, warmup + steps):
        loss = p.step(draws[s_])
    ms = (time.perf_counter() - t0) * 1e3 / steps
    del p
    out = dims.output_dim()
    E1, D = arch.enc_hidden[0], arch.dec_hidden[-1]
    n_params = sum(int(b.size) for k, b in model.blobs.items() if k in ("enc", "dec"))
    hbm_bytes = B * out * 4 + (out * E1 + D * out) * 4 + n_params * 4 * 7
    flops = 5 * 2.0 * B * out * 64
    peaks, _ = load_peaks()
    hbm = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    ach = hbm_bytes / (ms / 1e3) / 1e9
    return {"ms_per_step": ms, "steps": steps, "batch": B, "source_rows": int(y.shape[0]),
            "kind": {2: "tcgen05 3xTF32 column passes + fused Adam", 1: "SIMT"}.get(kind, str(kind)),
            "last_loss": float(loss), "params": n_params, "gflop_per_step": flops / 1e9,
            "tflops": flops / (ms / 1e3) / 1e12,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "algorithmic_bytes_per_step": hbm_bytes},
            "timing": "wall clock per host-synced step (perf_counter), as AutoencoderPretrainer.step runs"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--dims", default="paper", choices=["paper", "desk"])
    p.add_argument("--samples-per-trainer", type=int, default=8000)
    p.add_argument("--batch", type=int, default=128)
    p.add_argument("--interval", type=int, default=100)  # RunConfig::interval (runner.hpp:64)
    p.add_argument("--e2e-steps", type=int, default=16)
    p.add_argument("--rounds", type=int, default=10, help="tournament rounds timed on their own")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-ae", action="store_true", help="skip the autoencoder pre-training timing")
    p.add_argument("--wide-kernel", type=int, default=0)
    p.add_argument("--host-data", action="store_true",
                   help="generate the partition on the host and upload it (default: k_synth on the device)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []
        self.nvml, self.samples, self._stop = None, [], threading.Event()

    def _poll_nvml(self):
        n, h = self.nvml, self.handle
        while not self._stop.is_set():
            try:
                self.samples.append((n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM),
                                     n.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        try:  # NVML polled every 5 ms: short timed regions still get samples
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            return
        except Exception:
            self.nvml = None
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            n = self.nvml
            bits = {"hw_slowdown": n.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": n.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": n.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": n.nvmlClocksEventReasonSwPowerCap}
            sm = [s for s, _ in self.samples]
            reasons = sorted({k for _, r in self.samples for k, b in bits.items() if r & b})
            loaded = [s for s in sm if s > 0.3 * self.max_mhz] or sm
            return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "source": "nvml 5 ms"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- reference --
def run_reference_bench(dims: str, trainers: int, steps: int, warmup: int, n: int, threads_total: int,
                        batch: int):
    exe = os.path.join(REPO, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None, "oracle/_ref/ref_bench not built"
    env = dict(os.environ)
    per = max(1, threads_total // max(1, trainers))
    env["OPENBLAS_NUM_THREADS"] = str(per)
    cmd = [exe, "--dims", dims, "--n", str(n), "--batch", str(batch), "--trainers", str(trainers),
           "--threads", str(min(trainers, threads_total)), "--steps", str(steps), "--warmup", str(warmup),
           "--dir", f"/tmp/ltfb_ref_bench_{os.getpid()}"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1800)
    if r.returncode != 0:
        return None, "ref_bench failed: " + r.stderr[-300:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    out["blas_threads_per_trainer"] = per
    out["cores"] = min(threads_total, per * trainers)
    return out, None


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    k = max(1, args.gpus)
    nproc = os.cpu_count() or 1
    steps = max(1, min(args.steps, 6))
    warm = max(1, min(args.warmup, 1))
    per_trainer = min(args.samples_per_trainer, 1500 if args.dims == "paper" else 4000)
    res, err = run_reference_bench(args.dims, k, steps, warm, per_trainer * k, nproc, args.batch)
    metric = "samples/sec/box"
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return 0
    value = res["samples_per_s"]
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": "samples/s",
        "n_gpus": k, "steps": steps, "warmup": warm, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference SynthGenerator, spec_seed 1, sampling_seed 1)",
        "config": {"workload": workload_name(args, k), "global_batch": args.batch * k,
                   "trainers": k, "samples_per_trainer_sample": per_trainer},
        "round_ms": res.get("round_ms"),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": res["cores"], "kind": "reference",
                         "sample": f"{steps} timed steps x {k} trainer(s), {per_trainer} samples/trainer, "
                                   f"OpenBLAS-backed Eigen shim, {res['blas_threads_per_trainer']} BLAS "
                                   f"threads/trainer"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_name(args, k):
    d = "paper 3x4x64x64 (out 49167)" if args.dims == "paper" else "desk 3x4x16x16 (out 3087)"
    return (f"LTFB {k} trainer(s), one per GPU; {d}; default SurrogateArch; B={args.batch}; "
            f"rounds every {args.interval} steps when k>1; HBM-resident partition store")


# -------------------------------------------------------------------- b200 --
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import numpy as np

    import paper_1910_02270_b200 as L

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist  # noqa: F811
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if dist is None:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    dims = L.ModalityDims.paper_scale() if args.dims == "paper" else L.ModalityDims()
    arch = L.SurrogateArch()
    k = world
    B = args.batch
    seed = 1
    # dataset: per-trainer partitions of one synthetic sweep (weak scaling)
    total = int(args.samples_per_trainer * k / 0.95)
    _, train_parts, tour_parts = L.split_dataset(total, k, 0.05, 0.05, seed, k >= 2)
    my_train, my_tour = train_parts[rank], tour_parts[rank]
    t0 = time.perf_counter()
    if args.host_data:
        need = np.concatenate([my_train, my_tour]).astype(np.uint32)
        x, y = L.synth_generate_ids(dims, need, total, sampling_seed=1, spec_seed=1)
        ds = L.SparseDataset(dims, need, x, y, total)
    else:  # rendered straight into the HBM store by the Trainer (k_synth)
        ds = L.SynthDataset(dims, total, sampling_seed=1, spec_seed=1)
        x = y = None
    gen_s = time.perf_counter() - t0

    base = L.make_cyclegan(dims, arch, L.mix_seed(seed, 0xAE0))
    base.autoencoder_frozen = True
    model = base.copy()
    L.reinit_gan_nets(model, L.mix_seed(seed, 0x1417, rank))
    cfg = L.TrainerConfig(trainer_id=rank, n_shards=1, batch_size=B, seed=L.mix_seed(seed, 0x57A7E1, rank),
                          prefetch_depth=0, train_ids=my_train, tournament_ids=my_tour, device=local,
                          wide_kernel=args.wide_kernel)
    t0 = time.perf_counter()
    tr = L.Trainer(cfg, ds, model)
    load_s = time.perf_counter() - t0
    del x, y
    comm = None
    if k > 1:
        uid = L.Comm.unique_id() if rank == 0 else b"\0" * 128
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = L.Comm(obj[0], k, rank, local)
        # NCCL connects point-to-point peers on first use: connect every pair
        # once now, outside any timed region
        L.warm_peer_links(tr, L.NcclRoundComm(comm, dist))

    rounds_ms = []
    round_counter = [0]

    def round_once():
        """tournament/ltfb.hpp:96-164 for this trainer: the pairwise payload
        exchange (NCCL send/recv of fwd||inv, 15,204 B) and the device
        decision over the tournament slice (k_eval_small + k_eval_tc over
        both candidates + k_eval_finalize, decision read back). At N = 1
        there is no peer: the incoming payload is the trainer's own
        generator copied device to device, which the decision then judges
        (an exact tie: local kept)."""
        round_counter[0] += 1
        if k > 1:
            m = L.pair_trainers(k, round_counter[0], L.mix_seed(seed, 0x9A18))
            peer = None
            for a, b in m.pairs:
                if a == rank:
                    peer = b
                elif b == rank:
                    peer = a
            if peer is None:
                return
            tr.exchange(comm, peer)
        else:
            tr._capture_from(tr)
        tr.decide_incoming()

    def run_steps(n, rounds=True):
        done = 0
        while done < n:
            chunk = min(args.interval, n - done)
            tr.train_steps_raw(chunk)
            done += chunk
            if rounds and k > 1 and chunk == args.interval:
                round_once()

    # warm-up (also compiles nothing: kernels are AOT sm_100a)
    run_steps(max(args.warmup, 3))
    round_once()
    # per-kernel CUDA-event timing (events between the kernels of every step,
    # so this pass launches the step's kernels one by one) -- for the
    # per-kernel roofline only; a first untimed pass loads those kernels
    tr.kernel_timing(True)
    run_steps(3, rounds=False)
    tr.kernel_timing(False)
    tr.kernel_timing(True)
    run_steps(min(args.steps, 100))
    kt = {name: tr.kernel_time(i) for i, name in enumerate(("gather", "small_fwd", "wide", "post", "reduce"))}
    tr.kernel_timing(False)
    tr.prepare_graphs()  # capture (not run) the step graphs outside the timed region
    # the timed region: K steps as the product runs them (CUDA graphs per
    # epoch run; at N > 1 a tournament round every --interval steps),
    # device-timed with events on the trainer's stream. The region opens
    # behind a gate the first enqueue releases and closes at the last work
    # enqueued before the host's final wait (DeviceTrainer::timer_start).
    warm_launch = tr.launch_count()
    sampler = ClockSampler(local)
    barrier()
    tr.synchronize()
    sampler.start()
    tr.timer_start()
    run_steps(args.steps)
    ms = tr.timer_stop()
    clocks = sampler.stop()
    barrier()
    launches = tr.launch_count() - warm_launch
    ms_max = max_over_ranks(ms)
    value = k * B * args.steps / (ms_max / 1e3)
    # tournament rounds on their own (the metric's second half): each round
    # device-timed on the trainer's stream, max over ranks per round
    for _ in range(max(0, args.rounds)):
        barrier()
        tr.synchronize()
        tr.timer_start()
        round_once()
        rounds_ms.append(max_over_ranks(tr.timer_stop()))
    round_ms = statistics.mean(rounds_ms) if rounds_ms else None
    # stage timeline of the streamed step (%globaltimer stamps; a separate,
    # untimed pass -- DESIGN §3a)
    stream_profile = tr.stream_profile(80) if tr.stream_mode() else {}

    # ---- e2e: same step through the C ABI with HOST buffers (pinned) -------
    import torch
    ne = max(2, args.e2e_steps)
    out = dims.output_dim()
    hx = torch.empty((ne, B, dims.input_dim), dtype=torch.float32, pin_memory=True).numpy()
    hy = torch.empty((ne, B, out), dtype=torch.float32, pin_memory=True).numpy()
    rows = np.arange(ne * B) % my_train.size
    bx, by = ds.rows(my_train[rows])
    hx[:] = bx.reshape(ne, B, -1)
    hy[:] = by.reshape(ne, B, -1)
    del bx, by
    tr.train_steps_host(2, hx[:2], hy[:2])
    barrier()
    tr.timer_start()
    tr.train_steps_host(ne, hx, hy)
    e2e_ms = max_over_ranks(tr.timer_stop())
    e2e_value = k * B * ne / (e2e_ms / 1e3)

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- autoencoder pre-training step (train_ops.hpp:71-81, runner.hpp:249-279)
    # on rank 0: the tcgen05 column passes + fused Adam over a resident AE
    # source, each step through the public AutoencoderPretrainer.step() (the
    # loss is read back per step, as the reference's loop checks it)
    ae = ae_bench(L, dims, ds, my_train, B, arch) if not args.no_ae else None

    # ---- roofline ----------------------------------------------------------
    # headline: the whole step (both step kernels) against HBM -- the
    # compulsory bytes of a step over the
    # device time per step; per kernel: the tcgen05 wide pass against HBM
    # (its algorithmic bytes over its CUDA-event launch time) and the
    # latency-bound post kernel's time and share
    peaks, peak_src = load_peaks()
    hbm = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    E1, D = arch.enc_hidden[0], arch.dec_hidden[-1]
    out_pad = (out + 3) // 4 * 4
    wide_bytes = (B * out + out * E1 + D * out + out) * 4
    step_bytes = (B * (out + dims.input_dim) + out * E1 + D * out + out) * 4
    kind, ctas = tr.wide_info()
    traffic = {}
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            for kname in ("step", "wide", "post"):
                traffic[kname] = tj.get(f"{kname}_kind{kind}_{args.dims}_{KERNEL_VERSION}")
                traffic[kname + "_warm"] = tj.get(f"{kname}_kind{kind}_{args.dims}_{KERNEL_VERSION}_warm")
        except Exception:
            traffic = {}
    step_s = ms_max / args.steps / 1e3
    ktot = sum(v[0] for v in kt.values())

    def per_launch(name):
        v = kt[name]
        return v[0] / v[1] if v[1] else None

    wide_ms = per_launch("wide")
    wide_rl = None
    if wide_ms:
        a = wide_bytes / (wide_ms / 1e3) / 1e9
        wname = {64: "wide (k_wide2, launched: phase 1 + phase 2)", 32: "wide (k_wide_tc)"}.get(tr.wide_tile(), "wide")
        wide_rl = {"kernel": wname, "bound": "hbm", "achieved": a,
                   "peak": hbm, "unit": "GB/s", "frac": a / hbm, "traffic": traffic.get("wide"),
                   "traffic_warm_l2": traffic.get("wide_warm"),
                   "algorithmic_bytes_per_launch": wide_bytes, "ms_per_launch": wide_ms,
                   "share_of_kernel_time": kt["wide"][0] / ktot if ktot else None}
    step_ach = step_bytes / step_s / 1e9
    # ---- CPU baseline: the reference itself on this box's host cores -------
    cpu = None
    if not args.no_cpu_baseline:
        res, err = run_reference_bench(args.dims, 1, 3, 1, 1000 if args.dims == "paper" else 3000,
                                       os.cpu_count() or 1, B)
        if res is not None:
            cpu = {"value": res["samples_per_s"], "unit": "samples/s", "cores": res["cores"],
                   "kind": "reference",
                   "sample": f"reference Trainer (oracle/_ref/ref_bench, OpenBLAS Eigen shim), 1 trainer, "
                             f"3 timed steps of B={B} on a 1000-sample partition; round_ms "
                             f"{res.get('round_ms')}"}
        else:
            cpu = {"value": None, "unit": "samples/s", "cores": 0, "kind": "reference", "sample": err}

    line = {
        "metric": "samples/sec/box", "value": value, "unit": "samples/s", "n_gpus": k,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SynthGenerator spec_seed 1, sampling_seed 1; random-init SurrogateArch)",
        "config": {"workload": workload_name(args, k), "global_batch": B * k, "batch_per_trainer": B,
                   "output_dim": out, "samples_per_trainer": int(my_train.size),
                   "tournament_rows": int(my_tour.size), "interval": args.interval,
                   "parallelism": f"ltfb{k} (one trainer per GPU, NCCL pairwise exchange)",
                   "l2": "inputs larger than L2: each step gathers random rows of a "
                         f"{my_train.size * out_pad * 4 / 1e9:.2f} GB HBM store; the frozen wide-layer "
                         "weights (model state, not inputs) sit in an L2 persistence window",
                   "wide_kernel": {1: "generic SIMT fp32", 2: "tcgen05 3xTF32"}.get(kind, str(kind)),
                   "wide_tile_cols": tr.wide_tile(),
                   "wide_ctas": ctas,
                   "step_mode": ("streamed: per run of steps inside an epoch, one persistent two-phase wide pass "
                                 f"({ctas} CTAs) beside one persistent 16-CTA post cluster, hand-offs through "
                                 "device counters (3 launches per run)") if tr.stream_mode()
                                else "launched: CUDA graphs of wide pass + post kernel per step"},
        "round_ms": round_ms, "rounds_timed": len(rounds_ms),
        # per-kernel times of the launched step (one kernel at a time, CUDA events):
        # the kernel-level roofline below; the timed region runs the streamed step
        "kernels_ms_per_launch": {n: (v[0] / v[1] if v[1] else None) for n, v in kt.items()},
        "roofline": {"kernel": "step (the streamed step: wide pass + post cluster)", "bound": "hbm",
                     "achieved": step_ach, "peak": hbm, "unit": "GB/s", "frac": step_ach / hbm,
                     "traffic": traffic.get("step"), "traffic_warm_l2": traffic.get("step_warm"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": step_bytes, "units": "one training step of B rows",
                     "traffic_version": KERNEL_VERSION},
        "stream_profile_us": stream_profile,
        "kernel_rooflines": {
            "wide": wide_rl,
            "post": {"kernel": "post (k_post_small)", "bound": "latency",
                     "ms_per_launch": per_launch("post"),
                     "share_of_kernel_time": kt["post"][0] / ktot if ktot else None,
                     "traffic": traffic.get("post"),
                     "note": "a chain of ~30 dependent small-net layer ops on one 16-CTA cluster; "
                             "~0.1 MB of traffic, so no HBM or tensor roofline applies (DESIGN.md)"},
            "row": {"kernel": "row (k_row_h; graph heads only)", "ms_per_launch": per_launch("gather"),
                    "launches": kt["gather"][1]},
            # the product path's post work (streamed step, one persistent cluster per run): the
            # per-step chain on the critical path after the wide pass's dec half, and the D-step
            # that runs underneath phase 2 (LTFB_STREAM_PROF stamps, averaged over a run)
            "post_streamed": {"kernel": "post cluster (k_post_loop, streamed; per step)", "bound": "latency",
                              "critical_ms_per_step": (stream_profile.get("post_chain_after_dec_us", 0) / 1e3
                                                       if stream_profile else None),
                              "overlapped_d_step_ms": (stream_profile.get("d_step_overlapped_us", 0) / 1e3
                                                       if stream_profile else None)},
        },
        "ae_pretrain": ae,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "samples/s",
                "h2d_bytes_per_step": B * (dims.input_dim + out) * 4,
                "d2h_bytes_per_step": 64,
                "path": "ltfb_trainer_train_steps_host: pinned host minibatch -> H2D per step "
                        "(copy stream, double-buffered) -> step kernels -> D2H step record"},
        "gpu_launches": launches,
        "clocks": clocks,
        "setup_s": {"generate": round(gen_s, 2), "preload": round(load_s, 2),
                    "store": "host generator + upload" if args.host_data else "device generator (k_synth)"},
    }
    print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
