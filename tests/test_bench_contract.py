"""bench.py's JSON line (the driver's contract): one short N=1 run through the
product path, checked for the keys and the internal consistency the judge
reads (value vs ms_per_step, roofline fractions, e2e bytes, launches)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    steps, warmup = 20, 3
    p = subprocess.run([sys.executable, "bench.py", "--steps", str(steps), "--warmup", str(warmup),
                        "--no-cpu-baseline"], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "kernel_rooflines",
                "round_ms", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    B = d["config"]["global_batch"]
    # value = samples of the K timed steps / their device time
    assert d["value"] == pytest.approx(B / (d["ms_per_step"] / 1e3), rel=1e-6)
    r = d["roofline"]  # the whole step against HBM (the headline)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9) and 0 < r["frac"] < 1
    assert r["achieved"] == pytest.approx(r["algorithmic_bytes_per_launch"] / (d["ms_per_step"] / 1e3) / 1e9,
                                          rel=1e-6)
    w = d["kernel_rooflines"]["wide"]
    assert w["frac"] == pytest.approx(w["achieved"] / w["peak"], rel=1e-9)
    # (the streamed step overlaps the wide pass's phase 1 with the post cluster, so
    # since round 2h it is faster than the launched wide pass timed alone)
    assert 0 < r["frac"] < 1 and 0 < w["frac"] < 1
    # a tournament round is timed at N = 1 too (own payload, device decision)
    assert d["round_ms"] is not None and d["round_ms"] > 0 and d["rounds_timed"] >= 1
    out = d["config"]["output_dim"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == B * (5 + out) * 4 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < d["value"]
    # launched steps: the wide pass and the post kernel every step; the
    # streamed step: a persistent wide pass + post cluster (+ init) per run
    if d["config"]["step_mode"].startswith("streamed"):
        assert d["gpu_launches"] >= 3
    else:
        assert d["gpu_launches"] >= 2 * steps
