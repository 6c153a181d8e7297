"""Run-directory outputs (bench/output.hpp, bench/config.hpp,
surrogate/checkpoint.hpp) against run directories written by the unmodified
reference (tests/golden/run_*, oracle/golden_dump.cpp scenario "outputs")
and nlohmann::json's own double printing (tests/golden/nlohmann_doubles.txt).
CPU only: the records are re-read from the reference's events.jsonl and
re-serialised, so every byte of config.json / events.jsonl / summary.csv /
timings.csv / best_model.bin is compared."""
import json
import os
import struct

import numpy as np
import pytest

L = pytest.importorskip("paper_1910_02270_b200")
from paper_1910_02270_b200 import outputs as O  # noqa: E402
from paper_1910_02270_b200.runner import RunHistory, trainer_summary  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = ["run_tiny_k2", "run_tiny_single"]


def _read(run, name, mode="r"):
    with open(os.path.join(GOLD, run, name), mode) as f:
        return f.read()


def test_nlohmann_double_printing():
    n = 0
    with open(os.path.join(GOLD, "nlohmann_doubles.txt")) as f:
        for line in f:
            bits, want = line.split()
            v = struct.unpack("<d", bytes.fromhex(bits)[::-1])[0]
            assert O._fmt_double(v) == want, (bits, want)
            n += 1
    assert n >= 4000
    for v, want in [(0.0, "0.0"), (-0.0, "-0.0"), (1.0, "1.0"), (1e-05, "1e-05"), (0.0001, "0.0001"),
                    (1e15, "1e+15"), (123456789012345.0, "123456789012345.0"), (5e-324, "5e-324"),
                    (float("nan"), "null"), (float("inf"), "null")]:
        assert O._fmt_double(v) == want


def test_json_layout():
    v = {"pairs": [[0, 1], [2, 3]], "a": [32, 32], "e": [], "o": {}, "s": "a\"b\\c\n\t\x01 é", "b": False,
         "u": 18446744073709551615, "neg": -5}
    assert O.dumps(v) == ('{"a":[32,32],"b":false,"e":[],"neg":-5,"o":{},"pairs":[[0,1],[2,3]],'
                          '"s":"a\\"b\\\\c\\n\\t\\u0001 é","u":18446744073709551615}')
    assert O.dumps(v, 2).splitlines()[:3] == ["{", '  "a": [32,32],', '  "b": false,']
    assert '  "pairs": [\n    [0,1],\n    [2,3]\n  ],' in O.dumps(v, 2)


@pytest.mark.parametrize("run", RUNS)
def test_config_json_and_hash(run):
    text = _read(run, "config.json")
    j = json.loads(text)
    h = j.pop("config_hash")
    cfg = O.config_from_json(j)
    assert O.config_hash(cfg) == h
    cj = O.config_to_json(cfg)
    cj["config_hash"] = h
    assert O.dumps(cj, 2) + "\n" == text


def test_config_from_json_collects_errors():
    with pytest.raises(L.ConfigError) as e:
        O.config_from_json({"trainers": "two", "bogus": 1, "mode": "ltfb", "hidden_act": "swish"})
    msg = str(e.value)
    assert "trainers (" in msg and "bogus (unknown key)" in msg and "hidden_act (" in msg
    with pytest.raises(L.ConfigError):
        O.config_from_json([1, 2])


def _history_from_events(text):
    """RunHistory rebuilt from an events.jsonl (every field round-trips)."""
    h = RunHistory()
    segs = {}
    for r in O.parse_events(text):
        t = r["type"]
        if t == "run_start":
            h.config_hash, h.mode, h.n_trainers = r["config_hash"], r["mode"], r["trainers"]
        elif t == "pretrain":
            h.pretrain.append((r["step"], r["loss"]))
        elif t == "step":
            rec = L.StepRecord(r["trainer"], r["step"], r["epoch"], r["d_loss"], r["g_total"], r["g_fwd"],
                               r["g_adv"], r["g_cyc"], r["skipped"])
            h.steps.append(rec)
            seg = segs.setdefault(r["trainer"], L.HistorySegment())
            seg.steps.append(rec)
            seg.skipped_steps += 1 if r["skipped"] else 0
        elif t == "eval":
            rec = L.EvalRecord(r["trainer"], r["step"], r["slice"], r["forward_mae"], r["inverse_mae"],
                               r["combined"])
            h.evals.append(rec)
            segs.setdefault(r["trainer"], L.HistorySegment()).evals.append(rec)
        elif t == "epoch":
            rec = L.EpochRecord(r["trainer"], r["epoch"], r["steps"], r["files_opened"], r["bytes_read"],
                                r["samples_shuffled"], r["seconds"], r["partial"])
            h.epochs.append(rec)
            segs.setdefault(r["trainer"], L.HistorySegment()).epochs.append(rec)
        elif t == "round":
            h.rounds.append(L.RoundRecord(r["round"], r["step"], [tuple(p) for p in r["pairs"]], r["bye"]))
        elif t == "trainer_round":
            h.trainer_rounds.append(L.TrainerRoundRecord(r["round"], r["step"], r["trainer"], r["peer"],
                                                         r["local_metric"], r["incoming_metric"],
                                                         r["winner"] == "incoming", r["disc_hash"]))
        elif t == "transfer":
            h.transfers.append(L.TransferRecord(r["round"], r["from"], r["to"], r["payload"], r["bytes"],
                                                r["blob_hash"]))
        elif t == "run_end":
            h.best_trainer = r["best_trainer"]
            h.best_metric = L.EvalMetric(r["best_forward_mae"], r["best_inverse_mae"], r["best_combined"])
    return h, segs


@pytest.mark.parametrize("run", RUNS)
def test_events_summary_timings_roundtrip(run):
    text = _read(run, "events.jsonl")
    h, segs = _history_from_events(text)
    assert O.events_jsonl(h) == text
    assert O.timings_csv(h) == _read(run, "timings.csv")
    # summary.csv recomputed from the records alone (runner.hpp:400-432)
    h.summaries = [trainer_summary(t, max(r.step for r in seg.steps), seg, h.trainer_rounds, h.best_trainer)
                   for t, seg in sorted(segs.items())]
    assert O.summary_csv(h) == _read(run, "summary.csv")


@pytest.mark.parametrize("run", RUNS)
def test_checkpoint_roundtrip(run, tmp_path):
    raw = _read(run, "best_model.bin", "rb")
    m = O.load_model(os.path.join(GOLD, run, "best_model.bin"))
    p = tmp_path / "m.bin"
    O.save_model(p, m)
    assert p.read_bytes() == raw
    cfg = O.config_from_json({k: v for k, v in json.loads(_read(run, "config.json")).items()
                              if k != "config_hash"})
    assert m.dims == cfg.dims
    assert tuple(m.arch.fwd_hidden) == tuple(cfg.arch.fwd_hidden)
    # init seeds recorded per net: enc / dec from the AE base model seed,
    # fwd / inv / disc from the owning trainer's reinit seed (runner.hpp:286)
    base = L.mix_seed(cfg.seed, 0xAE0)
    assert m.init_seeds["enc"] == L.mix_seed(base, 1) and m.init_seeds["dec"] == L.mix_seed(base, 2)
    best = int(json.loads(_read(run, "events.jsonl").splitlines()[-1])["best_trainer"])
    assert m.init_seeds["fwd"] == L.mix_seed(L.mix_seed(cfg.seed, 0x1417, best), 3)


def test_checkpoint_errors(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(L.IoError):
        O.load_model(p)
    raw = _read(RUNS[0], "best_model.bin", "rb")
    p.write_bytes(raw[:100])
    with pytest.raises(L.IoError):
        O.load_model(p)


def test_write_run_outputs_matches_reference_layout(tmp_path):
    run = RUNS[0]
    h, segs = _history_from_events(_read(run, "events.jsonl"))
    h.summaries = [trainer_summary(t, max(r.step for r in seg.steps), seg, h.trainer_rounds, h.best_trainer)
                   for t, seg in sorted(segs.items())]
    cfg = O.config_from_json({k: v for k, v in json.loads(_read(run, "config.json")).items()
                              if k != "config_hash"})
    m = O.load_model(os.path.join(GOLD, run, "best_model.bin"))
    O.write_run_outputs(tmp_path / "out", cfg, h, m)
    for name in ("config.json", "events.jsonl", "summary.csv", "timings.csv", "best_model.bin"):
        assert (tmp_path / "out" / name).read_bytes() == _read(run, name, "rb"), name
    assert np.array_equal(m.blobs["fwd"], O.load_model(tmp_path / "out" / "best_model.bin").blobs["fwd"])


def test_bundles_written_like_the_reference(tmp_path):
    """ensure_dataset's generation branch (generate_dataset + write_bundles,
    runner.hpp:216-227) writes the reference's LBDS bytes, and BundleDataset
    (DatasetIndex::scan_dir + read_records) reads them back."""
    cfg = O.config_from_json({k: v for k, v in json.loads(_read("run_tiny_k2", "config.json")).items()
                              if k != "config_hash"})
    cfg.data_dir = str(tmp_path / "data")
    ds = L.ensure_dataset(cfg)
    want = open(os.path.join(GOLD, "run_tiny_k2_bundle_00000.lbds"), "rb").read()
    assert (tmp_path / "data" / "bundle_00000.lbds").read_bytes() == want
    assert ds.total == cfg.gen_n and ds.n_files == (cfg.gen_n + cfg.samples_per_file - 1) // cfg.samples_per_file
    assert ds.dims == cfg.dims
    ids = np.array([0, 799, 100, 99, 450], np.uint32)
    assert list(ds.file_of(ids)) == [0, 7, 1, 0, 4]
    x, y = ds.rows(ids)
    hx, hy = L.synth_generate_ids(cfg.dims, ids, cfg.gen_n, cfg.sampling_seed, cfg.spec_seed)
    assert np.array_equal(x, hx) and np.array_equal(y, hy)
    # an existing directory is scanned, not regenerated; generation disabled
    # on an empty directory is an IoError (runner.hpp:212-215)
    assert L.ensure_dataset(cfg).total == cfg.gen_n
    cfg.data_dir, cfg.generate = str(tmp_path / "empty"), False
    with pytest.raises(L.IoError):
        L.ensure_dataset(cfg)
    with pytest.raises(L.ContractError):
        ds.rows(np.array([800], np.uint32))
