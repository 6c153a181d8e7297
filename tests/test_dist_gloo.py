"""Multi-process (world size 2, gloo, CPU) test of the multi-GPU host logic:
runner.distributed_round -- local pairing, pairwise generator exchange over
torch.distributed, per-rank decision and adoption -- replaying the
reference's tiny_k2 LTFB experiment with an oracle-backed CPU trainer
(tests/_dist_worker.py). Checked bit-exactly against the reference's own
run (tests/golden/tournament.npz): split, AE pre-training, every step loss,
every round's pairing, metrics, decision and payload size."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def ranks(tmp_path_factory):
    pytest.importorskip("torch")
    out = tmp_path_factory.mktemp("dist")
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r), WORLD_SIZE="2",
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, os.path.join(REPO, "tests", "_dist_worker.py"), str(out)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        logs.append(o.decode(errors="replace"))
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(out / f"rank{r}.npz")) for r in range(2)]


def test_split_and_pretraining_replicated_identically(ranks, golden):
    g = golden("tournament")
    for r in ranks:
        assert np.array_equal(r["split_train"], g["tiny_k2_split_train_ids"])
        assert np.array_equal(r["split_val"], g["tiny_k2_split_validation"])
        assert np.array_equal(r["pretrain"], g["tiny_k2_pretrain_loss"])
        assert np.array_equal(r["ae_enc"], g["tiny_k2_ae_enc"])
        assert np.array_equal(r["ae_dec"], g["tiny_k2_ae_dec"])


def test_steps_match_reference(ranks, golden):
    g = golden("tournament")
    for t, r in enumerate(ranks):
        sel = g["tiny_k2_steps_trainer"] == t
        ref = np.stack([g["tiny_k2_steps_" + k][sel] for k in ("d_loss", "g_total", "g_fwd", "g_adv", "g_cyc")], 1)
        assert np.array_equal(r["steps"], ref)


def test_rounds_match_reference(ranks, golden):
    g = golden("tournament")
    pairs = np.stack([g["tiny_k2_round_pair_a"], g["tiny_k2_round_pair_b"]], 1)
    for t, r in enumerate(ranks):
        assert np.array_equal(r["pairs"], pairs)
        sel = g["tiny_k2_tr_trainer"] == t
        assert np.array_equal(r["tr_round"], g["tiny_k2_tr_round"][sel])
        assert np.array_equal(r["tr_peer"], g["tiny_k2_tr_peer"][sel])
        assert np.array_equal(r["tr_local"], g["tiny_k2_tr_local"][sel])
        assert np.array_equal(r["tr_incoming"], g["tiny_k2_tr_incoming"][sel])
        assert np.array_equal(r["tr_kept"].astype(np.int64), g["tiny_k2_tr_kept"][sel].astype(np.int64))
        sent = g["tiny_k2_xf_from"] == t
        assert np.array_equal(r["xf_bytes"], g["tiny_k2_xf_bytes"][sent])
        assert np.array_equal(r["xf_to"], g["tiny_k2_xf_to"][sent])


def test_sharded_validation_equals_whole_slice(ranks):
    """runner.sharded_validation over 2 gloo ranks (each holding half of the
    validation slice, every model evaluated on every shard, metrics combined
    in rank order) gives the whole-slice metrics of both models on both
    ranks (up to double summation order)."""
    for r in ranks:
        a, b = r["val_sharded"], r["val_full"]
        assert a.shape == b.shape == (2, 3)
        assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) < 1e-12
    assert np.array_equal(ranks[0]["val_sharded"], ranks[1]["val_sharded"])
