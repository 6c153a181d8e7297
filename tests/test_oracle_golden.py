"""Pins the plain-C oracle (oracle/ltfb_oracle.c) to the golden vectors the
UNMODIFIED reference produced (tests/golden/*.npz, see oracle/make_golden.py).

Everything here is bit-exact: the oracle restates the reference loop for
loop, and both use the strict k-ascending fp32 GEMM order.  Once pinned, the
oracle is the checker for the CUDA path on seeded inputs of any size.
"""
import numpy as np
import pytest

TINY_DIMS = [5, 20, 15, 1, 1, 4, 4]
DESK_DIMS = [5, 20, 15, 3, 4, 16, 16]
PAPER_DIMS = [5, 20, 15, 3, 4, 64, 64]


def test_rng(golden, oracle):
    g = golden("rng")
    parts = [(1,), (1, 2), (42, 0xA11), (7, 3, 0x9A12), (0,), (2**64 - 1, 5),
             (1, 0x57A7E1, 3), (12345, 0, 0x5CAFF1E)]
    assert [oracle.mix_seed(*p) for p in parts] == [int(v) for v in g["mix_seed"]]
    r = oracle.Rng(12345)
    assert [r.next() for _ in range(32)] == [int(v) for v in g["next"]]
    assert [r.uniform() for _ in range(16)] == list(g["uniform"])
    got = [r.below(int(n)) for n in g["below_n"] for _ in range(8)]
    assert got == [int(v) for v in g["below"]]
    assert [r.normal() for _ in range(8)] == list(g["normal"])
    assert np.array_equal(oracle.Rng(99).shuffle_u32(np.arange(57)), g["shuffle57_seed99"])
    assert oracle.fnv1a64(b"hello") == int(g["fnv_hello"][0])


def test_partition_pairing_split(golden, oracle):
    g = golden("plan")
    for tag, n, k, seed in (("part_100_4_5_", 100, 4, 5), ("part_1000_7_11_", 1000, 7, 11)):
        parts = oracle.partition_dataset(np.arange(n), k, seed)
        assert np.array_equal(np.concatenate(parts), g[tag + "ids"])
        assert [p.size for p in parts] == list(g[tag + "sizes"])
    i = 0
    byes = []
    for k in (2, 3, 4, 5, 8):
        for rnd in range(1, 26):
            pairs, bye = oracle.pair_trainers(k, rnd, 0x1234)
            byes.append(bye)
            for a, b in pairs:
                assert (g["pair_k"][i], g["pair_round"][i], g["pair_a"][i], g["pair_b"][i]) == (k, rnd, a, b)
                i += 1
    assert i == g["pair_a"].size
    assert byes == list(g["pair_byes"])
    for total, k, seed in ((800, 2, 42), (16000, 4, 101), (16000, 8, 1)):
        pfx = f"split_{total}_{k}_"
        val, train, tour = oracle.split_dataset(total, k, 0.05, 0.05, seed, k >= 2)
        assert np.array_equal(val, g[pfx + "validation"])
        assert np.array_equal(np.concatenate(train), g[pfx + "train_ids"])
        assert np.array_equal(np.concatenate(tour), g[pfx + "tour_ids"])
        assert [t.size for t in train] == list(g[pfx + "train_sizes"])


def test_epoch_plan(golden, oracle):
    g = golden("plan")
    _, train, _ = oracle.split_dataset(800, 2, 0.05, 0.05, 42, True)
    seed = int(g["plan_seed"][0])
    assert seed == oracle.mix_seed(42, 0x57A7E1, 0)
    for e in (1, 2, 3):
        perm = oracle.plan_perm(train[0], e, seed)
        assert np.array_equal(perm, g[f"plan_perm_e{e}"])
        sl = g[f"plan_slices_e{e}"].reshape(-1, 2)
        n = perm.size
        exp = [(b, min(n, b + 32)) for b in range(0, n, 32)]
        assert [tuple(map(int, s)) for s in sl] == exp


def test_synth(golden, oracle):
    g = golden("synth")
    x, y = oracle.Synth(TINY_DIMS, 3).generate(200, 17)
    assert np.array_equal(x.ravel(), g["tiny_x"]) and np.array_equal(y.ravel(), g["tiny_y"])
    x, y = oracle.Synth(TINY_DIMS, 3, 0.1).generate(20, 17)
    assert np.array_equal(y.ravel(), g["tiny_noisy_y"])
    gs = oracle.grid_side(16000)
    assert gs == int(g["grid_side_16000"][0])
    desk = oracle.Synth(DESK_DIMS, 1)
    ys = [desk.sample(oracle.sweep_point(int(i), gs, 1))[1] for i in g["desk_which"]]
    assert np.array_equal(np.concatenate(ys), g["desk_y"])
    paper = oracle.Synth(PAPER_DIMS, 1)
    assert np.array_equal(paper.sample(oracle.sweep_point(12345, gs, 1))[1], g["paper_y"])


def test_mlp_loss_adam(golden, oracle):
    g = golden("nn")
    for pfx in ("mlpA_", "mlpB_", "mlpC_"):
        w, acts, slopes = g[pfx + "widths"], g[pfx + "acts"], g[pfx + "slopes"]
        blob = oracle.mlp_init(w, int(g[pfx + "init_seed"][0]))
        assert np.array_equal(blob, g[pfx + "params"])
        x = g[pfx + "x"].reshape(-1, int(w[0]))
        out = oracle.mlp_forward(w, acts, slopes, blob, x)
        assert np.array_equal(out.ravel(), g[pfx + "out"])
        assert np.array_equal(out.ravel(), g[pfx + "apply"])
        pg, gi = oracle.mlp_backward(w, acts, slopes, blob, x, g[pfx + "gout"])
        assert np.array_equal(pg, g[pfx + "pgrad"])
        assert np.array_equal(gi.ravel(), g[pfx + "gin"])
    v, grad = oracle.mae(g["mae_p"], g["mae_t"])
    assert v == g["mae_value"][0] and np.array_equal(grad, g["mae_grad"])
    assert grad[4] == 0.0
    probs = np.array([oracle.stable_sigmoid(float(z)) for z in g["bce_logits"]], np.float32)
    assert np.array_equal(probs, g["bce_probs"])
    v, grad = oracle.bce(g["bce_probs"], g["bce_labels"])
    assert v == g["bce_value"][0] and np.array_equal(grad, g["bce_grad"])
    p = g["adam_p0"].copy()
    m, vv, t = np.zeros_like(p), np.zeros_like(p), 0
    for s in (1, 2, 3):
        t, ok = oracle.adam_step(p, g[f"adam_g{s}"], m, vv, t)
        assert ok and t == s
        assert np.array_equal(p, g[f"adam_p{s}"])
        assert np.array_equal(m, g[f"adam_m{s}"]) and np.array_equal(vv, g[f"adam_v{s}"])
    bad = g["adam_g1"].copy()
    bad[3] = np.inf
    before = p.copy()
    t2, ok = oracle.adam_step(p, bad, m, vv, t)
    assert not ok and t2 == t and np.array_equal(p, before)


def _surrogate_check(g, oracle, pfx, dims, arch, x, y, full_ae):
    gan = oracle.Gan(dims, arch, int(g[pfx + "seed"][0]))
    h = g[pfx + "init_hashes"]
    for i, net in enumerate(range(5)):
        assert oracle.fnv1a64(gan.blob(net)) == int(h[i]), oracle.NET_NAMES[net]
    dl, dg = gan.disc_backward(x, y)
    assert dl == g[pfx + "d_loss"][0] and np.array_equal(dg, g[pfx + "disc_grad"])
    losses, fg, ig = gan.gen_backward(x, y)
    assert np.array_equal(losses, g[pfx + "gen_losses"])
    assert np.array_equal(fg, g[pfx + "fwd_grad"]) and np.array_equal(ig, g[pfx + "inv_grad"])
    al, eg, decg = gan.ae_backward(y)
    assert al == g[pfx + "ae_loss"][0]
    if full_ae:
        assert np.array_equal(eg, g[pfx + "enc_grad"]) and np.array_equal(decg, g[pfx + "dec_grad"])
    else:
        s = int(g[pfx + "enc_grad_strided_stride"][0])
        assert np.array_equal(eg[::s], g[pfx + "enc_grad_strided"])
        assert np.array_equal(decg[::s], g[pfx + "dec_grad_strided"])
    ev = np.concatenate([gan.evaluate(x, y), gan.evaluate(x, y, 0.7, 0.3)])
    assert np.array_equal(ev, g[pfx + "eval"])
    # one discriminator_step + generator_step
    assert gan.adam(oracle.DISC, dg)
    losses2, fg2, ig2 = gan.gen_backward(x, y)
    assert gan.adam(oracle.FWD, fg2) and gan.adam(oracle.INV, ig2)
    assert np.array_equal(np.concatenate([[dl], losses2]), g[pfx + "step_losses"])
    for net, name in ((oracle.FWD, "fwd"), (oracle.INV, "inv"), (oracle.DISC, "disc")):
        assert np.array_equal(gan.blob(net), g[pfx + "after_" + name]), name


def test_surrogate_tiny_desk(golden, oracle):
    g = golden("surrogate")
    _surrogate_check(g, oracle, "tiny_", TINY_DIMS, oracle.Arch.tiny(),
                     g["tiny_x"].reshape(16, 5), g["tiny_y"].reshape(16, 31), True)
    _surrogate_check(g, oracle, "desk_", DESK_DIMS, oracle.Arch(),
                     g["desk_x"].reshape(16, 5), g["desk_y"].reshape(16, 3087), False)


@pytest.mark.slow
def test_surrogate_paper(golden, oracle):
    g = golden("surrogate")
    x, y = oracle.Synth(PAPER_DIMS, 1).generate(8, 5)
    assert np.array_equal(x.ravel(), g["paper_x"])
    _surrogate_check(g, oracle, "paper_", PAPER_DIMS, oracle.Arch(), x, y, False)


def _dataset(oracle, dims, meta):
    n, _per_file, spec_seed, sampling_seed = (int(v) for v in meta)
    return oracle.Synth(dims, spec_seed).generate(n, sampling_seed)


def _trainer_check(g, oracle, pfx, dims, arch, ds, nsteps=None):
    model_seed, shards, batch, seed, n_tour, steps = (int(v) for v in g[pfx + "cfg"])
    assert shards == 1
    x, y = ds
    gan = oracle.Gan(dims, arch, model_seed)
    part = np.arange(n_tour, x.shape[0], dtype=np.uint32)
    tr = oracle.Trainer(gan, x, y, part, batch, seed)
    steps = steps if nsteps is None else nsteps
    rec, sk, ep, aborted = tr.steps(steps)
    assert not aborted
    for j, name in enumerate(("d_loss", "g_total", "g_fwd", "g_adv", "g_cyc")):
        assert np.array_equal(rec[:, j], g[pfx + "steps_" + name][:steps]), name
    assert np.array_equal(ep, g[pfx + "steps_epoch"][:steps])
    if nsteps is None:
        for net, name in ((oracle.FWD, "fwd"), (oracle.INV, "inv"), (oracle.DISC, "disc")):
            assert np.array_equal(tr.gan.blob(net), g[pfx + "final_" + name]), name
        ev = tr.gan.evaluate(x[:n_tour], y[:n_tour])
        assert np.array_equal(ev, g[pfx + "eval1"])
        assert np.array_equal(tr.gan.moment(oracle.FWD, 0), g[pfx + "fwd_m"])
        assert [tr.gan.t(n) for n in (oracle.FWD, oracle.INV, oracle.DISC)] == list(g[pfx + "opt_t"])


def test_trainer_tiny_and_abort(golden, oracle):
    g = golden("trainer")
    ds = _dataset(oracle, TINY_DIMS, g["tiny_data"])
    _trainer_check(g, oracle, "tiny_s1_", TINY_DIMS, oracle.Arch.tiny(), ds)
    # poisoned forward network: 3 allowed skips + the aborting one
    gan = oracle.Gan(TINY_DIMS, oracle.Arch.tiny(), 6)
    gan.blob(oracle.FWD)[:] = np.where(np.arange(gan.blob(oracle.FWD).size) >= 0, 1e38, 0)
    # biases stay zero in the reference poison (only weights were set)
    widths = [5, 8, 20]
    off = 0
    for l in range(2):
        nw = widths[l] * widths[l + 1]
        gan.blob(oracle.FWD)[off + nw: off + nw + widths[l + 1]] = 0.0
        off += nw + widths[l + 1]
    x, y = ds
    tr = oracle.Trainer(gan, x, y, np.arange(30, 600, dtype=np.uint32), 32, 10, abort_threshold=3)
    rec, sk, ep, aborted = tr.steps(10)
    assert aborted and list(sk) == list(g["abort_steps_skipped"]) and tr.step == int(g["abort_step"][0])


def test_trainer_desk(golden, oracle):
    g = golden("trainer")
    ds = _dataset(oracle, DESK_DIMS, g["desk_data"])
    _trainer_check(g, oracle, "desk_s1_", DESK_DIMS, oracle.Arch(), ds)


@pytest.mark.slow
def test_trainer_paper_first_steps(golden, oracle):
    g = golden("trainer")
    ds = _dataset(oracle, PAPER_DIMS, g["paper_data"])
    _trainer_check(g, oracle, "paper_s1_", PAPER_DIMS, oracle.Arch(), ds, nsteps=2)


@pytest.mark.parametrize("pfx,arch", [("tiny_k2_", "tiny"), ("tiny_k4_", "tiny"), ("tiny_k3_", "tiny")])
def test_tournament_decisions_state_injection(golden, oracle, pfx, arch):
    """Pre-round generators captured from the reference are evaluated on each
    trainer's tournament slice; metrics and decisions must equal the
    reference's round records exactly (tournament/ltfb.hpp:96-164)."""
    g = golden("tournament")
    cfg = [int(v) for v in g[pfx + "cfg"]]
    gen_n, _spf, spec_seed, sampling_seed, k = cfg[:5]
    dims = [int(v) for v in g[pfx + "dims"]]
    x, y = oracle.Synth(dims, spec_seed).generate(gen_n, sampling_seed)
    tour_sizes = g[pfx + "split_tour_sizes"]
    tour_off = np.concatenate([[0], np.cumsum(tour_sizes).astype(np.int64)]).astype(np.int64)
    tour_ids = g[pfx + "split_tour_ids"]
    fl, il = g[pfx + "pre_round_fwd_len"], g[pfx + "pre_round_inv_len"]
    fo = np.concatenate([[0], np.cumsum(fl).astype(np.int64)]).astype(np.int64)
    io = np.concatenate([[0], np.cumsum(il).astype(np.int64)]).astype(np.int64)
    base = oracle.Gan(dims, oracle.Arch.tiny() if arch == "tiny" else oracle.Arch(), 0)
    base.blob(oracle.ENC)[:] = g[pfx + "ae_enc"]
    base.blob(oracle.DEC)[:] = g[pfx + "ae_dec"]
    for i in range(g[pfx + "tr_round"].size):
        rnd, t, p = int(g[pfx + "tr_round"][i]), int(g[pfx + "tr_trainer"][i]), int(g[pfx + "tr_peer"][i])
        ids = tour_ids[tour_off[t]:tour_off[t + 1]]
        metrics = []
        for who in (t, p):
            j = (rnd - 1) * k + who
            base.blob(oracle.FWD)[:] = g[pfx + "pre_round_fwd"][fo[j]:fo[j + 1]]
            base.blob(oracle.INV)[:] = g[pfx + "pre_round_inv"][io[j]:io[j + 1]]
            metrics.append(base.evaluate(x[ids], y[ids])[2])
        assert metrics[0] == g[pfx + "tr_local"][i]
        assert metrics[1] == g[pfx + "tr_incoming"][i]
        assert oracle.incoming_wins(metrics[0], metrics[1]) == bool(g[pfx + "tr_kept"][i])
