"""The product's host-side algorithms (libltfb_gpu.so C ABI, host code only)
against the reference golden vectors: bit-exact pairings, partitions,
splits, epoch permutations, parameter init and synthetic samples."""
import numpy as np
import pytest

L = pytest.importorskip("paper_1910_02270_b200")

TINY = L.ModalityDims(image_views=1, image_channels=1, image_h=4, image_w=4)
DESK = L.ModalityDims()
PAPER = L.ModalityDims.paper_scale()


def test_mix_seed_and_hash(golden):
    g = golden("rng")
    parts = [(1,), (1, 2), (42, 0xA11), (7, 3, 0x9A12), (0,), (2**64 - 1, 5),
             (1, 0x57A7E1, 3), (12345, 0, 0x5CAFF1E)]
    assert [L.mix_seed(*p) for p in parts] == [int(v) for v in g["mix_seed"]]
    assert L.fnv1a64(np.frombuffer(b"hello", np.uint8)) == int(g["fnv_hello"][0])


def test_pairings_partitions_splits(golden):
    g = golden("plan")
    for tag, n, k, seed in (("part_100_4_5_", 100, 4, 5), ("part_1000_7_11_", 1000, 7, 11)):
        parts = L.partition_dataset(np.arange(n), k, seed)
        assert np.array_equal(np.concatenate(parts), g[tag + "ids"])
    i, byes = 0, []
    for k in (2, 3, 4, 5, 8):
        for rnd in range(1, 26):
            m = L.pair_trainers(k, rnd, 0x1234)
            byes.append(m.bye)
            for a, b in m.pairs:
                assert (g["pair_a"][i], g["pair_b"][i]) == (a, b)
                i += 1
    assert byes == list(g["pair_byes"])
    for total, k, seed in ((800, 2, 42), (16000, 4, 101), (16000, 8, 1)):
        pfx = f"split_{total}_{k}_"
        val, train, tour = L.split_dataset(total, k, 0.05, 0.05, seed, k >= 2)
        assert np.array_equal(val, g[pfx + "validation"])
        assert np.array_equal(np.concatenate(train), g[pfx + "train_ids"])
        assert np.array_equal(np.concatenate(tour), g[pfx + "tour_ids"])
    _, train, _ = L.split_dataset(800, 2, 0.05, 0.05, 42, True)
    for e in (1, 2, 3):
        assert np.array_equal(L.epoch_permutation(train[0], e, int(g["plan_seed"][0])), g[f"plan_perm_e{e}"])


def test_pairing_edge_cases():
    assert L.pair_trainers(1, 1, 9).pairs == [] and L.pair_trainers(0, 1, 9).pairs == []
    m = L.pair_trainers(5, 2, 13)
    seen = {x for p in m.pairs for x in p}
    assert len(m.pairs) == 2 and 0 <= m.bye < 5 and m.bye not in seen and len(seen) == 4
    with pytest.raises(L.ContractError):
        L.partition_dataset(np.arange(3), 4, 1)
    with pytest.raises(L.ContractError):
        L.partition_dataset(np.arange(3), 0, 1)


def test_pairing_uniformity_k4():
    """tests/test_tournament.cpp:143-166: each of the 3 matchings of 4
    trainers appears with frequency 1/3 +- 0.02 over 10000 rounds."""
    counts = {}
    for r in range(1, 10001):
        m = L.pair_trainers(4, r, 77)
        key = tuple(sorted(tuple(sorted(p)) for p in m.pairs))
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 3
    for c in counts.values():
        assert abs(c / 10000 - 1 / 3) < 0.02


def test_incoming_wins_rule():
    nan, inf = float("nan"), float("inf")
    assert not L.incoming_wins(1.0, 1.0)          # ties keep local
    assert L.incoming_wins(1.0, 0.5)
    assert not L.incoming_wins(0.5, 1.0)
    assert not L.incoming_wins(1.0, nan)          # non-finite incoming loses
    assert L.incoming_wins(nan, 1.0)              # non-finite local loses
    assert not L.incoming_wins(nan, inf)          # both bad: keep local


def test_synth_matches_reference(golden):
    g = golden("synth")
    x, y = L.synth_generate(TINY, 200, sampling_seed=17, spec_seed=3)
    assert np.array_equal(x.ravel(), g["tiny_x"]) and np.array_equal(y.ravel(), g["tiny_y"])
    x, y = L.synth_generate(TINY, 20, sampling_seed=17, spec_seed=3, noise_level=0.1)
    assert np.array_equal(y.ravel(), g["tiny_noisy_y"])
    for i, which in enumerate(g["desk_which"]):
        _, y = L.synth_generate(DESK, 1, sampling_seed=1, spec_seed=1, first=int(which), total=16000)
        assert np.array_equal(y.ravel(), g["desk_y"][i * 3087:(i + 1) * 3087])
    _, y = L.synth_generate(PAPER, 1, sampling_seed=1, spec_seed=1, first=12345, total=16000)
    assert np.array_equal(y.ravel(), g["paper_y"])


def test_make_cyclegan_matches_reference(golden):
    g = golden("surrogate")
    m = L.make_cyclegan(TINY, L.SurrogateArch.tiny(), 3)
    for n in ("enc", "dec", "fwd", "inv", "disc"):
        assert np.array_equal(m.blobs[n], g["tiny_init_" + n])
    h = g["desk_init_hashes"]
    m = L.make_cyclegan(DESK, L.SurrogateArch(), 11)
    assert [m.enc_hash(), m.dec_hash(), m.fwd_hash(), m.inv_hash(), m.disc_hash(), m.model_hash()] == \
        [int(v) for v in h]
    t = golden("trainer")
    m = L.make_cyclegan(TINY, L.SurrogateArch.tiny(), 6)
    L.reinit_gan_nets(m, 99)
    ref = L.make_cyclegan(TINY, L.SurrogateArch.tiny(), 99)
    assert m.fwd_hash() == ref.fwd_hash() and m.disc_hash() == ref.disc_hash()
    assert t is not None


def test_ae_batch_draws_match_reference_rng(oracle):
    """runner.hpp:257-266: AE batch rows = Rng(mix_seed({seed, 0xae1})).below(rows),
    step-major, against the pinned oracle Rng."""
    seed, rows, batch, steps = 17, 1000, 128, 3
    got = L.ae_batch_rows(seed, rows, batch, steps)
    r = oracle.Rng(oracle.mix_seed(seed, 0xAE1))
    ref = np.array([r.below(rows) for _ in range(batch * steps)], np.uint32).reshape(steps, batch)
    assert np.array_equal(got, ref)


def test_run_config_refuses_unsupported_store_modes():
    """runner.hpp:91-110 + store.hpp:62-271: a config asking for the
    file-streaming store modes or a store budget is refused (ConfigError)
    instead of silently running the HBM preload store."""
    from paper_1910_02270_b200.runner import validate_run_config
    validate_run_config(L.RunConfig())
    for kw in ({"data_store": "dynamic"}, {"data_store": "none"}, {"store_budget_mb": 64}):
        with pytest.raises(L.ConfigError):
            validate_run_config(L.RunConfig(**kw))


def test_sharded_ae_plan_assembles_the_replicated_batch():
    """runner.sharded_ae_plan / sharded_ae_indices: with the union of the
    training partitions sharded over k ranks' stores, every rank's rows packed
    into its block and an all-gather of the blocks, the AE step's source rows
    are exactly the rows the replicated pre-training draws from the sorted
    union (runner.hpp:255-277)."""
    from paper_1910_02270_b200.runner import sharded_ae_indices, sharded_ae_plan
    rng = np.random.default_rng(4)
    total, k, b, steps, seed = 500, 3, 32, 6, 42
    ids = rng.permutation(total).astype(np.uint32)
    parts = [ids[:170], ids[170:330], ids[330:480]]  # ids[480:] is nobody's (validation)
    y = rng.standard_normal((total, 7)).astype(np.float32)  # a row per global id
    union = np.sort(np.concatenate(parts))
    draws = L.ae_batch_rows(seed, union.size, b, steps)
    owner, slot, bb = sharded_ae_plan(parts, b, steps, seed)
    assert bb == b
    for s in range(steps):
        src = np.zeros((k * b, 7), np.float32)
        for r in range(k):  # each rank fills its block from its own store
            mine = np.nonzero(owner[s] == r)[0]
            src[r * b:r * b + mine.size] = y[parts[r][slot[s][mine]]]
        got = src[sharded_ae_indices(owner[s], k, b)]
        assert np.array_equal(got, y[union[draws[s]]])
