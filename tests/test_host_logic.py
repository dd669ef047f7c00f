"""Host-side logic that needs no GPU: the partition predicates and seeded
generators of both the product library and the oracle, pinned to the
reference's tests (test_partition.cpp, random.hpp) and to each other."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2401_13185_b200 import cvgram as cv

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))


def test_mt19937_64_standard_value():  # random.hpp:14-18
    k = KATS["mt19937_64"]
    for make in (lambda s: cv.MT19937_64(s), lambda s: oracle.MT64(s)):
        r = make(k["seed"])
        nxt = r if callable(r) else r.next
        for _ in range(k["index"] - 1):
            (r() if callable(r) else r.next())
        last = r() if callable(r) else r.next()
        assert str(last) == k["value"]


def test_generators_agree_bitwise():  # random.hpp:21-55 in product and oracle
    for seed in (1, 8, 101):
        a, b = cv.MT19937_64(seed), oracle.MT64(seed)
        d = cv.random_dataset(37, 4, 3, a)
        x, y = b.random_dataset(37, 4, 3)
        assert d.x().tobytes() == x.tobytes() and d.y().tobytes() == y.tobytes()
        assert np.array_equal(cv.random_partitioning(37, 5, a).labels, b.random_partitioning(37, 5))


@pytest.mark.parametrize("impl", ["product", "oracle"])
def test_build_validation_partitions_examples(impl):  # test_partition.cpp:11-25
    for c in KATS["partition_examples"]["cases"]:
        labels = np.array(c["labels"], np.int32)
        sets = (cv.build_validation_partitions(cv.Partitioning(labels, c["p"])).sets if impl == "product"
                else oracle.build_validation_partitions(labels, c["p"]))
        assert [list(s) for s in sets] == c["sets"]


@pytest.mark.parametrize("impl", ["product", "oracle"])
def test_validate_partitioning_messages(impl):  # test_partition.cpp:27-37
    fn = cv.validate_partitioning if impl == "product" else oracle.validate_partitioning
    v = KATS["validate_messages"]
    for c in v["ok"]:
        assert fn(np.array(c["labels"], np.int32), c["p"]) is None
    for c in v["bad"]:
        msg = fn(np.array(c["labels"], np.int32), c["p"])
        assert msg is not None
        if "contains" in c:
            assert c["contains"] in msg


def test_validate_messages_identical_between_product_and_oracle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 12))
        p = int(rng.integers(0, 6))
        labels = rng.integers(-1, 7, n).astype(np.int32)
        assert cv.validate_partitioning(labels, p) == oracle.validate_partitioning(labels, p)
        if oracle.validate_partitioning(labels, p) is None:
            part = cv.Partitioning(labels, p)
            assert cv.check_scalable(part) == oracle.check_scalable(labels, p)


@pytest.mark.parametrize("impl", ["product", "oracle"])
def test_check_scalable(impl):  # test_partition.cpp:39-46
    s = KATS["check_scalable"]
    fn = (lambda l, p: cv.check_scalable(cv.Partitioning(l, p))) if impl == "product" else oracle.check_scalable
    for c in s["ok"]:
        assert fn(np.array(c["labels"], np.int32), c["p"]) is None
    for c in s["bad"]:
        msg = fn(np.array(c["labels"], np.int32), c["p"])
        assert msg is not None and c.get("contains", "") in msg


def test_partition_counting_identities():  # test_partition.cpp:48-64, acceptance.cpp:159-174
    rng = cv.MT19937_64(7)
    for _ in range(50):
        n = 2 + rng() % 60
        p = 2 + rng() % (n - 1)
        part = cv.random_partitioning(n, p, rng)
        assert cv.validate_partitioning(part) is None
        sets = cv.build_validation_partitions(part).sets
        assert sum(len(s) for s in sets) == n
        assert sum(n - len(s) for s in sets) == n * (p - 1)


def test_permuting_fold_names_permutes_sets():  # test_partition.cpp:66-85
    rng = cv.MT19937_64(11)
    n, p = 23, 5
    part = cv.random_partitioning(n, p, rng)
    perm = list(range(1, p + 1))
    for i in range(p - 1, 0, -1):
        j = rng() % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    renamed = cv.Partitioning(np.array([perm[l - 1] for l in part.labels], np.int32), p)
    before = cv.build_validation_partitions(part).sets
    after = cv.build_validation_partitions(renamed).sets
    for f in range(1, p + 1):
        assert list(after[perm[f - 1] - 1]) == list(before[f - 1])


@pytest.mark.parametrize("impl", ["product", "oracle"])
def test_complement_rows(impl):  # test_partition.cpp:87-91
    fn = cv.complement_rows if impl == "product" else oracle.complement_rows
    for c in KATS["complement_rows"]["cases"]:
        assert list(fn(np.array(c["v"], np.int64), c["n"])) == c["out"]


def test_dataset_pair_invariants():  # test_core.cpp:69-80
    for b in KATS["dataset_pair_invariants"]["bad"]:
        x, y = np.ones(b["x_shape"]), np.ones(b["y_shape"])
        if "nan_at" in b:
            x[tuple(b["nan_at"])] = np.nan
        with pytest.raises(cv.DimensionError):
            cv.DatasetPair(x, y)
    d = cv.DatasetPair(np.ones((3, 2)), np.ones((3, 1)))
    assert (d.n_rows(), d.n_features(), d.n_responses()) == (3, 2, 1)


def test_enumerate_configs():  # test_combos.cpp:9-27
    cfgs = cv.enumerate_configs()
    assert len(cfgs) == 16 and cfgs[0] == cv.PreprocessConfig() and cfgs[-1] == cv.PreprocessConfig(1, 1, 1, 1)
    assert len({c.mask for c in cfgs}) == 16 and [c.mask for c in cfgs] == list(range(16))


def test_fold_range_is_a_tree_partition():
    from paper_2401_13185_b200 import plan

    for p in (1, 2, 5, 7, 20, 100):
        for world in (1, 2, 3, 4, 8, 16):
            ranges = [plan.fold_range(p, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == p
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            if world & (world - 1) == 0 and p >= world:
                sizes = [b - a for a, b in ranges]
                assert max(sizes) - min(sizes) <= 1 + (world > 2)  # midpoint tree is near-balanced


def test_numpy_mt19937_64_and_partitioning_match_both_libraries():
    """workloads.py's numpy engine (used by both bench arms, no .so) draws the same stream
    as the product's and the oracle's std::mt19937_64, and its random_partitioning the same labels."""
    import workloads

    k = KATS["mt19937_64"]
    assert str(int(workloads.mt19937_64(k["seed"], k["index"])[-1])) == k["value"]
    for seed in (0, 1, 20240124, 2**64 - 1):
        o = oracle.MT64(seed)
        ref = [o.next() for _ in range(700)]
        assert [int(v) for v in workloads.mt19937_64(seed, 700)] == ref
    for n, p, seed in ((1, 1, 3), (2, 2, 5), (1000, 7, 11), (20011, 100, 20240124)):
        lab = workloads.random_partitioning(n, p, seed)
        assert np.array_equal(lab, cv.random_partitioning(n, p, seed).labels)
        assert np.array_equal(lab, oracle.MT64(seed).random_partitioning(n, p))


def test_numpy_alg7_matches_r64():
    """The numpy/OpenBLAS CPU point (oracle/numpy_alg7.py) restates the same algorithm as R64."""
    from oracle import numpy_alg7

    rng = np.random.default_rng(3)
    n, k, m, p = 600, 9, 3, 5
    x = rng.uniform(-5, 5, k) + rng.uniform(0.5, 2, k) * rng.standard_normal((n, k))
    y = x @ rng.standard_normal((k, m)) + rng.uniform(-3, 3, m)
    labels = rng.integers(1, p + 1, n).astype(np.int32)
    labels[:p] = np.arange(1, p + 1)
    for cfg in range(16):
        ref = oracle.fast_all_folds(x, y, labels, p, cfg)
        got = numpy_alg7.run_all_folds(x, y, labels, p, cfg)
        for r, (gx, gy) in zip(ref, got):
            assert oracle.max_rel_diff(gx, r.xtx_t) < 1e-8 and oracle.max_rel_diff(gy, r.xty_t) < 1e-8
