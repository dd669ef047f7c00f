"""The reference's own known-answer tests, restated once and run against both
the CPU oracle (pinning it) and the B200 engine (`-m gpu`).

Sources: /root/reference/proj/tests/test_fast.cpp, test_core.cpp,
test_baseline.cpp, test_partition.cpp, acceptance.cpp (citations per test);
values live in tests/golden/reference_kats.json.
"""
import json
import os

import numpy as np
import pytest

from engines import ERR_BY_NAME
from paper_2401_13185_b200 import cvgram as cv

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))
MICRO = KATS["micro_case"]


def micro():
    return np.array(MICRO["x"], float), np.array(MICRO["y"], float)


def test_precompute_global_worked_values(engine):  # test_fast.cpp:25-38
    x, y = micro()
    k = KATS["precompute_global_micro"]
    c = engine.precompute_global(x, y, k["cfg"])
    ex = k["exact"]
    assert c.xtx[0, 0] == ex["xtx"] and c.xty[0, 0] == ex["xty"]
    assert c.sum_x[0] == ex["sum_x"] and c.sum_y[0] == ex["sum_y"]
    assert c.sum_sq_x[0] == ex["sum_sq_x"] and c.sum_sq_y[0] == ex["sum_sq_y"]
    assert c.n_rows == ex["n_rows"]
    assert c.mean_x[0] == pytest.approx(k["approx"]["mean_x"]) and c.mean_y[0] == pytest.approx(k["approx"]["mean_y"])
    assert c.sum_x[0] == 3.0 * c.mean_x[0]


def test_precompute_global_degenerate(engine):  # test_fast.cpp:40-54
    d = KATS["precompute_global_degenerate"]
    z = d["zero"]
    c = engine.precompute_global(np.array(z["x"], float), np.array(z["y"], float), z["cfg"])
    assert not c.xtx.any() and not c.xty.any() and not c.mean_x.any() and not c.sum_sq_y.any()
    i = d["identity"]
    c2 = engine.precompute_global(np.array(i["x"], float), np.array(i["y"], float), i["cfg"])
    assert np.array_equal(c2.xtx, np.array(i["xtx"], float))
    assert np.array_equal(c2.xty, np.array(i["xty"], float))
    assert c2.mean_x.size == 0 and c2.sum_sq_x.size == 0  # unused fields stay empty


def test_training_mean(engine):  # test_fast.cpp:56-68
    t = KATS["training_mean"]
    for c in t["cases"]:
        out = engine.training_mean(np.array(c["g"], float), np.array(c["v"], float), c["n"], c["n_val"])
        assert abs(out[0] - c["out"][0]) <= 1e-15
    th = t["throws"]
    with pytest.raises(ERR_BY_NAME[th["error"]]):
        engine.training_mean(np.array(th["g"], float), np.array(th["v"], float), th["n"], th["n_val"])


def test_training_std(engine):  # test_fast.cpp:70-95
    t = KATS["training_std"]
    for c in t["cases"]:
        out = engine.training_std(np.array(c["m"], float), np.array(c["s"], float), np.array(c["q"], float),
                                  c["n_train"])
        if c.get("exact"):
            assert out[0] == c["out"][0]
        else:
            assert abs(out[0] - c["out"][0]) <= 1e-15
    th = t["throws"]
    with pytest.raises(ERR_BY_NAME[th["error"]]):
        engine.training_std(np.array(th["m"], float), np.array(th["s"], float), np.array(th["q"], float),
                            th["n_train"])
    cl = t["clamp"]
    v = cl["v"]
    out = engine.training_std(np.array([v]), np.array([3 * v]), np.array([3 * v * v * (1.0 - 1e-16)]), cl["n_train"])
    assert out[0] == cl["out"]


def test_fold_products_micro(engine):  # test_fast.cpp:97-122
    x, y = micro()
    f = KATS["fold_products_micro"]
    for c in f["cases"]:
        cache = engine.precompute_global(x, y, c["cfg"])
        r = engine.fold_products(cache, x, y, f["v_rows"], c["cfg"], c.get("fold_id", 0))
        if "fold_id" in c:
            assert r.fold_id == c["fold_id"]
        if "xtx" in c:
            assert abs(r.xtx_t[0, 0] - c["xtx"]) <= 1e-12
        assert abs(r.xty_t[0, 0] - c["xty"]) <= 1e-12


def test_fold_products_rejects_degenerate_folds(engine):  # test_fast.cpp:124-132
    x, y = micro()
    for c in KATS["fold_products_errors"]["cases"]:
        cache = engine.precompute_global(x, y, c["cfg"])
        with pytest.raises(ERR_BY_NAME[c["error"]]):
            engine.fold_products(cache, x, y, np.array(c["v_rows"], np.int64), c["cfg"])


def test_fast_matches_baseline_seeded(engine):  # test_fast.cpp:134-158
    import oracle

    s = KATS["seeded_equivalence"]
    rng = cv.MT19937_64(s["seed"])
    data = cv.random_dataset(s["n"], s["k"], s["m"], rng)
    part = cv.random_partitioning(s["n"], s["p"], rng)
    x, y = data.x(), data.y()
    for bits in range(16):
        fast = engine.run_all_folds(x, y, part.labels, part.p, bits)
        base = oracle.baseline_all_folds(x, y, part.labels, part.p, bits)
        assert len(fast) == len(base)
        for f, b in zip(fast, base):
            assert f.fold_id == b.fold_id
            assert cv.max_rel_diff(f.xtx_t, b.xtx_t) <= s["tol_products"]
            assert cv.max_rel_diff(f.xty_t, b.xty_t) <= s["tol_products"]
            if bits:
                assert cv.max_rel_diff(f.mean_x_t, b.mean_x_t) <= s["tol_means"]
                assert cv.max_rel_diff(f.mean_y_t, b.mean_y_t) <= s["tol_means"]
            if bits & 2:
                assert cv.max_rel_diff(f.std_x_t, b.std_x_t) <= s["tol_stds"]
            if bits & 1:
                assert cv.max_rel_diff(f.std_y_t, b.std_y_t) <= s["tol_stds"]


def test_loo_boundary(engine):  # test_fast.cpp:160-165
    x, y = micro()
    b = KATS["loo_boundary"]
    res = engine.run_all_folds(x, y, np.array(b["labels"], np.int32), b["p"], b["cfg"])
    assert len(res) == 3 and all(r.n_train == b["n_train"] for r in res)


def test_statistic_reconstruction(engine):  # test_fast.cpp:167-190
    rng = cv.MT19937_64(9)
    data = cv.random_dataset(50, 4, 2, rng)
    x, y = data.x(), data.y()
    cache = engine.precompute_global(x, y, 15)
    for _ in range(100):
        v = np.array([i for i in range(50) if rng() % 3 == 0], np.int64)
        if v.size == 0 or v.size > 48:
            continue
        r = engine.fold_products(cache, x, y, v, 15)
        xt = x[cv.complement_rows(v, 50)]
        mean = xt.mean(axis=0)
        assert cv.max_rel_diff(r.mean_x_t, mean) <= 1e-12
        var = ((xt - mean) ** 2).sum(axis=0) / (xt.shape[0] - 1.0)
        for j in range(4):
            if var[j] > 1e-20:
                assert r.std_x_t[j] == pytest.approx(np.sqrt(var[j]), rel=1e-10)


def test_centering_paired_data_is_noop(engine):  # test_fast.cpp:192-215
    rng = cv.MT19937_64(10)
    n = 8
    x, y = np.empty((n, 3)), np.empty((n, 2))
    for i in range(0, n, 2):
        for j in range(3):
            x[i, j] = rng.uniform01()
            x[i + 1, j] = -x[i, j]
        for j in range(2):
            y[i, j] = rng.uniform01()
            y[i + 1, j] = -y[i, j]
    labels = np.array([1, 1, 2, 2, 3, 3, 4, 4], np.int32)
    centered = engine.run_all_folds(x, y, labels, 4, 12)
    raw = engine.run_all_folds(x, y, labels, 4, 0)
    for c, r in zip(centered, raw):
        assert cv.max_rel_diff(c.xtx_t, r.xtx_t) <= 1e-12


def test_thread_count_does_not_change_a_bit(engine):  # test_fast.cpp:217-229
    rng = cv.MT19937_64(12)
    data = cv.random_dataset(60, 6, 2, rng)
    part = cv.random_partitioning(60, 9, rng)
    a = engine.run_all_folds(data.x(), data.y(), part.labels, 9, 15, n_threads=1)
    b = engine.run_all_folds(data.x(), data.y(), part.labels, 9, 15, n_threads=4)
    for s, p in zip(a, b):
        assert s.xtx_t.tobytes() == p.xtx_t.tobytes() and s.xty_t.tobytes() == p.xty_t.tobytes()


def test_baseline_micro_case(engine):  # test_baseline.cpp:23-53, acceptance.cpp:86-116 (both engines)
    x, y = micro()
    b = KATS["baseline_micro"]
    labels = np.array(b["labels"], np.int32)
    for run in (engine.run_all_folds, engine.baseline_all_folds):
        for c in b["fold2"]:
            res = run(x, y, labels, b["p"], c["cfg"])
            assert res[1].fold_id == 2
            assert abs(res[1].xtx_t[0, 0] - c["xtx"]) <= 1e-12 and abs(res[1].xty_t[0, 0] - c["xty"]) <= 1e-12
        with pytest.raises(ERR_BY_NAME[b["all_on_full_run_error"]]):
            run(x, y, labels, b["p"], 15)
    s = b["all_on_single_fold"]
    for r in (engine.fold_products(engine.precompute_global(x, y, s["cfg"]), x, y, s["v_rows"], s["cfg"], 2),
              engine.baseline_single_fold(x, y, s["v_rows"], s["cfg"], 2)):
        assert abs(r.xtx_t[0, 0] - s["xtx"]) <= 1e-12 and abs(r.xty_t[0, 0] - s["xty"]) <= 1e-12
        assert abs(r.std_x_t[0] - s["std_x"]) <= 1e-15 and abs(r.std_y_t[0] - s["std_y"]) <= 1e-15


@pytest.mark.parametrize("key", ["zero_variance", "zero_variance_acceptance"])
def test_zero_variance_training_column(engine, key):  # test_baseline.cpp:55-66, acceptance.cpp:254-263
    z = KATS[key]
    for run in (engine.run_all_folds, engine.baseline_all_folds):
        res = run(np.array(z["x"], float), np.array(z["y"], float), np.array(z["labels"], np.int32), z["p"], z["cfg"])
        if key == "zero_variance":
            assert res[0].std_x_t[0] == z["fold1"]["std_x"]
            assert abs(res[0].xtx_t[0, 0]) <= z["fold1"]["xtx_margin"]
        else:
            for r in res:
                assert r.std_x_t[0] == z["std_x0"]


def test_raw_fold_plus_validation_is_total(engine):  # test_baseline.cpp:68-81
    rng = cv.MT19937_64(3)
    data = cv.random_dataset(35, 4, 2, rng)
    part = cv.random_partitioning(35, 6, rng)
    x = data.x()
    res = engine.baseline_all_folds(x, data.y(), part.labels, 6, 0)
    idx = cv.build_validation_partitions(part)
    for r, rows in zip(res, idx.sets):
        xv = x[rows]
        assert cv.max_rel_diff(r.xtx_t + xv.T @ xv, x.T @ x) <= 1e-10


def test_xtx_symmetric_every_config(engine):  # test_baseline.cpp:83-93
    rng = cv.MT19937_64(4)
    data = cv.random_dataset(25, 5, 2, rng)
    part = cv.random_partitioning(25, 4, rng)
    for bits in range(16):
        for r in engine.baseline_all_folds(data.x(), data.y(), part.labels, 4, bits):
            assert np.abs(r.xtx_t - r.xtx_t.T).max() <= 1e-12


def test_centering_either_side_same_xty(engine):  # test_baseline.cpp:95-112, acceptance.cpp:118-142
    rng = cv.MT19937_64(5)
    data = cv.random_dataset(40, 3, 2, rng)
    part = cv.random_partitioning(40, 5, rng)
    for s in range(4):
        sx, sy = s >> 1, s & 1
        rx = engine.run_all_folds(data.x(), data.y(), part.labels, 5, 8 | sx * 2 | sy)
        ry = engine.run_all_folds(data.x(), data.y(), part.labels, 5, 4 | sx * 2 | sy)
        rb = engine.run_all_folds(data.x(), data.y(), part.labels, 5, 12 | sx * 2 | sy)
        gap = 0.0
        for a, b, c in zip(rx, ry, rb):
            assert cv.max_rel_diff(a.xty_t, b.xty_t) <= 1e-12
            assert cv.max_rel_diff(a.xty_t, c.xty_t) <= 1e-12
            gap = max(gap, cv.max_rel_diff(a.xtx_t, b.xtx_t))
        assert gap > 1e-6  # acceptance criterion 3: XᵀX does differ


def test_preprocessed_training_has_mean0_std1(engine):  # test_baseline.cpp:114-134
    rng = cv.MT19937_64(6)
    data = cv.random_dataset(30, 4, 2, rng)
    part = cv.random_partitioning(30, 3, rng)
    res = engine.baseline_all_folds(data.x(), data.y(), part.labels, 3, 15)
    idx = cv.build_validation_partitions(part)
    for r, rows in zip(res, idx.sets):
        xt = data.x()[cv.complement_rows(rows, 30)]
        z = (xt - r.mean_x_t) / r.std_x_t
        assert np.abs(z.mean(axis=0)).max() <= 1e-12
        assert np.allclose(z.std(axis=0, ddof=1), 1.0, atol=1e-10, rtol=0)


def test_scaling_non_scalable_rejected(engine):  # test_baseline.cpp:136-148 (both engines)
    x, y = np.full((2, 1), 2.0), np.ones((2, 1))
    mx, my = micro()
    for run in (engine.run_all_folds, engine.baseline_all_folds):
        with pytest.raises(cv.ScalabilityError):
            run(x, y, np.array([1, 2], np.int32), 2, 2)
        run(x, y, np.array([1, 2], np.int32), 2, 0)
        with pytest.raises(cv.PartitionError):
            run(mx, my, np.array([1, 1, 3], np.int32), 3, 0)
        with pytest.raises(cv.DimensionError):
            run(mx, my, np.array([1, 2], np.int32), 2, 0)


def test_hadamard_outer_divide(engine):  # test_core.cpp:9-67
    h = KATS["hadamard"]
    m, l, r = np.array(h["m"], float), np.array(h["l"], float), np.array(h["r"], float)
    out = engine.hadamard_outer_divide(m, l, r)
    for i in range(2):
        for j in range(2):
            assert out[i, j] == m[i, j] / (l[i] * r[j])
    assert out[0, 0] == 1.0 and out[0, 1] == 1.0 and out[1, 1] == 4.0
    assert out[1, 0] == pytest.approx(2.0 / 3.0)
    s = h["sqrt2"]
    assert abs(engine.hadamard_outer_divide(np.array(s["m"]), np.array(s["l"]), np.array(s["r"]))[0, 0] - 1) <= 1e-15
    rng = cv.MT19937_64(1)
    mm = np.array([[rng.uniform01() for _ in range(3)] for _ in range(5)])
    assert np.array_equal(engine.hadamard_outer_divide(mm, np.ones(5), np.ones(3)), mm)
    rng = cv.MT19937_64(2)
    for _ in range(20):
        u = lambda: 0.25 + rng.uniform01()  # noqa: E731
        m4 = np.array([[u() for _ in range(6)] for _ in range(4)])
        l4 = np.array([u() for _ in range(4)])
        r6 = np.array([u() for _ in range(6)])
        back = engine.hadamard_outer_divide(m4, l4, r6) * np.outer(l4, r6)
        assert np.allclose(back, m4, rtol=1e-15 * 4, atol=0)
    for bad in h["reject"]:
        with pytest.raises(cv.InvalidArgument):
            engine.hadamard_outer_divide(np.ones((2, 2)), np.array(bad["l"]), np.array(bad["r"]))


def test_acceptance_c1_oracle_equivalence(engine):  # acceptance.cpp:62-84
    import oracle

    a = KATS["acceptance_c1"]
    rng = cv.MT19937_64(a["seed"])
    data = cv.random_dataset(a["n"], a["k"], a["m"], rng)
    worst = 0.0
    for p in a["ps"]:
        part = cv.random_partitioning(a["n"], p, rng)
        cfgs = list(range(16))
        runs = engine.run_all_folds_configs(data.x(), data.y(), part.labels, p, cfgs)
        for bits, fast in zip(cfgs, runs):
            base = oracle.baseline_all_folds(data.x(), data.y(), part.labels, p, bits)
            for f, b in zip(fast, base):
                worst = max(worst, cv.max_rel_diff(f.xtx_t, b.xtx_t), cv.max_rel_diff(f.xty_t, b.xty_t))
    assert worst <= a["tol"]
