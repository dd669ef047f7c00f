"""The `cvgram` CLI (cvgram_cli.cpp) on the B200 engine: options, output
format and exit codes.  Validation-only paths run on CPU; engine runs are -m gpu."""
import filecmp
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, cwd=None):
    r = subprocess.run([sys.executable, "-m", "paper_2401_13185_b200", *args], capture_output=True, text=True,
                       cwd=cwd or ROOT, timeout=600)
    return r.returncode, r.stdout, r.stderr


def write_inputs(d, x, y, labels):
    from paper_2401_13185_b200.cli import write_matrix_csv

    write_matrix_csv(os.path.join(d, "x.csv"), x)
    write_matrix_csv(os.path.join(d, "y.csv"), y)
    with open(os.path.join(d, "p.txt"), "w") as f:
        f.write("".join(f"{l}\n" for l in labels))
    return [os.path.join(d, n) for n in ("x.csv", "y.csv", "p.txt")]


def test_exit_codes_before_any_device_work(tmp_path):
    x = np.arange(12.0).reshape(6, 2)
    y = np.ones((6, 1))
    xp, yp, pp = write_inputs(str(tmp_path), x, y, [1, 1, 3, 3, 1, 3])  # fold 2 empty
    assert cli("verify", "--x", xp, "--y", yp, "--partition", pp)[0] == 4
    xp, yp, pp = write_inputs(str(tmp_path), x[:3], y[:3], [1, 1, 2])  # fold 1 trains on 1 row
    assert cli("verify", "--x", xp, "--y", yp, "--partition", pp)[0] == 5
    assert cli("run", "--x", xp, "--y", yp, "--partition", pp, "--config", "bogus", "--out-dir",
               str(tmp_path / "o"))[0] == 2
    assert cli("verify")[0] == 2
    assert cli("bench", "--n", "10", "--k", "2", "--m", "1", "--p-list", "1", "--out", str(tmp_path / "t.csv"))[0] == 4
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3\n")
    assert cli("run", "--x", str(bad), "--y", yp, "--partition", pp, "--out-dir", str(tmp_path / "o"))[0] == 2


def test_csv_and_token_formats():
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200.cli import read_matrix_csv, write_matrix_csv

    assert cv.config_to_string(cv.parse_config("center+scale")) == "1111"
    assert cv.config_to_string(cv.parse_config("center")) == "1100"
    assert cv.config_to_string(cv.parse_config("0110")) == "0110"
    assert cv.format_double(0.1) == "0.10000000000000001"


@pytest.mark.gpu
def test_verify_random_passes():
    code, out, err = cli("verify", "--random", "200", "30", "5", "10", "101")
    assert code == 0, out + err
    assert out.count(" ok") == 16 and "verify: all 16 configs within tolerance" in out


@pytest.mark.gpu
def test_run_is_byte_identical_across_runs_and_matches_baseline(tmp_path):  # acceptance.cpp:267-304
    rng = np.random.default_rng(9)
    x = rng.normal(2, 1, (120, 6))
    y = rng.normal(0, 1, (120, 2))
    labels = 1 + np.arange(120) % 4
    xp, yp, pp = write_inputs(str(tmp_path), x, y, labels)
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    for d, eng in ((a, "fast"), (b, "fast"), (c, "baseline")):
        code, out, err = cli("run", "--x", xp, "--y", yp, "--partition", pp, "--config", "center+scale",
                             "--engine", eng, "--out-dir", str(d))
        assert code == 0, out + err
    names = sorted(os.listdir(a))
    assert names == sorted(os.listdir(b)) and len(names) == 9
    assert all(filecmp.cmp(a / n, b / n, shallow=False) for n in names)
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200.cli import read_matrix_csv

    for f in range(1, 5):
        fa, fc = read_matrix_csv(str(a / f"fold_{f}_xtx.csv")), read_matrix_csv(str(c / f"fold_{f}_xtx.csv"))
        assert cv.max_rel_diff(fa, fc) <= 1e-8
    assert (a / "stats.csv").read_text().splitlines()[0] == "fold,name,values"


@pytest.mark.gpu
def test_bench_writes_timing_csv(tmp_path):
    out = tmp_path / "t.csv"
    code, so, se = cli("bench", "--n", "2000", "--k", "20", "--m", "3", "--p-list", "10,100", "--config", "1111",
                       "--reps", "3", "--out", str(out))
    assert code == 0, so + se
    lines = out.read_text().splitlines()
    assert lines[0] == "engine,config,n,k,m,p,wall_time,reps" and len(lines) == 5
    assert lines[1].startswith("baseline,1111,2000,20,3,10,")


@pytest.mark.gpu
def test_classify_combos_on_engine_output():  # test_combos.cpp:29-74, acceptance.cpp:144-157
    from paper_2401_13185_b200 import cvgram as cv

    rng = cv.MT19937_64(104)
    data = cv.random_dataset(50, 5, 3, rng)
    part = cv.random_partitioning(50, 5, rng)
    rep = cv.classify_combos(data, part, 1e-9)
    assert rep.n_xty_classes == 8 and rep.n_pair_classes == 12 and not rep.degenerate
    assert rep.min_xty_separation >= 1e-3 and rep.min_pair_separation >= 1e-3
    text = cv.format_combo_table(rep)
    assert "distinct XtY classes: 8" in text and "distinct pair classes: 12" in text and "warning" not in text


@pytest.mark.gpu
def test_acceptance_c9_byte_identical_across_runs_and_devices(tmp_path):
    """acceptance.cpp:267-304 on the GPU engine: `verify` and `run` outputs are byte-identical across two runs
    and across thread counts, and across device counts (--devices 0,0: the sharded multi-device run in its
    one-GPU emulation); `run`'s files also match the long-double oracle (1e-10 normalized)."""
    import oracle
    from paper_2401_13185_b200 import cvgram as cv
    from paper_2401_13185_b200.cli import read_matrix_csv

    v = [cli("verify", "--random", "120", "8", "3", "6", "77", "--threads", t, *extra)
         for t, extra in (("1", ()), ("1", ()), ("4", ()), ("1", ("--devices", "0,0")))]
    assert all(c == 0 for c, _, _ in v), v
    assert v[0][1] == v[1][1] == v[2][1] == v[3][1]
    rng = cv.MT19937_64(109)
    data = cv.random_dataset(5000, 40, 2, rng)  # folds of 1000 rows: the multi-device run is sharded
    part = cv.random_partitioning(5000, 5, rng)
    xp, yp, pp = write_inputs(str(tmp_path), data.x(), data.y(), part.labels)
    outs = []
    for name, extra in (("o1", ("--threads", "1")), ("o2", ("--threads", "1")), ("o4", ("--threads", "4")),
                        ("od", ("--devices", "0,0"))):
        code, out, err = cli("run", "--x", xp, "--y", yp, "--partition", pp, "--config", "1111", "--out-dir",
                             str(tmp_path / name), *extra)
        assert code == 0, out + err
        outs.append(tmp_path / name)
    files = sorted(os.listdir(outs[0]))
    assert len(files) == 2 * 5 + 1
    for o in outs[1:]:
        match, mismatch, errors = filecmp.cmpfiles(outs[0], o, files, shallow=False)
        assert not mismatch and not errors, (o, mismatch, errors)
    truth = oracle.truth_all_folds(data.x(), data.y(), part.labels, 5, 15, n_threads=8)
    for r in truth:
        got = read_matrix_csv(str(outs[0] / f"fold_{r.fold_id}_xtx.csv"))
        sc = np.sqrt(np.abs(np.diag(r.xtx_t)))
        assert np.max(np.abs(got - r.xtx_t) / np.maximum(np.abs(r.xtx_t), np.outer(sc, sc))) <= 1e-10
