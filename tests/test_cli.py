"""CLI / bench surface: file formats, config parsing, aggregation and
exit codes on CPU; predict and bench end to end on the GPU."""

import numpy as np
import pytest

from paper_2403_12797_b200 import cli
from paper_2403_12797_b200.datagen import generate, load_csv, save_csv
from paper_2403_12797_b200.errors import ConfigError, CsvFormatError


def test_headers_match_reference_golden(golden):
    assert cli.RESULTS_HEADER == str(golden["headers/results"])
    assert cli.PLOTDATA_HEADER == str(golden["headers/plotdata"])


def test_csv_round_trip_bit_exact(tmp_path):
    ds = generate(257, 3, seed=11)
    path = tmp_path / "d.csv"
    save_csv(ds, path)
    back = load_csv(path)
    assert np.array_equal(back.X, ds.X) and np.array_equal(back.y, ds.y)


@pytest.mark.parametrize("text,line", [("", 0), ("a,b\n1,2\n", 1), ("x1,y\n1,2,3\n", 2), ("x1,y\n1,zz\n", 2),
                                       ("x1,y\n", 1)])
def test_csv_errors_carry_line(tmp_path, text, line):
    path = tmp_path / "bad.csv"
    path.write_text(text)
    with pytest.raises(CsvFormatError) as ei:
        load_csv(path)
    assert ei.value.line == line


def test_config_parsing(tmp_path):
    cfg_path = tmp_path / "c.txt"
    cfg_path.write_text("n_samples = 500  # comment\ndims = 2,3\neigen_counts.2 = 4,5\neigen_counts.3 = 3\n"
                        "reps = 2\nworkers = 8\n")
    cfg = cli.parse_config_file(cfg_path)
    assert cfg.n_samples == 500 and cfg.dims == (2, 3) and cfg.eigen_counts[2] == (4, 5) and cfg.reps == 2
    cfg_path.write_text("bogus = 1\n")
    with pytest.raises(ConfigError, match="unknown"):
        cli.parse_config_file(cfg_path)
    cfg_path.write_text("dims = 9\n")
    with pytest.raises(ConfigError, match="eigen_counts"):
        cli.parse_config_file(cfg_path)


def test_results_rows_and_plotdata(tmp_path):
    rows = [("cuda", 2, 5, r, ph, 0.1 * (r + 1) + i) for r in range(3) for i, ph in enumerate(cli.PHASES)]
    rows.append(("cuda", 2, 9, 0, cli.SKIP_PHASE, cli.SKIP_SECONDS))
    path = tmp_path / "r.csv"
    path.write_text(cli.RESULTS_HEADER + "\n" + "\n".join(cli.format_row(r) for r in rows) + "\n")
    back = cli.read_results_csv(path)
    assert len(back) == len(rows) and back[-1][4] == cli.SKIP_PHASE and back[-1][5] == -1.0
    tables = cli.aggregate_plotdata(back)
    (mode, n, mean_tot, std_tot, *rest), = tables[2]
    totals = [sum(0.1 * (r + 1) + i for i in range(4)) for r in range(3)]
    assert mode == "cuda" and n == 5
    assert mean_tot == pytest.approx(np.mean(totals)) and std_tot == pytest.approx(np.std(totals, ddof=1))
    paths = cli.write_plotdata_csvs(tables, tmp_path)
    assert paths[0].read_text().splitlines()[0] == cli.PLOTDATA_HEADER


def test_exit_codes_without_gpu(tmp_path, capsys):
    assert cli.main(["predict", "--train", str(tmp_path / "missing.csv"), "--test", "x", "--out", "o"]) == cli.EXIT_IO
    bad = tmp_path / "bad.csv"
    bad.write_text("q,r\n1,2\n")
    assert cli.main(["predict", "--train", str(bad), "--test", str(bad), "--out", "o"]) == cli.EXIT_IO
    with pytest.raises(SystemExit) as ei:
        cli.main(["predict"])
    assert ei.value.code == cli.EXIT_USAGE
    assert cli.main(["generate", "--n-samples", "20", "--dim", "2", "--seed", "3", "--out-dir", str(tmp_path)]) == 0
    assert (tmp_path / "train_N20_p2_seed3.csv").exists()


@pytest.mark.gpu
def test_predict_cli_matches_oracle(tmp_path):
    import fagp_oracle as O

    ds = generate(3000, 2, seed=200001)
    save_csv(ds, tmp_path / "train.csv")
    Xs = np.random.default_rng(0).uniform(-1, 1, (200, 2))
    (tmp_path / "test.csv").write_text("x1,x2\n" + "\n".join(f"{a:.17g},{b:.17g}" for a, b in Xs) + "\n")
    rc = cli.main(["predict", "--train", str(tmp_path / "train.csv"), "--test", str(tmp_path / "test.csv"),
                   "--out", str(tmp_path / "out.csv"), "--n-eigen", "8", "--noise-var", "0.0025", "--cov"])
    assert rc == cli.EXIT_OK
    lines = (tmp_path / "out.csv").read_text().splitlines()
    assert lines[0] == "x1,x2,mean,var"
    got = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    ref = O.posterior(ds.X, ds.y, Xs, [1.0, 1.0], [1.0, 1.0], 8, 0.0025)
    assert np.array_equal(got[:, :2], Xs)
    assert np.max(np.abs(got[:, 2] - ref["mean"]) / np.abs(ref["mean"])) < 1e-9
    assert np.max(np.abs(got[:, 3] - ref["var"]) / np.abs(ref["var"])) < 1e-9


@pytest.mark.gpu
def test_bench_cli_rows(tmp_path):
    out = tmp_path / "r.csv"
    rc = cli.main(["bench", "--out", str(out), "--reps", "2", "--dims", "1,2", "--n-samples", "2000",
                   "--n-test", "100", "--memory-cap", str(1 << 21), "--quiet"])
    assert rc == cli.EXIT_OK
    rows = cli.read_results_csv(out)
    skips = [r for r in rows if r[4] == cli.SKIP_PHASE]
    timed = [r for r in rows if r[4] != cli.SKIP_PHASE]
    assert timed and all(r[0] == "cuda" and r[5] >= 0 for r in timed)
    assert skips  # p=1, n=128 at N=2000 (2.18 MB estimate) exceeds a 2 MiB cap: the reference's sentinel
    assert cli.main(["plotdata", "--results", str(out), "--out-dir", str(tmp_path)]) == cli.EXIT_OK
