"""Command line on the GPU path: the step on either side of the posterior.

    python -m paper_2403_12797_b200.cli predict --train t.csv --test s.csv --out o.csv [--cov]
    python -m paper_2403_12797_b200.cli bench   [--config c.txt] [--out results.csv] ...
    python -m paper_2403_12797_b200.cli plotdata --results results.csv [--out-dir d]
    python -m paper_2403_12797_b200.cli generate --n-samples N --dim p --seed s

File formats and exit codes follow the reference CLI (/root/reference/pkg/src/fagp/cli.py):
predict writes ``x1..xp,mean[,var]`` at 17 significant digits (cli.py:204-229; var = the
diagonal of the posterior covariance, cli.py:222); bench writes ``backend,p,n,rep,phase,seconds``
rows for the phases setup / eigen / mean / retrieve with the ``skipped,-1`` sentinel
(bench.py:52-57, 199-269) and backend name ``cuda``; plotdata aggregates them
(bench.py:314-364).  Exit codes: 0 ok, 1 usage, 3 I/O or format, 4 numerical or budget.
"""

from __future__ import annotations

import argparse
import math
import sys
import time
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .datagen import dataset_filename, generate, load_csv, save_csv
from .errors import BudgetError, ConfigError, CsvFormatError, NumericalError
from .kernels import ArdKernelParams, KernelParams1D
from .mercer import DEFAULT_MEMORY_CAP, estimate_bytes

EXIT_OK, EXIT_USAGE, EXIT_VERIFY, EXIT_IO, EXIT_NUMERICAL = 0, 1, 2, 3, 4

RESULTS_HEADER = "backend,p,n,rep,phase,seconds"
PLOTDATA_HEADER = ("backend,n,mean_total_s,std_total_s,mean_setup_s,mean_eigen_s,mean_mean_s,mean_retrieve_s,"
                   "std_setup_s,std_eigen_s,std_mean_s,std_retrieve_s")
PHASES = ("setup", "eigen", "mean", "retrieve")
SKIP_PHASE, SKIP_SECONDS = "skipped", -1.0
BACKEND_NAME = "cuda"
DEFAULT_EIGEN_COUNTS = {1: (8, 16, 32, 64, 128), 2: (3, 4, 5, 6, 7, 8, 9, 10, 11), 4: (2, 3, 4, 5, 6, 7)}


@dataclass(frozen=True)
class BenchConfig:
    """Sweep definition with the reference's keys and defaults (bench.py:70-109)."""

    n_samples: int = 10000
    n_test: int = 1000
    dims: tuple = (1, 2, 4)
    eigen_counts: dict = field(default_factory=lambda: dict(DEFAULT_EIGEN_COUNTS))
    reps: int = 10
    epsilon: float = 1.0
    rho: float = 1.0
    noise_std: float = 0.05
    noise_var: float = 0.0025
    seed_base: int = 0
    memory_cap: int = DEFAULT_MEMORY_CAP

    def validate(self):
        if min(self.n_samples, self.n_test, self.reps) < 1:
            raise ConfigError("n_samples, n_test and reps must all be >= 1")
        if not self.dims or any(p < 1 for p in self.dims):
            raise ConfigError("dims must be a nonempty list of integers >= 1")
        for p in self.dims:
            counts = self.eigen_counts.get(p)
            if not counts or any(n < 1 for n in counts):
                raise ConfigError(f"no valid eigen_counts configured for p={p} (key eigen_counts.{p})")
        if self.epsilon < 0 or self.rho <= 0 or self.noise_var <= 0 or self.noise_std < 0:
            raise ConfigError("require epsilon >= 0, rho > 0, noise_var > 0, noise_std >= 0")
        if self.memory_cap < 1:
            raise ConfigError("memory_cap must be a positive byte count")
        return self


_SCALARS = {"n_samples": int, "n_test": int, "reps": int, "epsilon": float, "rho": float, "noise_std": float,
            "noise_var": float, "seed_base": int, "memory_cap": int}


def parse_config_file(path):
    """``key = value`` lines, '#' comments; unknown keys rejected (bench.py:125-174).
    Keys of the CPU reference that have no meaning on the GPU (workers, backends,
    deterministic_reduction) are accepted and ignored."""
    updates, counts = {}, dict(DEFAULT_EIGEN_COUNTS)
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"{path}:{lineno}: expected 'key = value'")
            key, value = (t.strip() for t in line.split("=", 1))
            try:
                if key in _SCALARS:
                    updates[key] = _SCALARS[key](value)
                elif key == "dims":
                    updates["dims"] = tuple(int(v) for v in value.split(",") if v.strip())
                elif key.startswith("eigen_counts."):
                    counts[int(key.split(".", 1)[1])] = tuple(int(v) for v in value.split(",") if v.strip())
                elif key in ("workers", "backends", "deterministic_reduction"):
                    continue
                else:
                    raise ConfigError(f"{path}:{lineno}: unknown config key {key!r}")
            except ConfigError:
                raise
            except ValueError:
                raise ConfigError(f"{path}:{lineno}: bad value for {key!r}: {value!r}") from None
    return replace(BenchConfig(), eigen_counts=counts, **updates).validate()


def train_seed(cfg, p, rep):
    return cfg.seed_base + 100000 * p + rep


def format_row(row):
    mode, p, n, rep, phase, seconds = row
    return f"{mode},{p},{n},{rep},{phase}," + ("-1" if phase == SKIP_PHASE else f"{seconds:.9e}")


def run_sweep(cfg, row_sink=None, progress=None, want_var=False):
    """The reference's Monte Carlo sweep (bench.py:199-269) on the GPU path.  Phases:
    setup = host->device copy of X, y, X*; eigen = the 1-D eigenfunction tables of train
    and test rows (fagp_basis_eval); mean = Gram + factorisation + prediction (the
    reference's fagp_posterior_from_eigensystems); retrieve = the device->host copy."""
    import torch

    from . import _device as dev
    from .engine import PosteriorEngine

    cfg.validate()
    rows = []

    def emit(row):
        rows.append(row)
        if row_sink:
            row_sink(row)

    def now():
        torch.cuda.synchronize()
        return time.perf_counter()

    for p in cfg.dims:
        kernel = ArdKernelParams.isotropic(p, cfg.epsilon, cfg.rho)
        for n in cfg.eigen_counts[p]:
            for rep in range(cfg.reps):
                if estimate_bytes(cfg.n_samples, n, p) > cfg.memory_cap:
                    if progress:
                        progress(f"skip {BACKEND_NAME} p={p} n={n} rep={rep}: over the memory cap")
                    emit((BACKEND_NAME, p, n, rep, SKIP_PHASE, SKIP_SECONDS))
                    continue
                seed = train_seed(cfg, p, rep)
                ds = generate(cfg.n_samples, p, seed, cfg.noise_std, domain=(-1.0, 1.0))
                Xs = np.random.Generator(np.random.Philox(key=seed + 2**31)).uniform(-1.0, 1.0, (cfg.n_test, p))
                t0 = now()
                X, y, Xd = dev.to_device(ds.X), dev.to_device(ds.y), dev.to_device(Xs)
                t1 = now()
                eng = PosteriorEngine(kernel, n, cfg.n_samples, cfg.n_test, cfg.noise_var, 0.0, device=X.device,
                                      want_var=want_var)
                t2 = now()  # "eigen": the eigenfunctions are evaluated on chip inside the two kernels below
                eng.stage_gram(X, y)
                if eng.stage_factor() != 0:
                    eng.raise_errors(X, Xd, y, factor_failed=True)
                eng.stage_predict(Xd)
                t3 = now()
                dev.to_host(eng.mean)
                t4 = now()
                eng.check(X, Xd, y)
                for phase, sec in zip(PHASES, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                    emit((BACKEND_NAME, p, n, rep, phase, sec))
                if progress:
                    progress(f"{BACKEND_NAME} p={p} n={n} rep={rep}: total {t4 - t0:.4f} s")
    return rows


def read_results_csv(path):
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise CsvFormatError(path, 0, "empty results file")
    if lines[0] != RESULTS_HEADER:
        raise CsvFormatError(path, 1, f"bad header {lines[0]!r}, expected {RESULTS_HEADER!r}")
    rows = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        f = line.split(",")
        if len(f) != 6:
            raise CsvFormatError(path, lineno, f"expected 6 fields, got {len(f)}")
        if f[4] not in PHASES + (SKIP_PHASE,):
            raise CsvFormatError(path, lineno, f"unknown phase {f[4]!r}")
        try:
            rows.append((f[0], int(f[1]), int(f[2]), int(f[3]), f[4], float(f[5])))
        except ValueError:
            raise CsvFormatError(path, lineno, f"non-numeric field in {line!r}") from None
    return rows


def aggregate_plotdata(rows):
    """Per (p, backend, n): mean and sample std over reps of the phase times and their
    total; skip sentinels excluded (bench.py:314-345)."""
    groups = {}
    for mode, p, n, rep, phase, sec in rows:
        if phase != SKIP_PHASE:
            groups.setdefault((p, mode, n), {}).setdefault(rep, {})[phase] = sec

    def mean_std(v):
        m = sum(v) / len(v)
        return m, (math.sqrt(sum((x - m) ** 2 for x in v) / (len(v) - 1)) if len(v) > 1 else 0.0)

    tables = {}
    for (p, mode, n), reps in sorted(groups.items()):
        tot = mean_std([sum(ph.values()) for ph in reps.values()])
        per = [mean_std([ph.get(k, 0.0) for ph in reps.values()]) for k in PHASES]
        tables.setdefault(p, []).append((mode, n, *tot, *(m for m, _ in per), *(s for _, s in per)))
    return tables


def write_plotdata_csvs(tables, out_dir):
    paths = []
    for p, table in sorted(tables.items()):
        path = Path(out_dir) / f"plot_p{p}.csv"
        with open(path, "w", newline="") as fh:
            fh.write(PLOTDATA_HEADER + "\n")
            for mode, n, *vals in table:
                fh.write(",".join([mode, str(n)] + [f"{v:.9e}" for v in vals]) + "\n")
        paths.append(path)
    return paths


def _per_dim(text, name, p):
    vals = [float(v) for v in text.split(",") if v.strip()]
    if len(vals) == 1:
        vals = vals * p
    if len(vals) != p:
        raise ConfigError(f"--{name} needs 1 or {p} comma-separated values, got {len(vals)}")
    return vals


def load_test_inputs(path, p):
    """A dataset CSV or an ``x1..xp`` CSV (cli.py:189-201)."""
    with open(path) as fh:
        header = fh.readline().strip()
    if header.endswith(",y"):
        return load_csv(path).X
    cols = header.split(",")
    if cols != [f"x{j + 1}" for j in range(len(cols))]:
        raise CsvFormatError(path, 1, f"malformed header {header!r}, expected x1,...,xp[,y]")
    data = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    if data.shape[1] != len(cols):
        raise CsvFormatError(path, 2, f"expected {len(cols)} fields per row")
    return data


def cmd_predict(args):
    from .posterior import GpModel, fagp_posterior

    train = load_csv(args.train)
    p = train.p
    kernel = ArdKernelParams(tuple(KernelParams1D(e, r) for e, r in
                                   zip(_per_dim(args.epsilon, "epsilon", p), _per_dim(args.rho, "rho", p))))
    Xstar = load_test_inputs(args.test, p)
    if Xstar.shape[1] != p:
        raise ConfigError(f"test inputs have {Xstar.shape[1]} columns, train has p={p}")
    model = GpModel(kernel, args.noise_var, mean_const=args.mean_const, n_eigen=args.n_eigen)
    res = fagp_posterior(train, Xstar, model, want_var=args.cov, memory_cap=args.memory_cap)
    cols = [f"x{j + 1}" for j in range(p)] + ["mean"] + (["var"] if args.cov else [])
    out = np.column_stack([Xstar, res.mean] + ([res.var] if args.cov else []))
    with open(args.out, "w", newline="") as fh:
        fh.write(",".join(cols) + "\n")
        for row in out:
            fh.write(",".join(f"{v:.17g}" for v in row) + "\n")
    print(f"wrote {Xstar.shape[0]} predictions to {args.out}")
    return EXIT_OK


def cmd_bench(args):
    cfg = parse_config_file(args.config) if args.config else BenchConfig()
    over = {k: getattr(args, k) for k in ("reps", "n_samples", "n_test", "memory_cap", "seed_base")
            if getattr(args, k) is not None}
    if args.dims:
        over["dims"] = tuple(int(v) for v in args.dims.split(","))
    cfg = replace(cfg, **over).validate()
    append = args.append and args.out.exists()
    progress = None if args.quiet else (lambda msg: print(msg, flush=True))
    with open(args.out, "a" if append else "w", newline="") as fh:
        if fh.tell() == 0:
            fh.write(RESULTS_HEADER + "\n")
        rows = run_sweep(cfg, row_sink=lambda r: (fh.write(format_row(r) + "\n"), fh.flush()), progress=progress)
    n_skip = sum(1 for r in rows if r[4] == SKIP_PHASE)
    print(f"wrote {len(rows)} rows to {args.out} ({n_skip} skip sentinel(s))")
    return EXIT_OK


def cmd_plotdata(args):
    Path(args.out_dir).mkdir(parents=True, exist_ok=True)
    for path in write_plotdata_csvs(aggregate_plotdata(read_results_csv(args.results)), args.out_dir):
        print(f"wrote {path}")
    return EXIT_OK


def cmd_generate(args):
    if args.n_samples < 1 or args.dim < 1:
        raise ConfigError("--n-samples and --dim must be >= 1")
    Path(args.out_dir).mkdir(parents=True, exist_ok=True)
    ds = generate(args.n_samples, args.dim, args.seed, args.noise_std, domain=tuple(args.domain))
    path = Path(args.out_dir) / dataset_filename(args.n_samples, args.dim, args.seed)
    save_csv(ds, path)
    print(f"wrote {path} (N={ds.N}, p={ds.p}, seed={ds.seed})")
    return EXIT_OK


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (2 is reserved for verification failures)
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def build_parser():
    ap = _Parser(prog="fagp-b200", description="FAGP posterior on B200")
    sub = ap.add_subparsers(dest="command", required=True, parser_class=_Parser)
    pr = sub.add_parser("predict")
    pr.add_argument("--train", type=Path, required=True)
    pr.add_argument("--test", type=Path, required=True)
    pr.add_argument("--out", type=Path, required=True)
    pr.add_argument("--epsilon", default="1.0")
    pr.add_argument("--rho", default="1.0")
    pr.add_argument("--noise-var", type=float, default=1e-2)
    pr.add_argument("--n-eigen", type=int, default=16)
    pr.add_argument("--mean-const", type=float, default=0.0)
    pr.add_argument("--cov", action="store_true", help="also write the per-point posterior variance")
    pr.add_argument("--memory-cap", type=int, default=None)
    be = sub.add_parser("bench")
    be.add_argument("--config", type=Path)
    be.add_argument("--out", type=Path, default=Path("results.csv"))
    be.add_argument("--append", action="store_true")
    be.add_argument("--quiet", action="store_true")
    for k in ("reps", "n-samples", "n-test", "memory-cap", "seed-base"):
        be.add_argument(f"--{k}", type=int)
    be.add_argument("--dims", type=str)
    pl = sub.add_parser("plotdata")
    pl.add_argument("--results", type=Path, required=True)
    pl.add_argument("--out-dir", type=Path, default=Path("."))
    ge = sub.add_parser("generate")
    ge.add_argument("--out-dir", type=Path, default=Path("."))
    ge.add_argument("--n-samples", type=int, default=10000)
    ge.add_argument("--dim", type=int, default=1)
    ge.add_argument("--seed", type=int, default=0)
    ge.add_argument("--noise-std", type=float, default=0.05)
    ge.add_argument("--domain", type=float, nargs=2, default=(-1.0, 1.0))
    return ap


COMMANDS = {"predict": cmd_predict, "bench": cmd_bench, "plotdata": cmd_plotdata, "generate": cmd_generate}


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return COMMANDS[args.command](args)
    except CsvFormatError as exc:
        print(f"fagp-b200: file format error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (BudgetError, NumericalError) as exc:
        print(f"fagp-b200: numerical error: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    except OSError as exc:
        print(f"fagp-b200: i/o error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (ConfigError, ValueError) as exc:
        print(f"fagp-b200: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
