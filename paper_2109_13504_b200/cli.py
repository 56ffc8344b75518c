"""Command line of the B200 backend -- the reference CLI (``megores``, M/bench.py:1-414) with
the resampling work on the GPU.

    python -m paper_2109_13504_b200 quality --algorithms megopolis,c1:128 --n-grid 1024,4096 ...
    python -m paper_2109_13504_b200 pf --algorithms megopolis,systematic --n 65536 ...
    python -m paper_2109_13504_b200 gen-weights --family gaussian --param 2 --n 4096 --out w.bin
    python -m paper_2109_13504_b200 plotdata --results results.csv --figure mse-vs-N

Same subcommands, flags, JSON config keys (unknown keys are an error), profiles, CSV schema
line and float formatting (shortest round-trip ``repr``), and the same exit status 2 with a
``megores: error:`` message on bad input (M/bench.py:362-368).  Experiment coordinates and
seeds are derived exactly as the reference does (M/bench.py:87-149), the weights come from the
reference's own formulas (numpy, ``weights.gen_*``), and the resamplers, the B rule, the
offspring histogram and the quality statistics are this package's bit-exact device paths -- so
a ``quality`` CSV is byte-identical to the reference's for the same spec
(tests/test_cli_gpu.py).  ``pf`` rows agree to ~1e-9 (the filter's libm-rounded stages,
DESIGN.md §8a).  ``traffic`` is the reference's analytical transaction model (M/warpsim.py),
which has no GPU counterpart here: measured sectors per request come from ncu instead
(DESIGN.md §4).

Extra flags: ``--rng megores|philox`` (default megores, the reference's stream);
``--device-weights-from N`` (quality, gen-weights): populations of at least N particles
(default 2^24, above every profile's grid) are synthesised in HBM by the device generators
(``weights.gen_gaussian_weights`` / ``gen_gamma_weights`` with ``device=``).
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from dataclasses import dataclass, field, fields

import numpy as np

from . import rng as _rng
from . import storage

SCHEMA_LINE = "# megores-results v1"  # M/bench.py:41
PROFILES = {  # M/bench.py:43-46
    "desk": {"n_grid": [1 << 10, 1 << 12, 1 << 14, 1 << 16], "k_runs": 32, "sequences": 4},
    "paper": {"n_grid": [1 << e for e in range(6, 23)], "k_runs": 256, "sequences": 16},
}
FAMILY_PARAMS = {"gaussian": [0.0, 1.0, 2.0, 3.0, 4.0], "gamma": [0.5, 2.0, 3.0, 10.0, 50.0]}
FIGURES = ("mse-vs-N", "bias-contribution", "traffic-ratio", "rmse-vs-B")


@dataclass
class ExperimentSpec:  # M/bench.py:53-80 (same keys and defaults)
    algorithms: list = field(default_factory=lambda: ["megopolis", "metropolis", "c1:128", "c2:128"])
    n_grid: list = field(default_factory=lambda: list(PROFILES["desk"]["n_grid"]))
    family: str = "gaussian"
    params: list | None = None
    k_runs: int = 32
    sequences: int = 4
    epsilon: float = 0.01
    seed: int = 0
    precision: str = "single"
    out: str = "results.csv"
    traffic_b: int = 8
    pf_n: int = 1 << 16
    pf_b_grid: list = field(default_factory=lambda: [16, 32, 64])
    pf_trajectories: int = 4
    pf_runs: int = 10
    pf_t_steps: int = 100

    def __post_init__(self):
        if self.family not in FAMILY_PARAMS:
            raise ValueError(f"unknown weight family {self.family!r}")
        if self.params is None:
            self.params = list(FAMILY_PARAMS[self.family])
        if not (self.algorithms and self.n_grid and self.params):
            raise ValueError("algorithm, N, and parameter grids must be non-empty")
        if self.k_runs < 2:
            raise ValueError("k_runs must be >= 2")


def algorithm_token(token: str):
    """'c1:128' -> ('c1', 128); bare names carry no partition size (M/bench.py:88-97)."""
    from .resample import ALGORITHMS

    name, _, part = token.partition(":")
    if name not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {name!r} (choose from {', '.join(ALGORITHMS)})")
    part_bytes = int(part) if part else None
    if name in ("c1", "c2") and part_bytes is None:
        raise ValueError(f"{name} needs a partition size, e.g. {name}:128")
    return name, part_bytes


parse_algorithm = algorithm_token  # the reference's name (M/bench.py:88)


def token_id(token: str) -> int:
    """The algorithm's seed coordinate: its first 8 bytes, little-endian (M/bench.py:83-85)."""
    return int.from_bytes(token.encode()[:8].ljust(8, b"\0"), "little")


# Populations of at least this many particles are synthesised in HBM (mgp_gen_gaussian /
# mgp_gen_gamma) instead of by the reference's host formulas: --device-weights-from.  The
# default lies above the paper profile's largest N (2^22), so the desk and paper grids keep the
# reference's exact weight bytes (and byte-identical CSVs); 2^24 .. 2^28 grids skip the host
# detour (scipy's gamma.ppf alone is ~1 s per 2^20 draws) at ~1e-14 relative (gamma) or
# last-bit libm (gaussian) agreement with the host bytes.
DEVICE_WEIGHTS_FROM = 1 << 24


def experiment_weights(spec: ExperimentSpec, n: int, param: float, seq: int, device_from: int = DEVICE_WEIGHTS_FROM):
    """The (n, param, seq) weight vector of a grid (M/bench.py:99-104)."""
    from .weights import GammaWeightParams, GaussianWeightParams, gen_gamma_weights, gen_gaussian_weights

    wseed = _rng.derive_seed(spec.seed, 0 if spec.family == "gaussian" else 1, n, int(param * 1000), seq)
    device = "cuda" if n >= device_from else None
    if spec.family == "gaussian":
        return gen_gaussian_weights(GaussianWeightParams(param, n), wseed, spec.precision, device=device)
    return gen_gamma_weights(GammaWeightParams(param, 1.0, n), wseed, spec.precision, device=device)


def quality_grid(spec: ExperimentSpec, rng_stream: str = "megores", device_from: int = DEVICE_WEIGHTS_FROM):
    """One averaged row per (algorithm, N, parameter); statistics per weight sequence, then
    averaged across sequences (M/bench.py:107-149).  All per-run work stays in HBM."""
    import torch

    from .metrics import QualityAccumulator
    from .resample import make_resampler
    from .weights import WeightVector, iterations_for

    rows = []
    for token in spec.algorithms:
        name, part_bytes = algorithm_token(token)
        make_resampler(name, partition_bytes=part_bytes, rng=rng_stream)  # argument validation
        for n in spec.n_grid:
            for param in spec.params:
                stats, bs = [], []
                for seq in range(spec.sequences):
                    wv = experiment_weights(spec, n, param, seq, device_from)
                    w = wv if wv.on_device else WeightVector(torch.from_numpy(np.ascontiguousarray(wv.values)).cuda(),
                                                             spec.precision)
                    b = iterations_for(w, spec.epsilon).b
                    bs.append(b)
                    acc = QualityAccumulator(n)
                    seeds = [_rng.derive_seed(spec.seed, token_id(token), n, seq, k) for k in range(spec.k_runs)]
                    acc.add_runs(name, w, b, seeds, partition_bytes=part_bytes, rng=rng_stream)
                    stats.append(acc.finalize())

                def avg(attr):
                    return float(np.mean([getattr(s, attr) for s in stats]))

                rows.append({"algorithm": token, "n": n, "family": spec.family, "param": param,
                             "b_mean": float(np.mean(bs)), "k": spec.k_runs, "sequences": spec.sequences,
                             "epsilon": spec.epsilon, "seed": spec.seed, "precision": spec.precision,
                             "mse_per_particle": avg("mse_per_particle"), "mse": avg("mse"),
                             "variance": avg("variance"), "bias_sq": avg("bias_sq"),
                             "bias_contribution": avg("bias_contribution")})
    return rows


def traffic_grid(spec: ExperimentSpec):
    """Transaction-model rows for the Metropolis-family algorithms (M/bench.py:152-178)."""
    from .resample import WarpConfig
    from .warpsim import rng_draws_per_iteration, trace_algorithm, traffic_report
    from .weights import WeightVector

    rows = []
    warp = WarpConfig()
    for token in spec.algorithms:
        name, part_bytes = algorithm_token(token)
        if name in ("multinomial", "systematic"):
            continue
        for n in spec.n_grid:
            w = WeightVector(np.ones(n), spec.precision)
            report = traffic_report(trace_algorithm(name, w, spec.traffic_b, warp, part_bytes, spec.seed))
            rows.append({"algorithm": token, "n": n, "b": spec.traffic_b,
                         "partition_bytes": part_bytes if part_bytes is not None else "", "seed": spec.seed,
                         "mean_transactions": report.per_iteration_mean, "max_transactions": report.per_warp_max,
                         "total_transactions": report.total_transactions,
                         "unnecessary_words": report.unnecessary_words,
                         "rng_draws_per_iteration": rng_draws_per_iteration(name)})
    return rows


def pf_grid(spec: ExperimentSpec):
    """Filter-benchmark rows (RMSE) and the timing sidecar (resample ratio), M/bench.py:181-204."""
    from .pfilter import FilterConfig, generate_trajectory, run_benchmark

    algos = [algorithm_token(t) for t in spec.algorithms]
    trajs = [generate_trajectory(spec.pf_t_steps, 0.0, _rng.derive_seed(spec.seed, 100 + i))
             for i in range(spec.pf_trajectories)]
    raw = run_benchmark(FilterConfig(n_particles=spec.pf_n, precision=spec.precision), trajs, spec.pf_runs,
                        spec.pf_b_grid, algos, spec.seed)
    rows, timings = [], []
    for r in raw:
        part = r["partition_bytes"]
        coords = {"algorithm": r["algorithm"] if part is None else f"{r['algorithm']}:{part}", "b": r["b"],
                  "n": r["n"], "t_steps": spec.pf_t_steps, "trajectories": spec.pf_trajectories,
                  "runs": spec.pf_runs, "seed": spec.seed}
        rows.append(dict(coords, rmse=r["rmse"]))
        timings.append(dict(coords, resample_ratio=r["resample_ratio"]))
    return rows, timings


def write_csv(path, rows) -> None:
    """Schema line, header, rows; floats as shortest round-trip repr (M/bench.py:207-215)."""
    if not rows:
        raise ValueError("no rows to write")
    with open(path, "w", newline="") as fh:
        fh.write(SCHEMA_LINE + "\n")
        out = csv.DictWriter(fh, fieldnames=list(rows[0]))
        out.writeheader()
        out.writerows({k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()} for r in rows)


def read_csv(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(line for line in fh if not line.startswith("#")))


def plot_data(rows, figure: str):
    """(x, series, value) triples of one figure (M/bench.py:224-252)."""
    if figure == "traffic-ratio":
        base = {int(r["n"]): float(r["mean_transactions"]) for r in rows
                if r["algorithm"].split(":")[0] == "megopolis"}
        if not base:
            raise ValueError("traffic-ratio needs a megopolis series as baseline")
        trip = [(int(r["n"]), r["algorithm"], float(r["mean_transactions"]) / base[int(r["n"])]) for r in rows]
    elif figure in ("mse-vs-N", "bias-contribution"):
        col = "mse_per_particle" if figure == "mse-vs-N" else "bias_contribution"
        trip = [(int(r["n"]), f"{r['algorithm']}|{r['param']}", float(r[col])) for r in rows]
    elif figure == "rmse-vs-B":
        trip = [(int(r["b"]), r["algorithm"], float(r["rmse"])) for r in rows]
    else:
        raise ValueError(f"unknown figure id {figure!r}")
    return [{"x": x, "series": s, "value": v} for x, s, v in trip]


# ---------------------------------------------------------------------------
# argument plumbing (M/bench.py:258-359)

def _csv_items(text, conv=str):
    if not text:
        return None
    return [conv(t.strip()) for t in text.split(",") if t.strip()]


# (flag, dest, type, help) per subcommand; "common" flags are added to all
_COMMON = [("--config", "config", str, "JSON experiment config"),
           ("--seed", "seed", int, "base seed (decimal 64-bit)"),
           ("--out", "out", str, "output CSV path")]
_FLAGS = {
    "quality": [("--profile", "profile", "profile", None), ("--precision", "precision", "precision", None),
                ("--algorithms", "algorithms", str, "comma list, e.g. megopolis,metropolis,c1:128"),
                ("--n-grid", "n_grid", str, "comma list of particle counts"),
                ("--family", "family", "family", None), ("--params", "params", str, "comma list of y / shapes"),
                ("--k-runs", "k_runs", int, None), ("--sequences", "sequences", int, None),
                ("--epsilon", "epsilon", float, None), ("--rng", "rng", "rng", None),
                ("--device-weights-from", "device_weights_from", int,
                 "synthesise populations of at least this N in HBM (default 2^24)")],
    "traffic": [("--profile", "profile", "profile", None), ("--algorithms", "algorithms", str, None),
                ("--n-grid", "n_grid", str, None), ("--b", "b", int, "iteration count to trace")],
    "pf": [("--precision", "precision", "precision", None), ("--algorithms", "algorithms", str, None),
           ("--n", "n", int, "particle count"), ("--b-grid", "b_grid", str, "comma list of budgets"),
           ("--trajectories", "trajectories", int, None), ("--runs", "runs", int, None),
           ("--t-steps", "t_steps", int, None)],
    "gen-weights": [("--precision", "precision", "precision", None), ("--family", "family", "family!", None),
                    ("--param", "param", "float!", "y or gamma shape alpha"), ("--n", "n", "int!", None),
                    ("--device-weights-from", "device_weights_from", int,
                     "generate in HBM when N is at least this (default 2^24)")],
    "plotdata": [("--results", "results", "str!", "input results CSV"), ("--figure", "figure", "figure!", None)],
}
_CHOICES = {"profile": sorted(PROFILES), "precision": ["single", "double"], "family": ["gaussian", "gamma"],
            "figure": list(FIGURES), "rng": ["megores", "philox"]}


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="megores", description="resampling quality / traffic / filter benchmarks "
                                                           "(B200 backend)")
    sub = ap.add_subparsers(dest="command", required=True)
    for cmd, flags in _FLAGS.items():
        p = sub.add_parser(cmd)
        for flag, dest, kind, hlp in _COMMON + flags:
            req = isinstance(kind, str) and kind.endswith("!")
            base = kind.rstrip("!") if isinstance(kind, str) else kind
            kw = {"dest": dest, "help": hlp, "required": req, "default": None}
            if base in _CHOICES:
                kw["choices"] = _CHOICES[base]
            else:
                kw["type"] = {"int": int, "float": float, "str": str}.get(base, base) if isinstance(base, str) else base
            p.add_argument(flag, **kw)
    return ap


def spec_from_args(args) -> ExperimentSpec:
    """JSON config, then profile, then explicit flags; unknown keys are an error (M/bench.py:258-288)."""
    values = {}
    if args.config:
        with open(args.config) as fh:
            values.update(json.load(fh))
    if getattr(args, "profile", None):
        values.update(PROFILES[args.profile])
    g = lambda k: getattr(args, k, None)  # noqa: E731
    flags = {"seed": g("seed"), "out": g("out"), "precision": g("precision"), "algorithms": _csv_items(g("algorithms")),
             "n_grid": _csv_items(g("n_grid"), int), "family": g("family"), "params": _csv_items(g("params"), float),
             "k_runs": g("k_runs"), "sequences": g("sequences"), "epsilon": g("epsilon"), "traffic_b": g("b"),
             "pf_n": g("n"), "pf_b_grid": _csv_items(g("b_grid"), int), "pf_trajectories": g("trajectories"),
             "pf_runs": g("runs"), "pf_t_steps": g("t_steps")}
    values.update({k: v for k, v in flags.items() if v is not None})
    unknown = set(values) - {f.name for f in fields(ExperimentSpec)}
    if unknown:
        raise ValueError(f"unknown config keys: {sorted(unknown)}")
    return ExperimentSpec(**values)


def _device_from(args) -> int:
    v = getattr(args, "device_weights_from", None)
    return DEVICE_WEIGHTS_FROM if v is None else int(v)


def run(args) -> int:
    cmd = args.command
    if cmd == "plotdata":
        out = args.out or "plotdata.csv"
        write_csv(out, plot_data(read_csv(args.results), args.figure))
        print(f"wrote {out}")
        return 0
    spec = spec_from_args(args)
    if cmd == "quality":
        write_csv(spec.out, quality_grid(spec, args.rng or "megores", _device_from(args)))
        print(f"wrote {spec.out}")
    elif cmd == "pf":
        rows, timings = pf_grid(spec)
        write_csv(spec.out, rows)
        write_csv(spec.out + ".timings.csv", timings)
        print(f"wrote {spec.out} (+ timings sidecar)")
    elif cmd == "gen-weights":
        from .weights import GammaWeightParams, GaussianWeightParams, WeightVector, gen_gamma_weights, gen_gaussian_weights

        device = "cuda" if args.n >= _device_from(args) else None
        if args.family == "gaussian":
            w = gen_gaussian_weights(GaussianWeightParams(args.param, args.n), spec.seed, spec.precision, device=device)
        else:
            w = gen_gamma_weights(GammaWeightParams(args.param, 1.0, args.n), spec.seed, spec.precision, device=device)
        if w.on_device:
            w = WeightVector(w.values.cpu().numpy(), spec.precision)
        storage.save_weights(spec.out, w)
        wd = np.asarray(w.values, dtype=np.float64)
        print(f"wrote {spec.out}: n={args.n} mean={wd.mean():.6g} max={wd.max():.6g} ratio={wd.mean() / wd.max():.6g}")
    elif cmd == "traffic":
        write_csv(spec.out, traffic_grid(spec))
        print(f"wrote {spec.out}")
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return run(args)
    except (ValueError, OSError) as exc:
        print(f"megores: error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
