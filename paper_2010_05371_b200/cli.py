"""Command-line front end of the GPU search, mirroring the reference CLI
(proj/tools/eapdtw_cli.cpp): the same subcommands, options, console lines and
stats JSON, with the search running on the B200 kernels.

    python -m paper_2010_05371_b200.cli search --data ref.txt --query q.txt \\
        --query-len 128 --window-ratio 0.1 --algo eap [--no-lb] [--no-tighten] \\
        [--allow-any-ratio] [--stats out.json] [--seed S]
    python -m paper_2010_05371_b200.cli bench --stats-dir DIR \\
        [--grid-lengths 128,256,512,1024] [--grid-ratios 0.1,0.2,0.3,0.4,0.5] \\
        [--algos full,lp,eap] [--synthetic 100000] [--seed 42]

Differences from the reference, all additive: ``--data``/``--query`` also
accept binary series (``.f64``/``.bin`` raw little-endian float64, ``.npy``)
so 1e8-point references need not be parsed as text; ``--device`` picks the
GPU; ``bench`` uploads its reference to HBM once for the whole grid
(``search_grid``) and ``--concurrency N`` searches N query lengths at once; ``trace`` captures the cells on the device
(``eapdtw_trace``) and writes the reference's CSV.  Exit status: 0 ok,
2 for the reference's CLI::ValidationError cases (bad --algo, ratio off the
grid, argument errors), 1 for every other error (eapdtw_cli.cpp:232-238).
"""
from __future__ import annotations

import argparse
import math
import os
import re
import sys

from . import seriesio
from .api import Algo, Context, DeviceSeries, SearchConfig, random_walk, search_grid
from .api import PRUNED, similarity_search, trace
from .seriesio import format_double

_ALGOS = {"full": Algo.full, "lp": Algo.left_prune, "eap": Algo.ea_pruned}
_RATIO_GRID = (0.1, 0.2, 0.3, 0.4, 0.5)
# std::stod with the whole string consumed (decimal or hex floats, inf/nan)
_FLOAT_PREFIX = re.compile(r"\s*[+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|"
                           r"0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)"
                           r"(?:[pP][+-]?\d+)?|inf(?:inity)?|nan)", re.IGNORECASE)


class ValidationError(Exception):
    """CLI::ValidationError (exit status 2)."""


def parse_algo(name: str) -> Algo:
    """eapdtw_cli.cpp:20-25"""
    try:
        return _ALGOS[name]
    except KeyError:
        raise ValidationError("--algo: expected one of full|lp|eap") from None


def on_ratio_grid(r: float) -> bool:
    """eapdtw_cli.cpp:39-44"""
    return any(math.fabs(r - g) < 1e-9 for g in _RATIO_GRID)


def ratio_label(r: float) -> str:
    """eapdtw_cli.cpp:52-58"""
    return format_double(r).replace(".", "p")


def parse_ub(text: str) -> float:
    """eapdtw_cli.cpp:27-37"""
    if text in ("inf", "INF", "+inf"):
        return PRUNED
    try:
        v = float.fromhex(text) if "x" in text.lower() else float(text)
    except ValueError:
        v = math.nan
    if math.isnan(v) or v < 0.0 or not _FLOAT_PREFIX.fullmatch(text):
        raise ValidationError("--ub: expected a non-negative float or 'inf'")
    return v


def result_lines(res) -> list[str]:
    """print_result (eapdtw_cli.cpp:46-50) + run_search's counter lines (:78-86)."""
    best, rep = res.best, res.report
    return [
        f"Location: {best.location}",
        f"Distance: {format_double(math.sqrt(best.distance_sq))}",
        f"Distance_sq: {format_double(best.distance_sq)}",
        f"Candidates: {rep.candidates_total}  pruned_kim: {rep.pruned_kim}"
        f"  pruned_keogh_eq: {rep.pruned_keogh_eq}  pruned_keogh_ec: {rep.pruned_keogh_ec}"
        f"  dtw_calls: {rep.dtw_calls}  dtw_abandoned: {rep.dtw_abandoned}",
        f"DP cells evaluated: {rep.dp_cells_evaluated}",
        f"Elapsed: {format_double(rep.elapsed_seconds)} s",
    ]


def bench_line(algo_name: str, length: int, ratio: float, res) -> str:
    """run_bench's per-grid-point line (eapdtw_cli.cpp:131-136)."""
    return (f"bench algo={algo_name} len={length} ratio={format_double(ratio)}"
            f" location={res.best.location} distance_sq={format_double(res.best.distance_sq)}"
            f" cells={res.report.dp_cells_evaluated}"
            f" elapsed={format_double(res.report.elapsed_seconds)}s")


def stats_file_name(algo_name: str, length: int, ratio: float) -> str:
    """eapdtw_cli.cpp:126-129"""
    return f"stats_{algo_name}_len{length}_ratio{ratio_label(ratio)}.json"


def run_search(a, out) -> int:
    """run_search (eapdtw_cli.cpp:61-89)"""
    if not a.allow_any_ratio and not on_ratio_grid(a.window_ratio):
        raise ValidationError("--window-ratio: outside the supported grid {0.1,0.2,0.3,0.4,0.5}; "
                              "pass --allow-any-ratio to override")
    algo = parse_algo(a.algo)
    reference = seriesio.read_series(a.data, mmap=True)
    query = seriesio.read_series(a.query)
    cfg = SearchConfig(query_length=a.query_len, window_ratio=a.window_ratio, algorithm=algo,
                       use_lower_bounds=not a.no_lb,
                       tighten_ub=(not a.no_tighten) and (not a.no_lb))
    ctx = Context(a.device)
    try:
        res = similarity_search(reference, query, cfg, ctx=ctx)
    finally:
        ctx.close()
    out.write("\n".join(result_lines(res)) + "\n")
    if a.stats:
        seriesio.emit_stats(res.report, res.best, a.stats)
    return 0


def run_trace(a, out) -> int:
    """run_trace (eapdtw_cli.cpp:91-108): one traced DTW of two series files."""
    sa = seriesio.read_series(a.a)
    sb = seriesio.read_series(a.b)
    ub = parse_ub(a.ub)
    algo = parse_algo(a.algo)
    ctx = Context(a.device)
    try:
        t = trace(sa, sb, algo, ub, ctx=ctx)
    finally:
        ctx.close()
    seriesio.write_trace_csv(t, a.out)
    return 0


def run_bench(a, out) -> int:
    """run_bench (eapdtw_cli.cpp:110-142): the grid on a synthetic random walk."""
    algos = [(name, parse_algo(name)) for name in a.algos]
    os.makedirs(a.stats_dir, exist_ok=True)
    max_len = max(a.grid_lengths)
    reference = random_walk(a.synthetic, a.seed)
    query = random_walk(max_len, a.seed + 1)
    ctx = Context(a.device)
    try:
        with DeviceSeries(reference, ctx=ctx) as ref:
            names = {algo: name for name, algo in algos}
            for algo, length, ratio, res in search_grid(ref, query, a.grid_lengths,
                                                        a.grid_ratios, [x for _, x in algos],
                                                        ctx=ctx, concurrency=a.concurrency):
                name = names[algo]
                seriesio.emit_stats(res.report, res.best,
                                    os.path.join(a.stats_dir, stats_file_name(name, length, ratio)))
                out.write(bench_line(name, length, ratio, res) + "\n")
                out.flush()
    finally:
        ctx.close()
    return 0


def _csv(conv):
    def parse(text):
        try:
            return [conv(t) for t in text.split(",") if t != ""]
        except ValueError:
            raise argparse.ArgumentTypeError(f"invalid list '{text}'") from None
    return parse


def _nonneg_int(text):
    v = int(text)
    if v < 0:
        raise argparse.ArgumentTypeError("expected a non-negative integer")
    return v


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors -> status 2 with "error: ..."
        raise ValidationError(message)


def make_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="eapdtw-b200", description=(
        "Exact DTW with pruning and early abandoning, plus subsequence similarity search, "
        "on the B200. Subsequence locations are 0-based."))
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    s = sub.add_parser("search", help="locate the query's nearest subsequence")
    s.add_argument("--data", required=True, help="reference series file (text, .f64, .npy)")
    s.add_argument("--query", required=True, help="query series file (text, .f64, .npy)")
    s.add_argument("--query-len", type=_nonneg_int, required=True, help="query prefix length")
    s.add_argument("--window-ratio", type=float, required=True,
                   help="warping window as a ratio of the query length")
    s.add_argument("--algo", required=True, help="DTW kernel: full|lp|eap")
    s.add_argument("--no-lb", action="store_true", help="disable the lower-bound cascade")
    s.add_argument("--no-tighten", action="store_true",
                   help="disable per-row threshold tightening")
    s.add_argument("--allow-any-ratio", action="store_true",
                   help="accept window ratios outside {0.1,0.2,0.3,0.4,0.5}")
    s.add_argument("--stats", default="", help="write run statistics (JSON) to this path")
    s.add_argument("--seed", type=_nonneg_int, default=0,
                   help="accepted for protocol compatibility; unused")
    s.add_argument("--device", type=int, default=0, help="CUDA device")

    t = sub.add_parser("trace", help="dump the evaluated DP matrix cells as CSV")
    t.add_argument("--a", required=True, help="first series file")
    t.add_argument("--b", required=True, help="second series file")
    t.add_argument("--ub", required=True, help="threshold (float or 'inf'); ignored by --algo full")
    t.add_argument("--algo", required=True, help="DTW kernel: full|lp|eap")
    t.add_argument("--out", required=True, help="output CSV path")
    t.add_argument("--device", type=int, default=0, help="CUDA device")

    b = sub.add_parser("bench", help="run the query-length x window-ratio grid")
    b.add_argument("--grid-lengths", type=_csv(int), default=[128, 256, 512, 1024])
    b.add_argument("--grid-ratios", type=_csv(float), default=[0.1, 0.2, 0.3, 0.4, 0.5])
    b.add_argument("--algos", type=_csv(str), default=["full", "lp", "eap"])
    b.add_argument("--stats-dir", required=True, help="directory for per-run statistics")
    b.add_argument("--synthetic", type=_nonneg_int, default=100000,
                   help="synthetic random-walk reference length")
    b.add_argument("--seed", type=_nonneg_int, default=42, help="random-walk seed")
    b.add_argument("--device", type=int, default=0, help="CUDA device")
    b.add_argument("--concurrency", type=int, default=1,
                   help="query lengths searched concurrently (contexts / streams); results "
                        "are identical, lines are printed once the grid completes")
    return p


def main(argv=None, out=None) -> int:
    out = out or sys.stdout
    try:
        a = make_parser().parse_args(argv)
        if a.cmd == "search":
            return run_search(a, out)
        if a.cmd == "bench":
            return run_bench(a, out)
        return run_trace(a, out)
    except ValidationError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 -- mirrors catch (const std::exception&)
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
