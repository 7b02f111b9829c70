"""Command line front end (the reference declares `spgemm = spgemm.cli:main`,
pyproject.toml:15, but ships no cli module; its intended surface is SPEC.md's
External Interfaces: subcommands gen / spgemm / microbench / bound / bandwidth /
verify, flags --algo --threads --reps --seed --l2-bytes --cache-line
--mem-budget --force-fine-only --csv --json, environment overrides with a
prefix, exit codes 0 success / 1 verification failure / 2 usage error).

    python -m paper_2501_07056_b200.cli gen rmat --scale 14 --edge-factor 16 -o a.spgc
    python -m paper_2501_07056_b200.cli spgemm a.spgc [b.spgc] --algo magnus --reps 3 --json
    python -m paper_2501_07056_b200.cli verify a.spgc
    python -m paper_2501_07056_b200.cli bound a.spgc
    python -m paper_2501_07056_b200.cli bandwidth
    python -m paper_2501_07056_b200.cli microbench --size 16777216 --length 1048576 --chunks 256

Every flag can also come from the environment as MAGNUS_<FLAG> (e.g.
MAGNUS_L2_BYTES=232448, MAGNUS_ALGO=esc); an explicit flag wins.  SpGEMM runs
on the current CUDA device (there is no CPU path); inputs are Matrix Market or
SPGC files (mmio.py).
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

ENV_PREFIX = "MAGNUS_"
EXIT_OK, EXIT_VERIFY, EXIT_USAGE = 0, 1, 2
CSV_FIELDS = ["benchmark", "params", "rep", "seconds", "rate", "unit"]


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def _env_defaults(p: argparse.ArgumentParser):
    """MAGNUS_<DEST> environment values become defaults (flags still win)."""
    for a in p._actions:
        if not a.option_strings or a.dest in ("help",):
            continue
        v = os.environ.get(ENV_PREFIX + a.dest.upper())
        if v is None:
            continue
        if isinstance(a, argparse._StoreTrueAction):
            a.default = v.lower() in ("1", "true", "yes", "on")
        else:
            a.default = a.type(v) if a.type else v


def _sys_flags(p):
    p.add_argument("--l2-bytes", type=int, default=None, help="SystemParams.l2_bytes (default: device probe)")
    p.add_argument("--cache-line", type=int, default=None, help="SystemParams.cache_line_bytes")
    p.add_argument("--mem-budget", type=int, default=None, help="SystemParams.memory_budget_bytes")
    p.add_argument("--force-fine-only", action="store_true")
    p.add_argument("--threads", type=int, default=1, help="accepted for API compatibility (device decides)")


def _out_flags(p):
    p.add_argument("--csv", default=None, help="append records to this CSV file")
    p.add_argument("--json", action="store_true", help="print records as JSON lines")


def build_parser():
    p = _Parser(prog="magnus-b200", description="B200 MAGNUS SpGEMM command line")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    g = sub.add_parser("gen", help="generate a matrix file (Matrix Market or .spgc/.bin cache)")
    g.add_argument("kind", choices=["rmat", "er", "banded", "config"])
    g.add_argument("-o", "--out", required=True)
    g.add_argument("--scale", type=int, default=12)
    g.add_argument("--edge-factor", type=int, default=16)
    g.add_argument("--n", type=int, default=4096, help="er: rows/cols")
    g.add_argument("--per-row", type=int, default=16, help="er: distinct columns per row")
    g.add_argument("--grid", type=int, default=16, help="banded: 27-point stencil grid edge")
    g.add_argument("--config", type=int, default=1, help="config: BASELINE.json config 1-4 (A only)")
    g.add_argument("--seed", type=int, default=1)

    s = sub.add_parser("spgemm", help="C = A.B on the device, timed")
    s.add_argument("a")
    s.add_argument("b", nargs="?")
    s.add_argument("--algo", choices=["magnus", "dense", "esc"], default="magnus")
    s.add_argument("--reps", type=int, default=1)
    s.add_argument("-o", "--out", default=None, help="write C to this file")
    _sys_flags(s)
    _out_flags(s)

    v = sub.add_parser("verify", help="MAGNUS against the Gustavson baselines: pattern bit-exact, values 1e-12")
    v.add_argument("a")
    v.add_argument("b", nargs="?")
    v.add_argument("--rtol", type=float, default=1e-12)
    _sys_flags(v)

    bd = sub.add_parser("bound", help="the paper's ideal-bound data volume and time (bound.py)")
    bd.add_argument("a")
    bd.add_argument("b", nargs="?")
    bd.add_argument("--bandwidth", type=float, default=None, help="bytes/s (default: measured device copy rate)")
    bd.add_argument("--s-val", type=int, default=8)
    _out_flags(bd)

    bw = sub.add_parser("bandwidth", help="device copy bandwidth (index+value arrays)")
    bw.add_argument("--bytes", type=int, default=1 << 30)
    bw.add_argument("--reps", type=int, default=5)
    _out_flags(bw)

    mb = sub.add_parser("microbench", help="locality-generation building blocks on the device")
    mb.add_argument("--size", type=int, default=1 << 24, help="stream elements")
    mb.add_argument("--length", type=int, default=1 << 20, help="index range")
    mb.add_argument("--chunks", type=int, default=256, help="chunks (power of two)")
    mb.add_argument("--reps", type=int, default=3)
    mb.add_argument("--seed", type=int, default=0)
    _out_flags(mb)
    for sp in (g, s, v, bd, bw, mb):
        _env_defaults(sp)
    return p


def _emit(args, records):
    if getattr(args, "json", False):
        for r in records:
            print(json.dumps(r))
    if getattr(args, "csv", None):
        new = not os.path.exists(args.csv)
        with open(args.csv, "a", newline="") as f:
            w = csv.DictWriter(f, fieldnames=CSV_FIELDS)
            if new:
                w.writeheader()
            for r in records:
                w.writerow({k: (json.dumps(r[k]) if k == "params" else r.get(k)) for k in CSV_FIELDS})
    if not getattr(args, "json", False):
        for r in records:
            print(f"{r['benchmark']:>14}  rep {r['rep']}  {r['seconds'] * 1e3:10.3f} ms  {r['rate']:.4g} {r['unit']}")


def _sysparams(args):
    from .planner import detect_device_params, with_overrides

    over = {k: v for k, v in (("l2_bytes", args.l2_bytes), ("cache_line_bytes", args.cache_line),
                              ("memory_budget_bytes", args.mem_budget)) if v is not None}
    return with_overrides(detect_device_params(), **over) if over else None


def _load(args):
    import torch

    from .mmio import read_matrix

    dev = f"cuda:{torch.cuda.current_device()}"
    A = read_matrix(args.a, device=dev)
    B = read_matrix(args.b, device=dev) if args.b else A
    return A, B


def _cmd_gen(args):
    from . import generate
    from .mmio import write_matrix

    if args.kind == "rmat":
        m = generate.rmat(args.scale, args.edge_factor, args.seed)
    elif args.kind == "er":
        m = generate.uniform_rows(args.n, args.n, args.per_row, args.seed)
    elif args.kind == "banded":
        m = generate.stencil27(args.grid)
    else:
        if args.config not in (1, 2, 3, 4):
            raise SystemExit(EXIT_USAGE)
        m = generate.make_config_cpu(args.config)[0]
    write_matrix(m, args.out)
    print(f"wrote {args.out}: {m.n_rows} x {m.n_cols}, nnz {m.nnz}")
    return EXIT_OK


def _run(algo, A, B, args):
    from . import gustavson
    from .magnus import spgemm_magnus

    if algo == "magnus":
        return spgemm_magnus(A, B, sys=_sysparams(args), threads=args.threads, force_fine_only=args.force_fine_only)
    return (gustavson.gustavson_dense if algo == "dense" else gustavson.gustavson_esc)(A, B, threads=args.threads)


def _cmd_spgemm(args):
    import torch

    from .mmio import write_matrix

    A, B = _load(args)
    records, res = [], None
    for rep in range(max(1, args.reps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = _run(args.algo, A, B, args)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        prods = res.counters["inter_prod_size"]
        records.append({"benchmark": f"spgemm_{args.algo}", "rep": rep, "seconds": dt, "rate": 2 * prods / dt / 1e9,
                        "unit": "GFLOP/s", "params": {"a": args.a, "b": args.b or args.a, **res.counters,
                                                      "phase_timings": res.phase_timings}})
    _emit(args, records)
    if args.out:
        write_matrix(res.C, args.out)
    return EXIT_OK


def _cmd_verify(args):
    import torch

    A, B = _load(args)
    m = _run("magnus", A, B, args)
    worst = 0.0
    for algo in ("dense", "esc"):
        g = _run(algo, A, B, args)
        if not (torch.equal(g.C.row_ptr, m.C.row_ptr) and torch.equal(g.C.col, m.C.col)):
            print(f"FAIL: pattern of {algo} differs from magnus")
            return EXIT_VERIFY
        d = (g.C.val - m.C.val).abs()
        scale = torch.maximum(g.C.val.abs(), m.C.val.abs())
        bad = d > args.rtol * scale
        # allowing for summation order: entries that cancel are held to 1e-12 of the row's value scale
        if bool(bad.any()):
            tol = args.rtol * m.C.val.abs().max()
            if bool((d[bad] > tol).any()):
                print(f"FAIL: {algo} values differ beyond {args.rtol} relative (max |diff| {float(d.max()):.3g})")
                return EXIT_VERIFY
        worst = max(worst, float((d / scale.clamp_min(1e-300)).max()) if d.numel() else 0.0)
    print(f"PASS: nnz(C) {int(m.C.row_ptr[-1])}, magnus == dense == esc pattern, max relative value difference {worst:.3g}")
    return EXIT_OK


def _device_bandwidth(nbytes: int, reps: int) -> float:
    """Best-of-reps device copy rate of an int64 index + f64 value array pair (reads + writes)."""
    import torch

    n = max(1, nbytes // 16)
    src = torch.ones(2 * n, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    best = None
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return 2 * src.numel() * 8 / best


def _cmd_bandwidth(args):
    bw = _device_bandwidth(args.bytes, args.reps)
    _emit(args, [{"benchmark": "bandwidth", "rep": 0, "seconds": 2 * args.bytes / bw, "rate": bw / 1e9, "unit": "GB/s",
                  "params": {"bytes": args.bytes}}])
    return EXIT_OK


def _cmd_bound(args):
    from .bound import bound_inputs_for, ideal_bound
    from .magnus import spgemm_magnus

    A, B = _load(args)
    res = spgemm_magnus(A, B)
    bw = args.bandwidth or _device_bandwidth(1 << 30, 3)
    rd, wr, t = ideal_bound(bound_inputs_for(A, B, res.counters["nnz_c"], res.counters["inter_prod_size"], bw,
                                             s_val=args.s_val))
    _emit(args, [{"benchmark": "ideal_bound", "rep": 0, "seconds": t, "rate": (rd + wr) / 1e9, "unit": "GB",
                  "params": {"read_bytes": rd, "write_bytes": wr, "bandwidth": bw, **res.counters}}])
    return EXIT_OK


def _cmd_microbench(args):
    from .microbench import StreamSpec, microbench_building_blocks

    recs = microbench_building_blocks(StreamSpec(args.size, args.length, args.seed), args.chunks, reps=args.reps)
    _emit(args, [{"benchmark": r.name, "rep": r.rep, "seconds": r.seconds, "rate": r.rate / 1e9, "unit": "Gelem/s",
                  "params": r.params} for r in recs])
    return EXIT_OK


def main(argv=None) -> int:
    from .errors import SpgemmError

    args = build_parser().parse_args(argv)
    try:
        return {"gen": _cmd_gen, "spgemm": _cmd_spgemm, "verify": _cmd_verify, "bound": _cmd_bound,
                "bandwidth": _cmd_bandwidth, "microbench": _cmd_microbench}[args.cmd](args)
    except (SpgemmError, OSError) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_USAGE if isinstance(e, (OSError, ValueError)) else EXIT_VERIFY


if __name__ == "__main__":
    sys.exit(main())
