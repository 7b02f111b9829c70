#!/usr/bin/env python
"""Benchmark of the B200 MAGNUS SpGEMM path (BASELINE.json metric: SpGEMM GFLOP/s,
2 x multiplications, plus achieved HBM GB/s against the roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One "step" = one full spgemm_magnus(A, B) (setup + symbolic + numeric, C
materialised in HBM) on the config's seeded synthetic inputs.  Multi-GPU
(torchrun, one rank per GPU): rows of A are split into contiguous blocks of
equal flop count, B is broadcast from rank 0 over NCCL, each rank computes its
C row block; value = all products / max-over-ranks time (strong scaling).

Prints ONE JSON line on rank 0.  --impl reference times the reference
algorithm's CPU restatement (oracle/, the reference is pure Python and cannot
travel to the GPU box) on a bounded row sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# C of cfg3 is ~116 GB: avoid caching-allocator fragmentation between steps
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0   # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=40.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("BENCH_SAMPLER_MS", "100")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's own start-up (NVML init) contends with the driver: let it finish
            # before the timed region opens (the samples still cover the whole region)
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < float(os.environ.get("BENCH_SAMPLER_WAIT", "5")):
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workload
def config_desc(cfg):
    from paper_2501_07056_b200.generate import CONFIGS
    p = CONFIGS[cfg]
    names = {1: "cfg1 C=A.A uniform n=16384 16/row", 2: "cfg2 C=A.A 27-pt stencil 64^3",
             3: "cfg3 C=A.A R-MAT 2^20 ef16 (.57,.19,.19,.05)", 4: "cfg4 C=A.B uniform 2^23 8/row",
             5: "cfg5 C=A.A R-MAT 2^24 ef32"}
    return names[cfg], p


def workload_config(cfg, A, B, inter_total, world):
    """The `config` object of the JSON line: identical in both arms (--impl ours / reference)."""
    name, _ = config_desc(cfg)
    return {"workload": name, "n": int(A.n_rows), "nnz_a": int(len(A.col)), "nnz_b": int(len(B.col)),
            "inter_products": int(inter_total), "gflop": 2 * int(inter_total) / 1e9,
            "l2": "flushed (256 MB write) before each step", "dtype": "f64 values, int32 columns",
            "parallelism": f"rows split by flop over {world} GPU(s), B broadcast"}


def host_system_params():
    """The reference's detect_system_params() (planner.py:179-222) restated for the host this
    runs on: L2 size and line of cpu0 from sysfs (64 B / 1 MiB fallbacks), memory budget a
    quarter of physical memory."""
    from paper_2501_07056_b200 import SystemParams
    base = "/sys/devices/system/cpu/cpu0/cache"
    line, l2 = None, None
    try:
        for e in sorted(os.listdir(base)):
            if not e.startswith("index"):
                continue
            with open(f"{base}/{e}/level") as f:
                if f.read().strip() != "2":
                    continue
            with open(f"{base}/{e}/size") as f:
                sz = f.read().strip()
            l2 = int(sz[:-1]) * (1024 if sz.endswith("K") else 1 << 20) if sz[-1] in "KM" else int(sz)
            with open(f"{base}/{e}/coherency_line_size") as f:
                line = int(f.read().strip())
            break
    except (OSError, ValueError):
        pass
    if not line or line & (line - 1):
        line = 64
    if not l2 or l2 <= 0:
        l2 = 1 << 20
    try:
        mem = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        mem = 8 << 30
    return SystemParams(cache_line_bytes=line, l2_bytes=l2, memory_budget_bytes=max(1, mem // 4))


def algorithmic_bytes(A, B, inter, c_nnz_row, rp_bytes_a, rp_bytes_b):
    """Per device row class: (symbolic bytes, numeric bytes) -- reads of A, of the B rows each
    product touches (row_ptr pair + col [+ val]), and (numeric) the C row written.  The §8(d)
    compulsory model restricted to the rows a kernel processes."""
    import torch
    nk = (A.row_ptr[1:] - A.row_ptr[:-1]).to(torch.int64)
    classes = {"warp": (inter > 0) & (inter <= 256), "block": (inter > 256) & (inter <= 4096), "heavy": inter > 4096,
               "dense": inter > 0}
    out = {}
    for name, m in classes.items():
        nkm = int(nk[m].sum())
        im = int(inter[m].sum())
        cm = int(c_nnz_row[m].sum())
        rows = int(m.sum())
        a_bytes = rows * 2 * rp_bytes_a + nkm * 12
        b_rp = nkm * 2 * rp_bytes_b
        sym = a_bytes - nkm * 8 + b_rp + im * 4 + rows * 8
        num = a_bytes + b_rp + im * 12 + cm * 12 + rows * 16
        out[name] = {"rows": rows, "inter": im, "nnz_c": cm, "sym_bytes": sym, "num_bytes": num,
                     "a_bytes": a_bytes, "b_bytes": b_rp + im * 12, "c_bytes": cm * 12 + rows * 16}
    return out


def compulsory_bytes(n_a, nnz_a, n_inter, nnz_c, rp_a, rp_b, rp_c, n_c):
    """A once + each product's B row (rp pair + col,val) + C once."""
    return ((n_a + 1) * rp_a + nnz_a * 12) + (2 * nnz_a * rp_b + n_inter * 12) + ((n_c + 1) * rp_c + nnz_c * 12)


# ------------------------------------------------------------------ CPU baseline (oracle port)
def cpu_baseline(A_host, B_host, sysp, seconds, inter_host, seed=0):
    """Oracle (reference restated in C, OpenMP over rows) on a random row sample of the same
    workload, sized for ~`seconds` of CPU work; rate = 2*sum(inter of sample)/time."""
    from oracle import oracle
    from paper_2501_07056_b200 import CsrMatrix
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n = A_host.n_rows
    rp = np.asarray(A_host.row_ptr, dtype=np.int64)

    def sub(rows):
        rows = np.sort(rows)
        lens = rp[rows + 1] - rp[rows]
        srp = np.zeros(rows.size + 1, np.int64)
        np.cumsum(lens, out=srp[1:])
        idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows]) if rows.size else np.empty(0, np.int64)
        return CsrMatrix(rows.size, A_host.n_cols, srp, np.asarray(A_host.col)[idx], np.asarray(A_host.val)[idx]), rows

    order = rng.permutation(n)
    # calibration on a small sample
    csum = np.cumsum(inter_host[order])
    target = 2e7
    k = int(np.searchsorted(csum, target)) + 1
    As, rows = sub(order[:k])
    t = time.perf_counter()
    oracle.spgemm(As, B_host, sysp, threads=threads)
    dt = time.perf_counter() - t
    rate = max(inter_host[rows].sum(), 1) / max(dt, 1e-6)
    target = min(rate * seconds, float(csum[-1]))
    k = int(np.searchsorted(csum, target)) + 1
    As, rows = sub(order[:min(k, n)])
    t = time.perf_counter()
    oracle.spgemm(As, B_host, sysp, threads=threads)
    dt = time.perf_counter() - t
    s_inter = int(inter_host[rows].sum())
    return {"value": 2.0 * s_inter / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"{rows.size} random rows of A ({s_inter} of {int(csum[-1])} products), full symbolic+numeric, "
                      f"{dt:.1f} s on {threads} host threads"}


# ------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    from paper_2501_07056_b200 import MagnusPlan, _lib, detect_device_params, generate, row_intermediate_stats
    from paper_2501_07056_b200.parallel import distribute, rebase

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=device)
    _lib.build()
    cfg = args.config
    name, p = config_desc(cfg)
    if cfg == 5:
        return run_waves_bench(args, world, rank, local, device)

    # inputs: rank 0 generates on its GPU; with N > 1 the exchange (B broadcast over NCCL, the
    # flop cuts, each rank's block of A) is part of every timed step
    t_gen = time.perf_counter()
    if rank == 0:
        A0, B0 = generate.make_config_device(cfg, rp_dtype=torch.int64 if cfg == 5 else torch.int32)
    else:
        A0 = B0 = None
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    sysp = detect_device_params()
    if world > 1:
        A_loc, B, cuts, total_inter = distribute(A0, B0, rank, world, device)
        A = A0 if rank == 0 else A_loc
        lo, hi = cuts[rank], cuts[rank + 1]
    else:
        A, B, A_loc = A0, B0, A0
    inter_loc = row_intermediate_stats(A_loc, B).inter_size
    if world == 1:
        total_inter = int(inter_loc.sum())
        lo, hi = 0, A.n_rows

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(profile=False, timed=None):
        """One job step; with N > 1 the exchange first (timed[0] brackets the local compute)."""
        if world > 1:
            A_blk, Bx, _, _ = distribute(A0, B0, rank, world, device)
        else:
            A_blk, Bx = A_loc, B
        if timed is not None:
            timed[0].record(stream)
        plan = MagnusPlan(A_blk, Bx, sys=sysp)
        if profile:
            plan.ctx.profile(True)
        rp = plan.symbolic()
        C, counters = plan.numeric(rp)
        launches = plan.launches()
        prof = plan.ctx.profile_read() if profile else None
        if profile:
            prof["_heavy"] = plan.ctx.heavy_stats()
        plan.close()
        if timed is not None:
            timed[1].record(stream)
        if world > 1:
            rebase(C, rank, world, device)
        return C, counters, launches, prof

    for _ in range(args.warmup):
        C, counters, _, _ = step()
        del C
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    times, ctimes, launches = [], [], 0
    for _ in range(args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        C, counters, nl, _ = step(timed=(c0, c1))
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        ctimes.append(c0.elapsed_time(c1))
        launches += nl
        del C
    clocks = sampler.stop()
    total_ms, compute_ms = sum(times), sum(ctimes)
    if world > 1:
        t = torch.tensor([total_ms, compute_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, compute_ms = float(t[0]), float(t[1])
    ms_step = total_ms / args.steps
    gflops = 2.0 * total_inter / (ms_step * 1e-3) / 1e9

    # kernel-level profile (one extra step, events bracket each launch on its stream)
    C, counters, _, prof = step(profile=True)
    hs = prof.pop("_heavy")
    c_nnz_row = (C.row_ptr[1:] - C.row_ptr[:-1])
    nnz_c_local = int(C.row_ptr[-1])
    rp_a = A_loc.row_ptr.element_size()
    ab = algorithmic_bytes(A_loc, B, inter_loc, c_nnz_row, rp_a, B.row_ptr.element_size())
    del C
    peak, peak_kind = hbm_peak()
    # per-kernel algorithmic bytes, SURVEY.md §8(d)'s compulsory model restricted to what each
    # kernel must move: the heavy expand reads A and the B rows its products touch, the heavy
    # reducers write C; the light-row kernels do all three for their rows.  The reorder buffer
    # (10 B per product written by the expand and read back by the reducers) is NOT algorithmic:
    # it is reported separately as intermediate traffic.
    hv = ab["heavy"]
    kern_bytes = {"bin_expand": hv["a_bytes"] + hv["b_bytes"],
                  "bin_big": hs["big_distinct"] * 12, "bin_reduce": hs["small_distinct"] * 12,
                  "num_heavy": hv["num_bytes"], "sym_heavy": hv["sym_bytes"],
                  "num_dense": ab["dense"]["num_bytes"], "sym_dense": ab["dense"]["sym_bytes"],
                  "num_block": ab["block"]["num_bytes"], "sym_block": ab["block"]["sym_bytes"],
                  "num_warp": ab["warp"]["num_bytes"], "sym_warp": ab["warp"]["sym_bytes"]}
    inter_bytes = {"bin_expand": hv["inter"] * 10, "bin_big": hs["big_products"] * 10,
                   "bin_reduce": hs["small_products"] * 10}
    dom = max(prof, key=lambda k: prof[k][0])
    nl_dom = max(prof[dom][1], 1)
    dom_ms = prof[dom][0] / nl_dom
    dom_bytes = kern_bytes.get(dom)
    if dom_bytes is not None:
        dom_bytes = dom_bytes // nl_dom   # the class's bytes are split over its launches (row batches)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9 if dom_bytes else None
    dom_inter = inter_bytes.get(dom, 0) // nl_dom
    # the heavy-row numeric pipeline as one unit: A + B rows touched + C of the heavy rows
    heavy_keys = [k for k in ("bin_expand", "bin_big", "bin_reduce", "num_heavy", "dir_num")
                  if k in prof]
    heavy_ms = sum(prof[k][0] for k in heavy_keys)
    heavy_roof = None
    if heavy_ms > 0:
        hb = hv["num_bytes"]
        heavy_roof = {"kernels": heavy_keys, "ms": round(heavy_ms, 3), "compulsory_bytes": hb,
                      "achieved": round(hb / (heavy_ms * 1e-3) / 1e9, 1), "peak": peak,
                      "frac": round(hb / (heavy_ms * 1e-3) / 1e9 / peak, 4), "unit": "GB/s",
                      "intermediate_bytes": hv["inter"] * 20}
    # DRAM traffic per launch of that kernel: a COMMITTED ncu capture of this workload (ncu cannot
    # run inside the timed bench); null when the capture does not cover this kernel
    traffic, traffic_file = None, None
    for cand in ("r2_cfg3_traffic.json", "r1_cfg3_traffic.json"):
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", cand)))
        except (OSError, ValueError):
            continue
        if cfg == 3 and world == 1 and dom in tj.get("kernels", {}):
            traffic, traffic_file = tj["kernels"][dom]["dram_bytes_per_launch"], cand
        break
    prof_share = {k: round(v[0], 3) for k, v in prof.items() if v[1]}

    # whole-job compulsory roofline
    nnz_c = nnz_c_local
    if world > 1:
        t = torch.tensor([nnz_c], dtype=torch.int64, device=device)
        dist.all_reduce(t)
        nnz_c = int(t)
    comp = compulsory_bytes(A.n_rows, A.col.numel(), total_inter, nnz_c, A.row_ptr.element_size(),
                            B.row_ptr.element_size(), 8, A.n_rows)
    # the paper's two-pass minimum-data-volume model (reference bound.py:44-72), for comparability
    from paper_2501_07056_b200 import bound_inputs_for, ideal_bound
    ib_r, ib_w, ib_t = ideal_bound(bound_inputs_for(A, B, nnz_c, total_inter, peak * 1e9 * world))
    ideal = {"read_bytes": int(ib_r), "write_bytes": int(ib_w), "t_ideal_ms": round(ib_t * 1e3, 3),
             "multiple": round(ms_step / (ib_t * 1e3), 2), "bandwidth": "measured HBM peak x n_gpus"}

    # e2e: host buffers through the public API (H2D of A, B + D2H of C inside the timed region)
    e2e = None
    if not args.no_e2e:
        # every rank: its row block of A and all of B from host memory, its C block back to host
        e2e = run_e2e(A_loc, B, sysp, args.e2e_steps or max(1, min(args.steps, 3)), total_inter)
        if world > 1:
            t = torch.tensor([e2e["ms_per_step"], e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]],
                             dtype=torch.float64, device=device)
            tmax = t.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(t)
            ms = float(tmax[0])
            e2e = {"value": round(2.0 * total_inter / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                   "h2d_bytes_per_step": int(t[1]), "d2h_bytes_per_step": int(t[2]), "ms_per_step": round(ms, 2),
                   "steps": e2e["steps"], "timing": "max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        A_h = A.numpy() if hasattr(A, "numpy") else A
        B_h = A_h if B is A else B.numpy()
        cpu = cpu_baseline(A_h, B_h, host_system_params(), args.cpu_seconds, inter_loc.cpu().numpy())

    if rank == 0:
        line = {
            "metric": "SpGEMM GFLOP/s (2 x mults)",
            "value": round(gflops, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded, generated on device; BASELINE.json config shapes and value distributions)",
            "config": workload_config(cfg, A, B, total_inter, world),
            "nnz_c": nnz_c,
            "system_params": {"cache_line_bytes": sysp.cache_line_bytes, "l2_bytes": sysp.l2_bytes},
            "ms_per_step_compute_only": round(compute_ms / args.steps, 4),
            "timing": "CUDA events on the launching stream, max over ranks; N>1 steps include the B broadcast, "
                      "the flop cuts and the A-block exchange",
            "hbm_gbs_compulsory": round(comp / (ms_step * 1e-3) / 1e9, 1),
            "roofline_step": {"bound": "hbm", "compulsory_bytes": comp,
                              "achieved": round(comp / (ms_step * 1e-3) / 1e9, 1), "peak": peak * world,
                              "frac": round(comp / (ms_step * 1e-3) / 1e9 / (peak * world), 4), "unit": "GB/s"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1) if achieved else None,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
                         "traffic_source": (f"committed ncu capture profiles/{traffic_file} (dram__bytes_read+write "
                                            "per launch; not measured in this run)") if traffic else None,
                         "algorithmic_bytes_per_launch": dom_bytes, "bytes_model": "SURVEY.md 8(d) compulsory share",
                         "intermediate_bytes_per_launch": dom_inter, "ms_per_launch": round(dom_ms, 4)},
            "roofline_heavy": heavy_roof,
            "ideal_bound": ideal,
            "kernel_ms": prof_share,
            "heavy_chunks": hs,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "gen_s": round(t_gen, 2),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_waves_bench(args, world, rank, local, device):
    """cfg5 (R-MAT 2^24 ef32, C ~1.3e12 nonzeros ~ 15 TB: no HBM holds it): each
    rank computes its flop-balanced row block in row waves (waves.py) into a reused C buffer;
    every wave's C block is materialised in HBM and discarded.  Timed: the exchange (N > 1) and
    all waves.  No e2e (C cannot be read back), no kernel profile step."""
    import torch
    import torch.distributed as dist

    from paper_2501_07056_b200 import detect_device_params, generate, row_intermediate_stats
    from paper_2501_07056_b200.parallel import distribute
    from paper_2501_07056_b200.waves import spgemm_magnus_waves

    t_gen = time.perf_counter()
    A0 = generate.make_config_device(5, rp_dtype=torch.int64)[0] if rank == 0 else None
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    sysp = detect_device_params()
    stream = torch.cuda.current_stream()

    def step():
        if world > 1:
            A_blk, Bx, cuts, total = distribute(A0, A0, rank, world, device)
        else:
            A_blk, Bx = A0, A0
            total = None
        rep = spgemm_magnus_waves(A_blk, Bx, sys=sysp, consumer=lambda lo, hi, C: None)
        return rep, total

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    times, rep, total = [], None, None
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep, total = step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    ms = sum(times) / len(times)
    nnz = rep.nnz_c
    inter_loc = rep.inter_products
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        t = torch.tensor([nnz, inter_loc, rep.waves], dtype=torch.int64, device=device)
        dist.all_reduce(t)
        nnz, inter_loc, waves = (int(x) for x in t.tolist())
    else:
        waves = rep.waves
    total_inter = inter_loc
    if rank == 0:
        A = A0
        peak, peak_kind = hbm_peak()
        comp = compulsory_bytes(A.n_rows, A.col.numel(), total_inter, nnz, 8, 8, 8, A.n_rows)
        line = {
            "metric": "SpGEMM GFLOP/s (2 x mults)", "value": round(2.0 * total_inter / (ms * 1e-3) / 1e9, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, generated on device; BASELINE.json config shapes and value distributions)",
            "config": workload_config(5, A, A, total_inter, world),
            "nnz_c": nnz, "waves": waves,
            "mode": "row waves into a reused C buffer per rank (C ~ 15 TB cannot be held); each wave's C is "
                    "materialised in HBM and discarded",
            "roofline_step": {"bound": "hbm", "compulsory_bytes": comp,
                              "achieved": round(comp / (ms * 1e-3) / 1e9, 1), "peak": peak * world,
                              "frac": round(comp / (ms * 1e-3) / 1e9 / (peak * world), 4), "unit": "GB/s"},
            "roofline": None, "e2e": {"unavailable": "C (~15 TB) cannot be read back to the host"},
            "cpu_baseline": None, "clocks": clocks, "gen_s": round(t_gen, 2),
            "timing": "CUDA events, max over ranks; N>1 steps include the B broadcast and the A-block exchange",
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class HostBuffer:
    """Page-locked host array without the caching host allocator's power-of-two rounding
    (C of cfg3 is ~117 GB): numpy memory registered with cudaHostRegister."""

    def __init__(self, n, dtype):
        import torch
        self.arr = np.empty(max(int(n), 1), dtype=dtype)
        self.rt = torch.cuda.cudart()
        err = self.rt.cudaHostRegister(self.arr.ctypes.data, self.arr.nbytes, 0)
        self.registered = int(err) == 0
        self.t = torch.from_numpy(self.arr)

    def close(self):
        if self.registered:
            self.rt.cudaHostUnregister(self.arr.ctypes.data)
            self.registered = False


def run_e2e(A, B, sysp, steps, total_inter):
    """Same metric through the public API with HOST buffers: page-locked host inputs are copied
    in, spgemm runs, and C (row_ptr, col, val) is read back into page-locked host arrays --
    all inside the timed region (buffers are allocated and registered outside it)."""
    import torch

    from paper_2501_07056_b200 import CsrMatrix, MagnusPlan

    def pinned_copy(t):
        h = HostBuffer(t.numel(), {torch.int32: np.int32, torch.int64: np.int64, torch.float64: np.float64}[t.dtype])
        h.t.copy_(t)
        return h

    bufs = [pinned_copy(t) for t in (A.row_ptr, A.col, A.val)]
    Ah = CsrMatrix(A.n_rows, A.n_cols, bufs[0].t, bufs[1].t, bufs[2].t)
    Bh = Ah
    if B is not A:
        bufs += [pinned_copy(t) for t in (B.row_ptr, B.col, B.val)]
        Bh = CsrMatrix(B.n_rows, B.n_cols, bufs[3].t, bufs[4].t, bufs[5].t)
    h2d = sum(b.arr.nbytes for b in bufs)
    # size the output once (symbolic only), outside the timed region
    plan = MagnusPlan(A, B, sys=sysp)
    rp = plan.symbolic()
    nnz = int(rp[-1])
    plan.close()
    del rp
    out_rp, out_col, out_val = HostBuffer(A.n_rows + 1, np.int64), HostBuffer(nnz, np.int32), HostBuffer(nnz, np.float64)
    times = []
    for it in range(steps + 1):                       # (the first, untimed, warms the memory pool)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = MagnusPlan(Ah, Bh, sys=sysp)           # H2D of the host inputs inside
        rp = plan.symbolic()
        out_rp.t.copy_(rp, non_blocking=True)
        # C's col / val are read back while later heavy-row batches compute
        C, _ = plan.numeric(rp, host_out=(out_col.t, out_val.t))
        torch.cuda.synchronize()
        if it:
            times.append(time.perf_counter() - t0)
        plan.close()
        del C, rp
    d2h = (A.n_rows + 1) * 8 + nnz * 12
    for b in bufs + [out_rp, out_col, out_val]:
        b.close()
    t = sum(times) / len(times)
    return {"value": round(2.0 * total_inter / t / 1e9, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(t * 1e3, 2), "steps": len(times)}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm's CPU restatement (oracle/, C + OpenMP) with all
    host threads and the reference's own host SystemParams (detect_system_params), on bounded
    row samples of the same workload (rank 0 only).  Inputs are generated on the host (numpy):
    nothing of the device library is loaded in this arm."""
    if rank != 0:
        return
    from paper_2501_07056_b200 import generate
    t = time.perf_counter()
    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable": "cfg5 host generation exceeds the bench budget"}))
        return
    A, B = generate.make_config_cpu(args.config)
    t_gen = time.perf_counter() - t
    rp = np.asarray(A.row_ptr, np.int64)
    deg = np.diff(np.asarray(B.row_ptr, np.int64))
    per = deg[np.asarray(A.col).astype(np.int64)]
    cs = np.r_[0, np.cumsum(per)]
    inter = cs[rp[1:]] - cs[rp[:-1]]
    sysp = host_system_params()
    seconds = max(5.0, min(args.cpu_seconds, 30.0))
    vals = []
    for s in range(max(1, args.warmup // 3) + args.steps):
        r = cpu_baseline(A, B, sysp, seconds / max(args.steps, 1) * 2, inter, seed=s)
        if s >= max(1, args.warmup // 3):
            vals.append(r)
    v = float(np.mean([r["value"] for r in vals]))
    line = {"impl": "reference", "metric": "SpGEMM GFLOP/s (2 x mults)", "value": round(v, 5), "unit": "GFLOP/s",
            "n_gpus": world, "steps": len(vals), "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, numpy on the host)",
            "config": workload_config(args.config, A, B, int(inter.sum()), world),
            "cpu_baseline": {"value": round(v, 5), "unit": "GFLOP/s", "cores": vals[0]["cores"], "kind": "port",
                             "sample": vals[-1]["sample"],
                             "system_params": {"cache_line_bytes": sysp.cache_line_bytes, "l2_bytes": sysp.l2_bytes}},
            "e2e": {"value": round(v, 5), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gen_s": round(t_gen, 1), "wall_s": round(time.perf_counter() - t, 1)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
