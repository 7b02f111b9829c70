"""Locality-generation building blocks on the device -- reference bench.py:1-196.

Same workload and API as the reference: a synthetic intermediate-product
stream (indices uniform in [0, length), values in [0, 1)) and each stage of
single-level locality generation timed in isolation over it:

    histogram      chunk occupancy counts (index >> shift)        k_mb_hist
    prefix_sum     chunk offsets from the histogram               k_scan_* (magnus_mb_scan)
    reorder        stable scatter into chunk order, local index    k_mb_tile_hist + scan + k_mb_scatter
    dense_accum    per-chunk dense accumulation (sequential)       k_mb_dense
    sort_accum     per-chunk sort-merge accumulation               stable sort + ESC compress kernels
    stream         contiguous copy of both arrays (peak baseline)  k_mb_stream

``total`` = histogram + prefix_sum + reorder + dense_accum.  Every timed run
checks its stage checksums (counts sum to the stream size, the reorder is a
permutation with intra-chunk stability, distinct counts agree between the two
accumulators and with the stream, value sums are conserved), so timing never
bypasses verification.  Times are CUDA-event times on the launching stream.
Differences from the reference: the stream lives in HBM (u32 indices); the
sort accumulator's sort step is the library's own stable LSD radix sort
(csrc/radix_sort.cuh, `magnus_sort_pairs`); chunk counts are bounded by
shared memory (reorder <= 4096 chunks, dense chunk length <= 16384).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _lib
from .errors import InputError
from .planner import ceil_pow2, exact_log2


@dataclass(frozen=True)
class StreamSpec:
    """reference bench.py:31-42"""

    size: int
    length: int   # exclusive upper bound on index values
    seed: int = 0

    def __post_init__(self):
        if self.length < 1:
            raise InputError("stream length must be >= 1")
        if self.size < 0:
            raise InputError("stream size must be non-negative")


@dataclass
class BenchRecord:
    """reference bench.py:45-51"""

    name: str
    params: dict = field(default_factory=dict)
    seconds: float = 0.0
    rate: float = 0.0   # elements per second
    rep: int = 0


def _torch():
    import torch
    return torch


def make_stream(spec: StreamSpec, device=None):
    """(idx int32 holding u32 indices < length, vals f64 in [0, 1)) on the device, seeded."""
    torch = _torch()
    device = device or torch.device("cuda", torch.cuda.current_device())
    if spec.length > 1 << 32:
        raise InputError("device streams hold 32-bit indices (length <= 2^32)")
    g = torch.Generator(device=device)
    g.manual_seed(int(spec.seed))
    idx = torch.randint(0, spec.length, (spec.size,), generator=g, device=device, dtype=torch.int64)
    vals = torch.rand(spec.size, generator=g, device=device, dtype=torch.float64)
    return idx.to(torch.int32), vals


def _sp(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _timed(fn):
    torch = _torch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3


def measure_bandwidth(n_bytes: int = 1 << 28, reps: int = 3):
    """Best-of-reps device copy rate of an index/value array pair (reference bench.py:57-85).
    Returns (bytes_per_second, bytes_moved_per_rep); one rep reads and writes both arrays."""
    torch = _torch()
    if reps < 1:
        raise InputError("reps must be >= 1")
    n = max(1, n_bytes // 16)
    src = torch.ones(2 * n, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    L = _lib.lib()
    moved = 2 * src.numel() * 8
    best = float("inf")
    for _ in range(reps + 1):
        best = min(best, _timed(lambda: _lib.check(L.magnus_mb_stream(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                                                      src.numel() * 8, _sp(torch)))))
    if not torch.equal(src[-1:], dst[-1:]):
        raise RuntimeError("stream copy failed")
    return moved / best, moved


def microbench_building_blocks(spec: StreamSpec, n_chunks: int, reps: int = 1, rng_check: bool = True):
    """Time each building block over one generated stream; returns BenchRecords (reference
    bench.py:88-196).  Raises if any stage's checksum fails."""
    torch = _torch()
    if n_chunks < 1 or n_chunks & (n_chunks - 1):
        raise InputError("n_chunks must be a power of two")
    if n_chunks > spec.length:
        raise InputError("n_chunks must not exceed the stream length")
    if reps < 1:
        raise InputError("reps must be >= 1")
    span = ceil_pow2(spec.length)
    chunk_len = span // n_chunks
    shift = exact_log2(chunk_len)
    if n_chunks > 4096 or chunk_len > 1 << 14:
        raise InputError("device building blocks: n_chunks <= 4096 and chunk length <= 16384")
    L = _lib.lib()
    idx, vals = make_stream(spec)
    n = spec.size
    dev = idx.device
    params = {"size": spec.size, "length": spec.length, "n_chunks": n_chunks, "seed": spec.seed}
    counts = torch.empty(n_chunks, dtype=torch.int64, device=dev)
    offsets = torch.empty(n_chunks + 1, dtype=torch.int64, device=dev)
    col_out = torch.empty(n, dtype=torch.int32, device=dev)
    val_out = torch.empty(n, dtype=torch.float64, device=dev)
    scratch = torch.empty(int(L.magnus_mb_reorder_scratch_bytes(n, n_chunks)) // 8 + 1, dtype=torch.int64, device=dev)
    d_col = torch.empty(n, dtype=torch.int32, device=dev)
    d_val = torch.empty(n, dtype=torch.float64, device=dev)
    distinct = torch.empty(n_chunks, dtype=torch.int64, device=dev)
    s_col = torch.empty(n, dtype=torch.int32, device=dev)
    s_val = torch.empty(n, dtype=torch.float64, device=dev)
    run = torch.empty(n + 1, dtype=torch.int64, device=dev)
    copy_i = torch.empty(n, dtype=torch.int32, device=dev)
    copy_v = torch.empty(n, dtype=torch.float64, device=dev)
    ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    sp = _sp(torch)
    expected_distinct = int(torch.unique(idx).numel())
    total_v = float(vals.sum())
    scan_scratch = torch.empty(int(L.magnus_mb_scan_scratch_bytes(n_chunks)) // 8 + 1, dtype=torch.int64, device=dev)

    def scan():
        _lib.check(L.magnus_mb_scan(ptr(counts), n_chunks, ptr(offsets), ptr(scan_scratch), sp))

    records = []
    for rep in range(reps):
        t_hist = _timed(lambda: _lib.check(L.magnus_mb_histogram(ptr(idx), n, shift, n_chunks, ptr(counts), sp)))
        if int(counts.sum()) != n:
            raise RuntimeError("histogram checksum failed: counts do not sum to the stream size")
        t_prefix = _timed(scan)
        if int(offsets[-1]) != n:
            raise RuntimeError("prefix-sum checksum failed")
        t_reorder = _timed(lambda: _lib.check(L.magnus_mb_reorder(ptr(idx), ptr(vals), n, shift, n_chunks, ptr(scratch),
                                                                  scratch.numel() * 8, ptr(col_out), ptr(val_out), sp)))
        if rng_check and n:
            chunk_of = torch.repeat_interleave(torch.arange(n_chunks, device=dev), counts)
            rebuilt = col_out.to(torch.int64) + chunk_of * chunk_len
            if not torch.equal(torch.sort(rebuilt).values, torch.sort(idx.to(torch.int64)).values):
                raise RuntimeError("reorder checksum failed: output is not a permutation of the input")
            # stability: inside a chunk, equal local indices keep stream order (values identify positions)
            order = torch.argsort(idx.to(torch.int64), stable=True)
            if not torch.equal(vals[order], val_out[torch.argsort(rebuilt, stable=True)]):
                raise RuntimeError("reorder checksum failed: intra-chunk order not stable")
        t_dense = _timed(lambda: _lib.check(L.magnus_mb_dense(ptr(col_out), ptr(val_out), ptr(offsets), n_chunks, chunk_len,
                                                              ptr(d_col), ptr(d_val), ptr(distinct), sp)))
        distinct_dense = int(distinct.sum())

        def sort_accum():
            keys = col_out.to(torch.int64) + torch.repeat_interleave(torch.arange(n_chunks, device=dev), counts) * chunk_len
            sk, perm = _lib.sort_pairs(keys, max(1, int(span - 1).bit_length()))
            runs = C.c_int64(0)
            _lib.check(L.magnus_esc_compress(ptr(sk), ptr(perm), ptr(val_out), n, 0, ptr(s_col), ptr(s_val), ptr(run),
                                             C.byref(runs), sp))
            return int(runs.value)

        holder = {}
        t_sort = _timed(lambda: holder.setdefault("runs", sort_accum()))
        distinct_sort = holder["runs"]
        if distinct_dense != expected_distinct or distinct_sort != expected_distinct:
            raise RuntimeError("accumulation checksum failed: distinct-column counts disagree")
        starts = offsets[:-1]
        mask_idx = torch.repeat_interleave(starts, distinct) + (
            torch.arange(distinct_dense, device=dev) - torch.repeat_interleave(torch.cumsum(distinct, 0) - distinct, distinct))
        vsum_dense = float(d_val[mask_idx].sum())
        vsum_sort = float(s_val[:distinct_sort].sum())
        for vs in (vsum_dense, vsum_sort):
            if abs(vs - total_v) > 1e-9 * max(1.0, abs(total_v)):
                raise RuntimeError("accumulation checksum failed: value sums not conserved")
        t_stream = _timed(lambda: (_lib.check(L.magnus_mb_stream(ptr(idx), ptr(copy_i), (n * 4) // 16 * 16, sp)),
                                   _lib.check(L.magnus_mb_stream(ptr(vals), ptr(copy_v), (n * 8) // 16 * 16, sp))))
        if n >= 4 and (int(copy_i[(n // 4) * 4 - 1]) != int(idx[(n // 4) * 4 - 1]) or
                       float(copy_v[(n // 2) * 2 - 1]) != float(vals[(n // 2) * 2 - 1])):
            raise RuntimeError("stream checksum failed")
        for name, t in (("histogram", t_hist), ("prefix_sum", t_prefix), ("reorder", t_reorder), ("dense_accum", t_dense),
                        ("sort_accum", t_sort), ("stream", t_stream),
                        ("total", t_hist + t_prefix + t_reorder + t_dense)):
            records.append(BenchRecord(name, dict(params), t, spec.size / t if t > 0 else 0.0, rep))
    return records
