"""Row waves: C = A·B when C does not fit in HBM (BASELINE cfg5: ~1.3e12 nonzeros, ~15 TB).

Rows of C are independent, so A is cut into contiguous row blocks
("waves") whose C fits a bounded device buffer; each wave runs the same single-GPU
path (`MagnusPlan`: setup, symbolic, numeric) on one context, so the B-derived
device state (validation, skip list, B window index) is built once for all waves;
each wave's C block is handed to a consumer (checksum, host copy, a file) and the
buffer is reused.  This realises the reference's memory-budgeted batching
(`build_coarse_batches`, magnus.py:277-314, budget `memory_budget_bytes`
planner.py:51) at the level of the whole C.

Wave cuts use an upper bound of each row's nnz(C): min(inter, n_cols) (intermediate
products, or the full row); a wave holds rows whose bounds sum to at most the
buffer's entries (a single row above it gets a wave of its own, sized exactly by
its symbolic pass).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .matrix import CsrMatrix


def wave_cuts(inter, n_cols: int, cap_entries: int):
    """Contiguous row cuts [c0=0, c1, ..., n]: sum of min(inter, n_cols) per wave <= cap_entries
    (a row whose bound alone exceeds it forms its own wave).  inter: per-row products (numpy or
    torch); host arithmetic on an int64 prefix."""
    x = np.minimum(np.asarray(inter.cpu() if hasattr(inter, "cpu") else inter, dtype=np.int64), max(int(n_cols), 1))
    cs = np.concatenate(([0], np.cumsum(x)))
    n = x.size
    cuts = [0]
    while cuts[-1] < n:
        lo = cuts[-1]
        hi = int(np.searchsorted(cs, cs[lo] + cap_entries, side="right")) - 1
        cuts.append(max(hi, lo + 1))
    return cuts


@dataclass
class WaveReport:
    waves: int
    rows: int
    nnz_c: int
    inter_products: int
    checksums: list = field(default_factory=list)


def row_block_view(A: CsrMatrix, lo: int, hi: int) -> CsrMatrix:
    rp = A.row_ptr
    a0, a1 = int(rp[lo]), int(rp[hi])
    return CsrMatrix(hi - lo, A.n_cols, rp[lo:hi + 1] - a0, A.col[a0:a1], A.val[a0:a1], A.canonical)


def wave_checksum(C) -> tuple:
    """Order-sensitive checksum of a C block (device tensors): sums of the value bits and of the
    columns, each weighted by position mod a prime -- any changed, moved or missing entry shows."""
    import torch
    n = int(C.col.numel())
    if n == 0:
        return (0, 0)
    pos = torch.arange(n, device=C.col.device, dtype=torch.int64) % 1000003 + 1
    v = (C.val.view(torch.int64) % 1000003) * pos
    c = C.col.to(torch.int64) * pos
    return (int(v.sum() % (1 << 61)), int(c.sum() % (1 << 61)))


def spgemm_magnus_waves(A, B, sys=None, thresholds=None, force_fine_only=False, buffer_bytes=None, consumer=None,
                        inter=None) -> WaveReport:
    """C = A·B in row waves on the current device; `consumer(lo, hi, C_block)` receives each wave's
    rows [lo, hi) (device CsrMatrix, valid until the consumer returns; default: checksum)."""
    import torch

    from .magnus import MagnusPlan, row_intermediate_stats

    dev = torch.device("cuda", torch.cuda.current_device())
    if inter is None:
        inter = row_intermediate_stats(A, B).inter_size
    if buffer_bytes is None:
        free, _ = torch.cuda.mem_get_info(dev)
        buffer_bytes = int(free * 0.35)
    cap = max(1, int(buffer_bytes) // 12)
    cuts = wave_cuts(inter, B.n_cols, cap)
    col_buf = torch.empty(cap, dtype=torch.int32, device=dev)
    val_buf = torch.empty(cap, dtype=torch.float64, device=dev)
    rep = WaveReport(0, A.n_rows, 0, int(inter.sum()))
    plan = None
    try:
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            blk = row_block_view(A, lo, hi)
            if plan is None:
                plan = MagnusPlan(blk, B, sys, thresholds, force_fine_only)
            else:
                plan.reset(blk)
            rp = plan.symbolic()
            nnz = plan.nnz
            if nnz <= cap:
                out = (col_buf[:nnz], val_buf[:nnz])
            else:   # one row above the bound's budget: exact size from its symbolic pass
                out = (torch.empty(nnz, dtype=torch.int32, device=dev), torch.empty(nnz, dtype=torch.float64, device=dev))
            Cb, _ = plan.numeric(rp, out=out)
            if consumer is None:
                rep.checksums.append(wave_checksum(Cb))
            else:
                consumer(lo, hi, Cb)
            rep.waves += 1
            rep.nnz_c += nnz
            del out, Cb
    finally:
        if plan is not None:
            plan.close()
    return rep
