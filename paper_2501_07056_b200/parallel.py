"""Multi-GPU SpGEMM: flop-balanced row blocks of A, B replicated, C row blocks
concatenated.

One process per GPU.  Rows of C are independent, so the only exchange is the
replication of B (one broadcast from rank 0 over NCCL/NVLink) plus an
all-gather of one int64 per rank to rebase C's row_ptr; there is no collective
inside the hot loop.  Every rank's rows are computed by exactly the same
single-GPU path, so C is bit-identical for any number of ranks.

The host logic (split, broadcast, rebasing) is backend-agnostic: the tests run
it with gloo on CPU ranks and an injected local product.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .matrix import CsrMatrix


@dataclass
class RowBlock:
    """This rank's block of C: global rows [row_lo, row_hi), row_ptr rebased to C's global nnz offsets."""

    row_lo: int
    row_hi: int
    nnz_offset: int
    C: CsrMatrix          # local rows; C.row_ptr is global (starts at nnz_offset)
    nnz_total: int
    counters: dict


def flop_cuts(inter, world: int):
    """Contiguous row cuts with ~equal sum(inter) per part; inter = per-row intermediate sizes."""
    import torch
    t = inter if isinstance(inter, torch.Tensor) else torch.as_tensor(np.asarray(inter, dtype=np.int64))
    cs = torch.cumsum(t.to(torch.int64), 0)
    total = int(cs[-1]) if cs.numel() else 0
    cuts = [0]
    for r in range(1, world):
        target = torch.tensor(total * r // world, dtype=torch.int64, device=cs.device)
        cuts.append(max(cuts[-1], int(torch.searchsorted(cs, target))))
    cuts.append(int(t.numel()))
    return cuts, total


def row_block(A: CsrMatrix, lo: int, hi: int) -> CsrMatrix:
    """Rows [lo, hi) of A as a CSR view with row_ptr rebased to 0."""
    rp = A.row_ptr
    a0, a1 = int(rp[lo]), int(rp[hi])
    return CsrMatrix(hi - lo, A.n_cols, rp[lo:hi + 1] - a0, A.col[a0:a1], A.val[a0:a1], A.canonical)


def broadcast_csr(M, src: int, device, group=None):
    """Replicate a CSR matrix (torch tensors) from rank `src` to every rank of the group."""
    import torch
    import torch.distributed as dist

    if M is not None:
        meta = torch.tensor([M.n_rows, M.n_cols, int(M.col.numel()), M.row_ptr.element_size()], dtype=torch.int64,
                            device=device)
    else:
        meta = torch.zeros(4, dtype=torch.int64, device=device)
    dist.broadcast(meta, src, group=group)
    n, m, nnz, rpb = (int(x) for x in meta.tolist())
    if M is None:
        M = CsrMatrix(n, m, torch.empty(n + 1, dtype=torch.int64 if rpb == 8 else torch.int32, device=device),
                      torch.empty(nnz, dtype=torch.int32, device=device),
                      torch.empty(nnz, dtype=torch.float64, device=device))
    for t in (M.row_ptr, M.col, M.val):
        dist.broadcast(t, src, group=group)
    return M


def _default_local(A, B, sys, thresholds, force_fine_only):
    from .magnus import spgemm_magnus
    res = spgemm_magnus(A, B, sys=sys, thresholds=thresholds, force_fine_only=force_fine_only)
    return res.C, res.counters


def _default_inter(A, B):
    from .magnus import row_intermediate_stats
    return row_intermediate_stats(A, B).inter_size


def spgemm_magnus_distributed(A, B, sys=None, thresholds=None, force_fine_only=False, group=None, device=None,
                              local_fn=None, inter_fn=None) -> RowBlock:
    """C = A.B over the ranks of `group` (torch.distributed must be initialised).

    A and B (CsrMatrix of torch tensors) need only exist on rank 0 (pass None
    elsewhere); B is broadcast, A too (each rank then takes its block).  Returns
    this rank's RowBlock.  `local_fn(A_block, B, sys, thresholds, force_fine_only)
    -> (C_block, counters)` and `inter_fn(A, B) -> per-row intermediate sizes`
    default to the CUDA path.
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    local_fn = local_fn or _default_local
    inter_fn = inter_fn or _default_inter
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else \
            torch.device("cpu")
    same = torch.tensor([1 if (rank == 0 and A is B) else 0], dtype=torch.int64, device=device)
    dist.broadcast(same, 0, group=group)
    B = broadcast_csr(B if rank == 0 else None, 0, device, group)
    A = B if int(same) else broadcast_csr(A if rank == 0 else None, 0, device, group)
    inter = inter_fn(A, B)
    cuts, _ = flop_cuts(inter, world)
    lo, hi = cuts[rank], cuts[rank + 1]
    C, counters = local_fn(row_block(A, lo, hi), B, sys, thresholds, force_fine_only)
    nnz_local = torch.tensor([int(C.row_ptr[-1])], dtype=torch.int64, device=device)
    all_nnz = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(all_nnz, nnz_local, group=group)
    per = [int(x) for x in all_nnz]
    off = sum(per[:rank])
    rp = C.row_ptr
    rp = rp + off if not isinstance(rp, np.ndarray) else rp + np.int64(off)
    Cg = CsrMatrix(C.n_rows, C.n_cols, rp, C.col, C.val, True)
    return RowBlock(lo, hi, off, Cg, sum(per), counters)
