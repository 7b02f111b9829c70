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


def scatter_row_blocks(A, cuts, rank: int, world: int, device, group=None):
    """Rank r receives rows [cuts[r], cuts[r+1]) of A (rank 0 holds A) as a rebased CSR block:
    point-to-point sends from rank 0, so no rank receives more of A than its own block."""
    import torch
    import torch.distributed as dist

    if rank == 0:
        for r in range(1, world):
            blk = row_block(A, cuts[r], cuts[r + 1])
            meta = torch.tensor([blk.n_rows, blk.n_cols, int(blk.col.numel()), blk.row_ptr.element_size()],
                                dtype=torch.int64, device=device)
            dist.send(meta, r, group=group)
            for t in (blk.row_ptr, blk.col, blk.val):
                dist.send(t.contiguous(), r, group=group)
        return row_block(A, cuts[0], cuts[1])
    meta = torch.zeros(4, dtype=torch.int64, device=device)
    dist.recv(meta, 0, group=group)
    n, m, nnz, rpb = (int(x) for x in meta.tolist())
    blk = CsrMatrix(n, m, torch.empty(n + 1, dtype=torch.int64 if rpb == 8 else torch.int32, device=device),
                    torch.empty(nnz, dtype=torch.int32, device=device), torch.empty(nnz, dtype=torch.float64, device=device))
    for t in (blk.row_ptr, blk.col, blk.val):
        dist.recv(t, 0, group=group)
    return blk


def distribute(A, B, rank: int, world: int, device, group=None, inter_fn=None):
    """The exchange step of SURVEY.md §8(e): B replicated from rank 0 (one NCCL broadcast over
    NVLink), the flop-balanced cuts computed on rank 0 from its per-row intermediate sizes and
    broadcast, and each rank's block of A (a slice of the replicated B when C = A·A, else a
    point-to-point send from rank 0).  Returns (A_block, B, cuts, total_products)."""
    import torch
    import torch.distributed as dist

    inter_fn = inter_fn or _default_inter
    same = torch.tensor([1 if (rank == 0 and A is B) else 0], dtype=torch.int64, device=device)
    dist.broadcast(same, 0, group=group)
    B = broadcast_csr(B if rank == 0 else None, 0, device, group)
    if rank == 0:
        cuts, total = flop_cuts(inter_fn(A if not int(same) else B, B), world)
        ct = torch.tensor(cuts + [total], dtype=torch.int64, device=device)
    else:
        ct = torch.zeros(world + 2, dtype=torch.int64, device=device)
    dist.broadcast(ct, 0, group=group)
    vals = [int(x) for x in ct.tolist()]
    cuts, total = vals[:world + 1], vals[world + 1]
    if int(same):
        A_blk = row_block(B, cuts[rank], cuts[rank + 1])
    else:
        A_blk = scatter_row_blocks(A, cuts, rank, world, device, group)
    return A_blk, B, cuts, total


def _default_local(A, B, sys, thresholds, force_fine_only):
    from .magnus import spgemm_magnus
    res = spgemm_magnus(A, B, sys=sys, thresholds=thresholds, force_fine_only=force_fine_only)
    return res.C, res.counters


def _default_inter(A, B):
    from .magnus import row_intermediate_stats
    return row_intermediate_stats(A, B).inter_size


def rebase(C, rank: int, world: int, device, group=None):
    """all_gather of one int64 per rank: this block's offset in C's global nnz, and the total."""
    import torch
    import torch.distributed as dist

    nnz_local = torch.tensor([int(C.row_ptr[-1])], dtype=torch.int64, device=device)
    all_nnz = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(all_nnz, nnz_local, group=group)
    per = [int(x) for x in all_nnz]
    return sum(per[:rank]), sum(per)


def spgemm_magnus_distributed(A, B, sys=None, thresholds=None, force_fine_only=False, group=None, device=None,
                              local_fn=None, inter_fn=None) -> RowBlock:
    """C = A.B over the ranks of `group` (torch.distributed must be initialised).

    A and B (CsrMatrix of torch tensors) need only exist on rank 0 (pass None
    elsewhere); B is broadcast, each rank receives only its flop-balanced block
    of A.  Returns this rank's RowBlock.  `local_fn(A_block, B, sys, thresholds,
    force_fine_only) -> (C_block, counters)` and `inter_fn(A, B) -> per-row
    intermediate sizes` default to the CUDA path.
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    local_fn = local_fn or _default_local
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else \
            torch.device("cpu")
    A_blk, B, cuts, _ = distribute(A, B, rank, world, device, group, inter_fn)
    lo, hi = cuts[rank], cuts[rank + 1]
    C, counters = local_fn(A_blk, B, sys, thresholds, force_fine_only)
    off, total = rebase(C, rank, world, device, group)
    rp = C.row_ptr
    rp = rp + off if not isinstance(rp, np.ndarray) else rp + np.int64(off)
    Cg = CsrMatrix(C.n_rows, C.n_cols, rp, C.col, C.val, True)
    return RowBlock(lo, hi, off, Cg, total, counters)
