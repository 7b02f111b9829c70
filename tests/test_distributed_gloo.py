"""Multi-rank host logic on CPU (gloo, world size 2): flop-balanced row split,
broadcast of A/B from rank 0, per-rank products, row_ptr rebasing.  The local
product is the CPU oracle (test-only injection); concatenating the rank blocks
must give exactly the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_07056_b200 import CsrMatrix, SystemParams, generate
from paper_2501_07056_b200.parallel import flop_cuts, spgemm_magnus_distributed

SYS = SystemParams(cache_line_bytes=64, l2_bytes=4096)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_torch(m):
    return CsrMatrix(m.n_rows, m.n_cols, torch.from_numpy(np.asarray(m.row_ptr, np.int64)),
                     torch.from_numpy(np.asarray(m.col).astype(np.int32)), torch.from_numpy(np.asarray(m.val)))


def _local_oracle(Ab, B, sys, thresholds, ffo):
    from oracle import oracle
    An = CsrMatrix(Ab.n_rows, Ab.n_cols, Ab.row_ptr.numpy(), Ab.col.numpy(), Ab.val.numpy())
    Bn = CsrMatrix(B.n_rows, B.n_cols, B.row_ptr.numpy(), B.col.numpy(), B.val.numpy())
    r = oracle.spgemm(An, Bn, sys, thresholds, ffo, threads=1)
    return CsrMatrix(Ab.n_rows, B.n_cols, torch.from_numpy(r.row_ptr), torch.from_numpy(r.col.view(np.int32)),
                     torch.from_numpy(r.val)), r.counters


def _inter_np(A, B):
    deg = np.diff(B.row_ptr.numpy())
    per = deg[A.col.numpy().astype(np.int64)]
    cs = np.r_[0, np.cumsum(per)]
    rp = A.row_ptr.numpy()
    return torch.from_numpy(cs[rp[1:]] - cs[rp[:-1]])


def _worker(rank, world, port, outdir, ab=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if ab:
        A = _to_torch(generate.uniform_rows(3000, 4096, 6, seed=3)) if rank == 0 else None
        B = _to_torch(generate.rmat(12, 8, seed=5)) if rank == 0 else None
    else:
        A = B = _to_torch(generate.rmat(11, 8, seed=17)) if rank == 0 else None
    blk = spgemm_magnus_distributed(A, B, sys=SYS, local_fn=_local_oracle, inter_fn=_inter_np)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), lo=blk.row_lo, hi=blk.row_hi, rp=blk.C.row_ptr.numpy(),
             col=blk.C.col.numpy(), val=blk.C.val.numpy(), total=blk.nnz_total)
    dist.destroy_process_group()


def test_flop_cuts_balance():
    inter = np.array([5, 0, 100, 3, 3, 3, 50, 50, 0, 1], dtype=np.int64)
    cuts, total = flop_cuts(inter, 3)
    assert cuts[0] == 0 and cuts[-1] == inter.size and total == inter.sum()
    assert all(a <= b for a, b in zip(cuts, cuts[1:]))


@pytest.mark.parametrize("ab", [False, True])
def test_two_rank_gloo_equals_single(tmp_path, ab):
    """C = A·A (A block sliced from the replicated B) and C = A·B (A blocks sent point-to-point)."""
    from oracle import oracle
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), ab), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    if ab:
        A, B = generate.uniform_rows(3000, 4096, 6, seed=3), generate.rmat(12, 8, seed=5)
    else:
        A = B = generate.rmat(11, 8, seed=17)
    ref = oracle.spgemm(A, B, SYS)
    assert parts[0]["lo"] == 0 and parts[-1]["hi"] == A.n_rows and parts[0]["hi"] == parts[1]["lo"]
    rp = np.concatenate([parts[0]["rp"][:-1], parts[1]["rp"]])
    np.testing.assert_array_equal(rp, ref.row_ptr)
    np.testing.assert_array_equal(np.concatenate([p["col"] for p in parts]).view(np.uint32), ref.col)
    np.testing.assert_array_equal(np.concatenate([p["val"] for p in parts]).view(np.uint64), ref.val.view(np.uint64))
    assert int(parts[0]["total"]) == int(ref.row_ptr[-1])
