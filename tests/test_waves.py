"""Row waves (waves.py): C = A·B in bounded row blocks for products whose C does not fit
(BASELINE cfg5).  Host logic on CPU; on the GPU the concatenated waves equal the one-shot
product bit for bit, with the B-derived state reused across waves."""

import numpy as np
import pytest

from paper_2501_07056_b200.waves import wave_cuts


def test_wave_cuts_bounds():
    inter = np.array([5, 0, 100, 3, 3, 3, 50, 50, 0, 1])
    cuts = wave_cuts(inter, 60, 10)
    assert cuts == [0, 2, 3, 6, 7, 8, 10]
    rng = np.random.default_rng(3)
    x = rng.integers(0, 5000, 4000)
    for cap in (1, 100, 7000, 10 ** 9):
        c = wave_cuts(x, 3000, cap)
        assert c[0] == 0 and c[-1] == x.size and all(a < b for a, b in zip(c, c[1:]))
        b = np.minimum(x, 3000)
        for lo, hi in zip(c[:-1], c[1:]):
            assert hi - lo == 1 or b[lo:hi].sum() <= cap


@pytest.mark.gpu
@pytest.mark.parametrize("buffer_entries", [30000, 400000])
def test_waves_equal_one_shot(buffer_entries):
    import torch

    from paper_2501_07056_b200 import CsrMatrix, SystemParams, generate, spgemm_magnus
    from paper_2501_07056_b200.waves import spgemm_magnus_waves, wave_checksum
    B200 = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 31)
    A = generate.rmat_device(14, 16, seed=5)
    full = spgemm_magnus(A, A, sys=B200).C
    parts = []

    def keep(lo, hi, Cb):
        parts.append((lo, hi, Cb.row_ptr.clone(), Cb.col.clone(), Cb.val.clone()))

    rep = spgemm_magnus_waves(A, A, sys=B200, buffer_bytes=buffer_entries * 12, consumer=keep)
    assert rep.waves == len(parts) and rep.waves > 1
    assert rep.nnz_c == int(full.row_ptr[-1])
    assert parts[0][0] == 0 and parts[-1][1] == A.n_rows
    cols = torch.cat([p[3] for p in parts])
    vals = torch.cat([p[4] for p in parts])
    assert torch.equal(cols, full.col) and torch.equal(vals.view(torch.int64), full.val.view(torch.int64))
    for lo, hi, rp, _, _ in parts:
        assert torch.equal(rp, full.row_ptr[lo:hi + 1] - full.row_ptr[lo])
    rep2 = spgemm_magnus_waves(A, A, sys=B200, buffer_bytes=buffer_entries * 12)
    assert len(rep2.checksums) == rep.waves
    blk = CsrMatrix(parts[0][1] - parts[0][0], A.n_cols, parts[0][2], parts[0][3], parts[0][4])
    assert rep2.checksums[0] == wave_checksum(blk)
