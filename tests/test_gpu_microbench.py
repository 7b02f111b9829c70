"""Building-block kernels (csrc/microbench.cuh; reference bench.py:88-196) against
numpy restatements: histogram counts, stable reorder (stable_scatter_positions
matrix.py:187-204), per-chunk dense accumulation bit-exact with sequential sums
(np.bincount), sort accumulation, and the full microbenchmark with its checksums."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2501_07056_b200 import _lib, microbench  # noqa: E402
from paper_2501_07056_b200.errors import InputError  # noqa: E402

pytestmark = pytest.mark.gpu


def p(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("size,length,nch", [(100_000, 4096, 64), (1 << 20, 1 << 16, 4096), (3333, 1 << 14, 1),
                                             (1 << 18, 1 << 20, 1024)])
def test_stages_match_numpy(size, length, nch):
    L = _lib.lib()
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    idx, vals = microbench.make_stream(microbench.StreamSpec(size, length, seed=7))
    chunk_len = (1 << (length - 1).bit_length()) // nch
    shift = chunk_len.bit_length() - 1
    hi, hv = idx.cpu().numpy().astype(np.int64), vals.cpu().numpy()
    counts = torch.empty(nch, dtype=torch.int64, device="cuda")
    _lib.check(L.magnus_mb_histogram(p(idx), size, shift, nch, p(counts), sp))
    ref_counts = np.bincount(hi >> shift, minlength=nch)
    np.testing.assert_array_equal(counts.cpu().numpy(), ref_counts)
    offsets = torch.empty(nch + 1, dtype=torch.int64, device="cuda")
    sc = torch.empty(int(L.magnus_mb_scan_scratch_bytes(nch)) // 8 + 1, dtype=torch.int64, device="cuda")
    _lib.check(L.magnus_mb_scan(p(counts), nch, p(offsets), p(sc), sp))
    ref_off = np.r_[0, np.cumsum(ref_counts)]
    np.testing.assert_array_equal(offsets.cpu().numpy(), ref_off)
    scratch = torch.empty(int(L.magnus_mb_reorder_scratch_bytes(size, nch)) // 8 + 1, dtype=torch.int64, device="cuda")
    oc = torch.empty(size, dtype=torch.int32, device="cuda")
    ov = torch.empty(size, dtype=torch.float64, device="cuda")
    _lib.check(L.magnus_mb_reorder(p(idx), p(vals), size, shift, nch, p(scratch), scratch.numel() * 8, p(oc), p(ov), sp))
    order = np.argsort(hi >> shift, kind="stable")   # stable scatter == stable sort by chunk
    np.testing.assert_array_equal(oc.cpu().numpy(), hi[order] & (chunk_len - 1))
    np.testing.assert_array_equal(ov.cpu().numpy().view(np.uint64), hv[order].view(np.uint64))
    dc = torch.empty(size, dtype=torch.int32, device="cuda")
    dv = torch.empty(size, dtype=torch.float64, device="cuda")
    dn = torch.empty(nch, dtype=torch.int64, device="cuda")
    _lib.check(L.magnus_mb_dense(p(oc), p(ov), p(offsets), nch, chunk_len, p(dc), p(dv), p(dn), sp))
    dc_h, dv_h, dn_h = dc.cpu().numpy(), dv.cpu().numpy(), dn.cpu().numpy()
    lc, lv = hi[order] & (chunk_len - 1), hv[order]
    for c in list(range(min(nch, 8))) + [nch - 1]:
        s0, s1 = ref_off[c], ref_off[c + 1]
        u, inv = np.unique(lc[s0:s1], return_inverse=True)
        sums = np.bincount(inv, weights=lv[s0:s1], minlength=u.size)   # sequential from 0.0 in slice order
        assert dn_h[c] == u.size
        np.testing.assert_array_equal(dc_h[s0:s0 + u.size], u)
        np.testing.assert_array_equal(dv_h[s0:s0 + u.size].view(np.uint64), sums.view(np.uint64))


def test_full_microbenchmark_records():
    recs = microbench.microbench_building_blocks(microbench.StreamSpec(1 << 22, 1 << 20, seed=3), 256, reps=2)
    names = [r.name for r in recs]
    assert names.count("reorder") == 2 and names[-1] == "total"
    assert all(r.seconds > 0 and r.rate > 0 for r in recs)
    bw, moved = microbench.measure_bandwidth(1 << 26, reps=2)
    assert bw > 1e11 and moved == 2 * (1 << 26)


def test_input_errors():
    with pytest.raises(InputError):
        microbench.microbench_building_blocks(microbench.StreamSpec(100, 64), 3)
    with pytest.raises(InputError):
        microbench.microbench_building_blocks(microbench.StreamSpec(100, 64), 128)
    with pytest.raises(InputError):
        microbench.StreamSpec(10, 0)


@pytest.mark.parametrize("n,bits", [(0, 8), (1, 1), (1000, 10), (4097, 20), ((1 << 20) + 3, 20), (300000, 52)])
def test_sort_pairs_matches_stable_sort(n, bits):
    """magnus_sort_pairs (hand-written LSD radix sort, csrc/radix_sort.cuh) == a stable sort of the keys: sorted keys and
    the permutation (ties keep their order), for few and many distinct keys."""
    from paper_2501_07056_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(n + bits)
    hi = min(1 << bits, 1 << 62)
    keys = torch.randint(0, hi, (n,), dtype=torch.int64, device="cuda", generator=g)
    if n > 10:
        keys[::7] = keys[3]   # many ties
    sk, perm = _lib.sort_pairs(keys, bits)
    rk, rperm = torch.sort(keys, stable=True)
    assert torch.equal(sk, rk)
    assert torch.equal(perm, rperm)
