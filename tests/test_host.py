"""Host-side logic (no GPU): planner known answers (SPEC.md examples), the
accumulator policy, the C-ABI library's exports, planner agreement between the
Python planner, the C-ABI planner and the oracle."""

import ctypes as C
import os
import random

import numpy as np
import pytest

from oracle import oracle
from paper_2501_07056_b200 import (AccumThresholds, InputError, SystemParams, compute_chunk_plan, generate,
                                   merge_chunks_for_sort, select_accumulator)
from paper_2501_07056_b200 import _lib
from paper_2501_07056_b200.accumulators import Accum
from paper_2501_07056_b200.planner import NUMERIC, SYMBOLIC, fine_level_storage, max_l2_cols, round_pow2_of_sqrt

HDRS = [os.path.join(os.path.dirname(__file__), "..", "include", h) for h in ("magnus_b200.h", "magnus_gen.h")]


def test_planner_spec_examples():
    # SPEC.md:293  mC=2^18, numeric, val_bytes=4, line 64 -> n_fine=128, len=2^11
    p = compute_chunk_plan(SystemParams(val_bytes=4), 1 << 18, NUMERIC)
    assert (p.s_dense_accum, p.s_chunk_fine, p.n_chunks_fine, p.chunk_len_fine) == (5, 136, 128, 2048)
    # SPEC.md:294-295 / :454  m_max_l2 = 2^32 @ 2 MiB and 2^30 @ 1 MiB (symbolic)
    assert max_l2_cols(2 << 20, 1, 136) == 1 << 32
    assert max_l2_cols(1 << 20, 1, 136) == 1 << 30
    # SPEC.md:296  mC=2^33 with m_max=2^32 -> 2 coarse chunks
    p = compute_chunk_plan(SystemParams(l2_bytes=2 << 20), 1 << 33, SYMBOLIC)
    assert p.use_coarse and p.n_chunks_coarse == 2 and p.chunk_len_coarse == 1 << 32


def test_accumulator_policy_spec_examples():
    th = AccumThresholds()
    assert select_accumulator(0, th) is Accum.SORT
    assert select_accumulator(255, th) is Accum.SORT
    assert select_accumulator(256, th) is Accum.DENSE
    assert list(merge_chunks_for_sort([10, 10, 10, 10], 32)) == [0, 3, 4]
    assert list(merge_chunks_for_sort([32], 32)) == [0, 1]
    assert list(merge_chunks_for_sort([40], 32)) == [0, 1]
    with pytest.raises(InputError):
        AccumThresholds(sort_dense_crossover=16, sort_sweet_spot=32)


def test_round_pow2_of_sqrt_matches_float_definition():
    rng = random.Random(5)
    for _ in range(2000):
        num, den = rng.randint(1, 1 << 40), rng.randint(1, 1 << 12)
        r = round_pow2_of_sqrt(num, den)
        if num < den:
            assert r == 1
            continue
        # nearest on the log2 scale, ties up
        x = 0.5 * np.log2(num / den)
        k = int(np.floor(x))
        expect = 1 << (k + 1 if x - k >= 0.5 - 1e-12 else k)
        if abs((x - k) - 0.5) > 1e-9:
            assert r == expect


def test_planner_optimality_and_oracle_agreement():
    # Eq.(2) at the returned n_fine <= at its power-of-two neighbours
    rng = random.Random(11)
    for _ in range(50):
        sysp = SystemParams(cache_line_bytes=1 << rng.randint(5, 8), l2_bytes=rng.randint(1 << 10, 1 << 22))
        m_c = rng.randint(1, 1 << 34)
        for phase in (SYMBOLIC, NUMERIC):
            p = compute_chunk_plan(sysp, m_c, phase)
            span = p.chunk_len_fine * p.n_chunks_fine
            cap = max(1, span // max(1, sysp.cache_line_bytes // 4))
            s = fine_level_storage(p.n_chunks_fine, span, p.s_dense_accum, p.s_chunk_fine)
            if p.n_chunks_fine // 2 >= 1:
                assert s <= fine_level_storage(p.n_chunks_fine // 2, span, p.s_dense_accum, p.s_chunk_fine) or \
                    p.n_chunks_fine == cap
            if p.n_chunks_fine * 2 <= cap:
                assert s <= fine_level_storage(p.n_chunks_fine * 2, span, p.s_dense_accum, p.s_chunk_fine)
            o = oracle.chunk_plan(sysp, m_c, phase == NUMERIC)
            assert o["n_chunks_fine"] == p.n_chunks_fine and o["chunk_len_fine"] == p.chunk_len_fine
            assert bool(o["use_coarse"]) == p.use_coarse and o["m_max_l2"] == p.m_max_l2


def _header_symbols():
    import re
    txt = "".join(open(h).read() for h in HDRS)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|int64_t|size_t)\s+(magnus_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    _lib.build()
    L = _lib.lib()
    syms = _header_symbols()
    assert set(syms) == set(_lib.EXPORTS) | set(_lib.GEN_EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.magnus_version()


def test_abi_chunk_plan_matches_python_planner():
    _lib.build()
    L = _lib.lib()
    rng = random.Random(3)
    for _ in range(200):
        sysp = SystemParams(cache_line_bytes=1 << rng.randint(4, 8), l2_bytes=rng.randint(64, 1 << 23),
                            val_bytes=rng.choice([4, 8]))
        m_c = rng.randint(1, 1 << 36)
        for numeric in (0, 1):
            out = _lib.Plan()
            s = _lib.Sys(sysp.cache_line_bytes, sysp.l2_bytes, sysp.memory_budget_bytes, 4, 4, sysp.val_bytes)
            assert L.magnus_compute_chunk_plan(C.byref(s), m_c, numeric, 1, C.byref(out)) == 0
            p = compute_chunk_plan(sysp, m_c, NUMERIC if numeric else SYMBOLIC)
            for f, _ in _lib.Plan._fields_:
                assert int(getattr(out, f)) == int(getattr(p, f)), f


def test_generators_are_deterministic_and_canonical():
    from paper_2501_07056_b200.matrix import validate_csr
    a = generate.rmat(10, 16, seed=7)
    b = generate.rmat(10, 16, seed=7)
    np.testing.assert_array_equal(a.col, b.col)
    np.testing.assert_array_equal(a.val, b.val)
    assert validate_csr(a)
    u = generate.uniform_rows(1000, 5000, 16, seed=3)
    assert validate_csr(u)
    assert (np.diff(u.row_ptr) == 16).all()
    s = generate.stencil27(8)
    assert validate_csr(s)
    assert s.nnz == (3 * 8 - 2) ** 3


def test_ideal_bound_formula():
    """reference bound.py:44-53: two-pass read volume and single write of C."""
    from paper_2501_07056_b200 import IdealBoundInputs, InputError, bound_inputs_for, col_index_bytes, ideal_bound
    inp = IdealBoundInputs(n_a=10, nnz_a=30, n_inter_prod=100, n_c=10, nnz_c=50, s_row_ptr=8, s_col_idx=4, s_val=8,
                           bandwidth_bytes_per_sec=1e3)
    r, w, t = ideal_bound(inp)
    assert r == 2 * 11 * 8 + 30 * (32 + 8 + 8) + 100 * (8 + 8)
    assert w == 11 * 8 + 50 * 12
    assert t == (r + w) / 1e3
    assert col_index_bytes(2 ** 32) == 4 and col_index_bytes(2 ** 32 + 1) == 8
    with pytest.raises(InputError):
        IdealBoundInputs(n_a=-1, nnz_a=0, n_inter_prod=0, n_c=0, nnz_c=0)
    with pytest.raises(InputError):
        IdealBoundInputs(n_a=1, nnz_a=0, n_inter_prod=0, n_c=0, nnz_c=0, bandwidth_bytes_per_sec=0)
    from paper_2501_07056_b200 import generate
    A = generate.uniform_rows(64, 64, 4, seed=1)
    b = bound_inputs_for(A, A, nnz_c=200, n_inter_prod=256, bandwidth_bytes_per_sec=2.0)
    assert (b.n_a, b.nnz_a, b.s_row_ptr, b.s_col_idx, b.s_val) == (64, 256, 8, 4, 8)
