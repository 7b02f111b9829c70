"""The per-entry summation rule the CUDA kernels implement, checked bit-exact
against the reference's golden outputs (host-logic test, no GPU).

For output entry (i, c) with contributions x_0..x_{d-1} in ascending k
(Gustavson order, reference gustavson.py:44-59; the stable reorders
matrix.py:187-204 and the coarse CSC traversal magnus.py:327 preserve it):

* row category Dense (magnus.py:492-503): ((+0.0 + x_0) + x_1) + ...
  (np.bincount / np.add.at, accumulators.py:88-95);
* row category Sort (magnus.py:483-490): x_0 + pairwise(x_1..x_{d-1})
  (np.add.reduceat, accumulators.py:129);
* Fine / Coarse: the numeric-plan fine chunk f = c >> shift_fine holds n_f of
  the row's intermediate elements; n_f >= crossover -> Dense rule, else Sort
  rule (_accumulate_chunks magnus.py:159-190; merge_chunks_for_sort never
  splits a column's contributions).
"""

import numpy as np
import pytest

from oracle import oracle
from paper_2501_07056_b200.planner import NUMERIC, compute_chunk_plan

from golden_util import expected, inputs, runs

SEQ0, PW = 0, 1


def rule_values(A, B, sysp, force_fine_only=False, crossover=256):
    inter, mn, mx, cat = oracle.setup(A, B, sysp, None, force_fine_only)
    plan = compute_chunk_plan(sysp, max(B.n_cols, 1), NUMERIC, allow_coarse=not force_fine_only)
    rp_out, cols_out, vals_out = [0], [], []
    Arp, Acol, Aval = np.asarray(A.row_ptr), np.asarray(A.col).astype(np.int64), np.asarray(A.val)
    Brp, Bcol, Bval = np.asarray(B.row_ptr), np.asarray(B.col).astype(np.int64), np.asarray(B.val)
    for i in range(A.n_rows):
        cs, vs = [], []
        for t in range(Arp[i], Arp[i + 1]):
            k = Acol[t]
            cs.append(Bcol[Brp[k]:Brp[k + 1]])
            vs.append(Bval[Brp[k]:Brp[k + 1]] * Aval[t])
        cs = np.concatenate(cs) if cs else np.empty(0, np.int64)
        vs = np.concatenate(vs) if vs else np.empty(0)
        order = np.argsort(cs, kind="stable")
        cs, vs = cs[order], vs[order]
        chunk_n = np.bincount(cs >> plan.shift_fine) if cs.size else np.empty(0, np.int64)
        uniq, starts = np.unique(cs, return_index=True)
        ends = np.r_[starts[1:], cs.size]
        for c, s, e in zip(uniq, starts, ends):
            if cat[i] == 1:
                mode = SEQ0
            elif cat[i] == 0:
                mode = PW
            else:
                mode = SEQ0 if chunk_n[c >> plan.shift_fine] >= crossover else PW
            if mode == SEQ0:
                acc = 0.0
                for x in vs[s:e]:
                    acc += x
            else:
                acc = vs[s] + oracle.pairwise_sum(vs[s + 1:e]) if e - s > 1 else vs[s]
            cols_out.append(c)
            vals_out.append(acc)
        rp_out.append(len(cols_out))
    return np.array(rp_out), np.array(cols_out, dtype=np.int64), np.array(vals_out)


SMALL = [r for r in runs() if not r.get("error") and r["case"] in ("rmat9", "hub", "stencil6", "rand4", "rand10")]


@pytest.mark.parametrize("rec", SMALL, ids=[f"{r['case']}-{r['sys']}-{int(r['force_fine_only'])}" for r in SMALL])
def test_rule_reproduces_reference(rec):
    from golden_util import system
    A, B = inputs(rec["case"])
    rp, col, val = rule_values(A, B, system(rec["sys"]), rec["force_fine_only"])
    erp, ecol, evals = expected(rec)
    np.testing.assert_array_equal(rp, erp)
    np.testing.assert_array_equal(col, ecol.astype(np.int64))
    np.testing.assert_array_equal(val.view(np.uint64), evals.view(np.uint64))
