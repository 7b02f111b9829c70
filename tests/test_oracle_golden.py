"""Pin the CPU oracle (oracle/) against the reference's own outputs: bit-exact
row_ptr, col and value bits, identical counters, identical errors."""

import numpy as np
import pytest

from oracle import oracle
from paper_2501_07056_b200.errors import OverBudgetError

from golden_util import expected, inputs, runs, system

RUNS = runs()


@pytest.mark.parametrize("rec", RUNS, ids=[f"{r['case']}-{r['sys']}-{int(r.get('force_fine_only', 0))}" for r in RUNS])
def test_oracle_matches_reference(rec):
    A, B = inputs(rec["case"])
    sysp = system(rec["sys"], rec)
    if rec.get("error"):
        with pytest.raises(OverBudgetError):
            oracle.spgemm(A, B, sysp, force_fine_only=rec.get("force_fine_only", False))
        return
    res = oracle.spgemm(A, B, sysp, force_fine_only=rec["force_fine_only"], threads=2)
    rp, col, val = expected(rec)
    np.testing.assert_array_equal(res.row_ptr, rp)
    np.testing.assert_array_equal(res.col, col)
    np.testing.assert_array_equal(res.val.view(np.uint64), val.view(np.uint64))
    assert res.counters == rec["counters"]
