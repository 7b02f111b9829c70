"""CPU oracle of the Gustavson baselines (oracle_gustavson) pinned bit-exact to
the reference's gustavson_dense / gustavson_esc (gustavson.py:155-268) outputs."""

import numpy as np
import pytest

import golden_util as gu
import gustavson_golden as gg
from oracle import oracle


@pytest.mark.parametrize("case", gg.cases())
@pytest.mark.parametrize("algo", ["dense", "esc"])
def test_oracle_gustavson_matches_reference(case, algo):
    A, B = gu.inputs(case)
    rp, col, val, counters = gg.expected(case, algo)
    r = oracle.gustavson(A, B, esc=(algo == "esc"))
    np.testing.assert_array_equal(r.row_ptr, rp)
    np.testing.assert_array_equal(r.col, col)
    np.testing.assert_array_equal(r.val.view(np.uint64), val.view(np.uint64))
    assert r.counters == counters
