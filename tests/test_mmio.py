"""Matrix-file layer (paper_2501_07056_b200.mmio) against the reference's mmio.py
(golden tests/golden/io_v1.npz, made by make_golden_io.py from the unmodified
reference): parsed CSR bit-exact, same ParseError line numbers, byte-identical
SPGC and Matrix Market output; round trips; device loading (gpu)."""

import json
import os

import numpy as np
import pytest

import golden_util as gu
from paper_2501_07056_b200 import CsrMatrix, ParseError, generate
from paper_2501_07056_b200 import mmio

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "io_v1.npz"))
MAN = json.loads(bytes(Z["manifest"]).decode())


def _write(tmp_path, name, data: bytes):
    p = tmp_path / name
    p.write_bytes(data)
    return p


@pytest.mark.parametrize("rec", MAN["good"], ids=[r["key"] for r in MAN["good"]])
def test_read_matches_reference(tmp_path, rec):
    k = rec["key"]
    M = mmio.read_matrix_market(_write(tmp_path, "m.mtx", Z[f"{k}/text"].tobytes()))
    assert [M.n_rows, M.n_cols] == rec["shape"]
    assert str(M.col.dtype) == rec["col_dtype"]
    np.testing.assert_array_equal(M.row_ptr, Z[f"{k}/rp"])
    np.testing.assert_array_equal(M.col, Z[f"{k}/col"])
    np.testing.assert_array_equal(M.val.view(np.uint64), Z[f"{k}/val"].view(np.uint64))


@pytest.mark.parametrize("rec", MAN["bad"], ids=[r["name"] for r in MAN["bad"]])
def test_parse_errors_match_reference(tmp_path, rec):
    with pytest.raises(ParseError) as e:
        mmio.read_matrix_market(_write(tmp_path, "bad.mtx", Z[f"bad_{rec['name']}/text"].tobytes()))
    assert e.value.line == rec["line"]


@pytest.mark.parametrize("rec", MAN["writers"], ids=[r["case"] for r in MAN["writers"]])
def test_writers_byte_identical(tmp_path, rec):
    A, _ = gu.inputs(rec["case"])
    mmio.write_binary_cache(A, tmp_path / "a.spgc")
    assert (tmp_path / "a.spgc").read_bytes() == Z[f"w_{rec['case']}/spgc"].tobytes()
    mmio.write_matrix_market(A, tmp_path / "a.mtx", comment=rec["comment"])
    assert (tmp_path / "a.mtx").read_bytes() == Z[f"w_{rec['case']}/mtx"].tobytes()


def test_round_trips(tmp_path):
    A = generate.rmat(10, 8, seed=3)
    for name in ("a.spgc", "a.bin", "a.mtx"):
        mmio.write_matrix(A, tmp_path / name)
        M = mmio.read_matrix(tmp_path / name)
        np.testing.assert_array_equal(M.row_ptr, np.asarray(A.row_ptr, np.int64))
        np.testing.assert_array_equal(M.col, np.asarray(A.col).astype(np.uint32))
        np.testing.assert_array_equal(M.val.view(np.uint64), np.asarray(A.val).view(np.uint64))
    empty = CsrMatrix(4, 6, np.zeros(5, np.int64), np.empty(0, np.uint32), np.empty(0))
    mmio.write_matrix(empty, tmp_path / "e.spgc")
    M = mmio.read_matrix(tmp_path / "e.spgc")
    assert (M.n_rows, M.n_cols, M.nnz) == (4, 6, 0)


def test_cache_errors(tmp_path):
    A = generate.rmat(8, 4, seed=1)
    mmio.write_binary_cache(A, tmp_path / "a.spgc")
    raw = (tmp_path / "a.spgc").read_bytes()
    for bad, msg in ((b"XXXX" + raw[4:], "bad magic"), (raw[:-8], "truncated"), (raw[:20], "bad magic"),
                     (raw[:4] + b"\x02" + raw[5:], "version"), (raw[:32] + b"\x03" + raw[33:], "widths")):
        with pytest.raises(ParseError, match=msg):
            mmio.read_binary_cache(_write(tmp_path, "b.spgc", bad))


def test_duplicates_summed_in_input_order():
    r = np.array([0, 0, 0, 1])
    c = np.array([2, 2, 2, 0])
    v = np.array([1e16, 1.0, -1e16, 5.0])
    M = mmio.csr_from_coo(r, c, v, 2, 3)
    assert M.val[0] == (0.0 + 1e16 + 1.0) - 1e16   # np.bincount order
    np.testing.assert_array_equal(M.row_ptr, [0, 1, 2])


@pytest.mark.gpu
def test_device_load_feeds_spgemm(tmp_path):
    torch = pytest.importorskip("torch")
    from oracle import oracle
    from paper_2501_07056_b200 import SystemParams, spgemm_magnus

    A = generate.rmat(11, 8, seed=5)
    mmio.write_binary_cache(A, tmp_path / "a.spgc")
    D = mmio.read_binary_cache(tmp_path / "a.spgc", device="cuda")
    assert D.row_ptr.is_cuda and D.col.dtype == torch.int32
    sysp = SystemParams(cache_line_bytes=128, l2_bytes=232448, memory_budget_bytes=1 << 30)
    res = spgemm_magnus(D, D, sys=sysp)
    ref = oracle.spgemm(A, A, sysp)
    np.testing.assert_array_equal(res.C.col.cpu().numpy().view(np.uint32), ref.col)
    np.testing.assert_array_equal(res.C.val.cpu().numpy().view(np.uint64), ref.val.view(np.uint64))
