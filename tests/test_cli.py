"""Command line front end (cli.py; SPEC.md External Interfaces): subcommands, flags,
MAGNUS_* environment overrides, CSV/JSON records, exit codes 0 / 1 / 2."""

import json
import os

import numpy as np
import pytest

from paper_2501_07056_b200 import cli, generate, mmio


def test_gen_writes_readable_files(tmp_path):
    for kind, extra, fname in (("rmat", ["--scale", "8", "--edge-factor", "4"], "r.spgc"),
                               ("er", ["--n", "300", "--per-row", "5"], "e.mtx"),
                               ("banded", ["--grid", "4"], "b.bin"), ("config", ["--config", "1"], "c.spgc")):
        assert cli.main(["gen", kind, "-o", str(tmp_path / fname), "--seed", "2", *extra]) == 0
        m = mmio.read_matrix(tmp_path / fname)
        assert m.nnz > 0
    r = mmio.read_matrix(tmp_path / "r.spgc")
    ref = generate.rmat(8, 4, seed=2)
    np.testing.assert_array_equal(r.col, np.asarray(ref.col).astype(np.uint32))
    assert mmio.read_matrix(tmp_path / "b.bin").nnz == 27 * 8 + 18 * 24 + 12 * 24 + 8 * 8   # 4^3 stencil: corners/edges/faces/inner


def test_usage_errors_exit_2(tmp_path, capsys):
    for argv in ([], ["nope"], ["gen"], ["gen", "rmat"], ["spgemm"], ["spgemm", "a", "--algo", "bad"],
                 ["microbench", "--chunks", "x"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2


def test_environment_overrides(monkeypatch):
    monkeypatch.setenv("MAGNUS_ALGO", "esc")
    monkeypatch.setenv("MAGNUS_L2_BYTES", "4096")
    monkeypatch.setenv("MAGNUS_FORCE_FINE_ONLY", "1")
    a = cli.build_parser().parse_args(["spgemm", "x.spgc"])
    assert (a.algo, a.l2_bytes, a.force_fine_only) == ("esc", 4096, True)
    a = cli.build_parser().parse_args(["spgemm", "x.spgc", "--algo", "dense"])
    assert a.algo == "dense"


def test_missing_file_is_usage_error(tmp_path):
    assert cli.main(["gen", "rmat", "-o", str(tmp_path / "no" / "such" / "dir.spgc"), "--scale", "4"]) == 2


@pytest.mark.gpu
def test_gpu_subcommands(tmp_path, capsys):
    a = str(tmp_path / "a.spgc")
    assert cli.main(["gen", "rmat", "--scale", "11", "--edge-factor", "8", "-o", a]) == 0
    capsys.readouterr()
    for algo in ("magnus", "dense", "esc"):
        csvp = str(tmp_path / "r.csv")
        assert cli.main(["spgemm", a, "--algo", algo, "--reps", "2", "--json", "--csv", csvp,
                         "-o", str(tmp_path / f"c_{algo}.spgc")]) == 0
        recs = [json.loads(x) for x in capsys.readouterr().out.strip().splitlines()]
        assert len(recs) == 2 and recs[0]["benchmark"] == f"spgemm_{algo}" and recs[0]["rate"] > 0
    cs = [mmio.read_matrix(tmp_path / f"c_{algo}.spgc") for algo in ("magnus", "dense", "esc")]
    for c in cs[1:]:
        np.testing.assert_array_equal(c.col, cs[0].col)
    assert open(csvp).read().count("\n") == 7   # header + 3 x 2 records
    assert cli.main(["verify", a]) == 0
    assert "PASS" in capsys.readouterr().out
    assert cli.main(["bound", a, "--json"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["params"]["read_bytes"] > 0
    assert cli.main(["bandwidth", "--bytes", str(1 << 26), "--json"]) == 0
    assert json.loads(capsys.readouterr().out)["rate"] > 100
    assert cli.main(["microbench", "--size", str(1 << 20), "--length", str(1 << 16), "--chunks", "64", "--reps", "1",
                     "--json"]) == 0
    names = [json.loads(x)["benchmark"] for x in capsys.readouterr().out.strip().splitlines()]
    assert names == ["histogram", "prefix_sum", "reorder", "dense_accum", "sort_accum", "stream", "total"]
