"""Matrix Market / permutation / manifest I/O and the csrk CLI (reference
pkg/tests/test_io.py, test_bench.py CLI parts).  Parsing and argument
handling run on CPU; commands that compute run under -m gpu."""

from __future__ import annotations

import argparse
import io
import json

import numpy as np
import pytest

import paper_2203_05096_b200 as ck
from conftest import random_csr, tridiagonal
from paper_2203_05096_b200.cli import _parse_block_dims, build_parser, main


def read_str(text):
    return ck.read_matrix_market(io.StringIO(text))


def _dense(a):
    d = np.zeros((a.n_rows, a.n_cols))
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.astype(np.int64)))
    np.add.at(d, (rows, a.col_idx.astype(np.int64)), a.vals)
    return d


def test_parse_fields_and_symmetries():
    a = read_str("%%MatrixMarket matrix coordinate real general\n% c\n\n2 3 2\n1 1 2.5\n2 3 -1.0\n")
    assert (a.n_rows, a.n_cols, a.nnz) == (2, 3, 2) and _dense(a)[1, 2] == -1.0
    s = read_str("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 2\n2 1 3\n")
    assert s.nnz == 3 and _dense(s)[0, 1] == 3.0
    k = read_str("%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 1\n3 1 2.0\n")
    assert _dense(k)[0, 2] == -2.0
    p = read_str("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n")
    assert p.vals.tolist() == [1.0, 1.0]
    i = read_str("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n")
    assert i.vals.dtype == np.float64 and i.vals.tolist() == [7.0]
    d = read_str("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n2 2 4\n")
    assert d.nnz == 2 and _dense(d)[0, 0] == 3.0


@pytest.mark.parametrize("text,match", [
    ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", "complex"),
    ("%%NotMatrixMarket matrix coordinate real general\n", "line 1"),
    ("%%MatrixMarket matrix array real general\n1 1\n", "format"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "header declared 2"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", "line 4"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "line 3"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 1 1.0\n", "line 3"),
    ("", "empty"),
])
def test_parse_errors_carry_line_numbers(text, match):
    with pytest.raises(ck.MatrixMarketError, match=match):
        read_str(text)


def test_write_read_round_trip_and_permutation_files(tmp_path):
    rng = np.random.default_rng(3)
    a = random_csr(rng, 25, 30, 0.2, -1.0, 1.0)
    path = tmp_path / "a.mtx"
    ck.write_matrix_market(a, path)
    b = ck.read_matrix_market(path)
    np.testing.assert_array_equal(b.row_ptr, a.row_ptr)
    np.testing.assert_array_equal(b.col_idx, a.col_idx)
    np.testing.assert_array_equal(b.vals, a.vals)
    buf = io.StringIO()
    ck.write_matrix_market(ck.build_csr(3, 3, [(i, i, 1.0) for i in range(3)]), buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general" and lines[1] == "3 3 3"
    perm = ck.Permutation.from_forward(rng.permutation(17))
    ck.write_permutation_file(perm, tmp_path / "p.txt")
    q = ck.read_permutation_file(tmp_path / "p.txt")
    np.testing.assert_array_equal(q.fwd, perm.fwd)


def test_manifest_parsing(tmp_path):
    path = tmp_path / "m.csv"
    path.write_text("id,name,n,nnz,max,class\nr1,grid,1.00,5.00,5,regular\n"
                    "i1,web,2.5,10.1,900,irregular\n")
    entries = ck.load_manifest(path)
    assert entries[0] == ck.ManifestEntry("r1", "grid", 1.0, 5.0, 5, "regular")
    assert entries[1].matrix_class == "irregular"
    path.write_text("id,name,n,nnz,max,class\nr1,grid,1.00,5.00,5,weird\n")
    with pytest.raises(ValueError, match="unknown class"):
        ck.load_manifest(path)
    path.write_text("bad,header\n")
    with pytest.raises(ValueError, match="header"):
        ck.load_manifest(path)


def test_cli_parsing():
    assert _parse_block_dims("8,12") == ck.BlockDims(8, 12, 1)
    assert _parse_block_dims("4,8,12") == ck.BlockDims(4, 8, 12)
    for bad in ("8", "1,2,3,4"):
        with pytest.raises(argparse.ArgumentTypeError):
            _parse_block_dims(bad)
    args = build_parser().parse_args(["run", "m.mtx"])
    assert (args.warmups, args.reps, args.tolerance, args.profile, args.format, args.tune) \
        == (5, 20, 1e-10, "volta", "json", "auto")
    with pytest.raises(SystemExit):
        main([])


@pytest.fixture
def mtx(tmp_path):
    path = tmp_path / "tri9.mtx"
    ck.write_matrix_market(tridiagonal(9), path)
    return str(path)


def test_cli_usage_errors_exit_2(mtx, capsys):
    assert main(["run", mtx, "--kernel", "cpu2", "--k", "3"]) == 2
    assert "conflicts" in capsys.readouterr().err
    assert main(["run", "/nonexistent/m.mtx", "--kernel", "ref"]) == 2
    assert "error:" in capsys.readouterr().err
    with pytest.raises(SystemExit) as exc:
        main(["compare", mtx, "--targets", "warp9"])
    assert exc.value.code == 2


@pytest.mark.gpu
def test_cli_commands_on_device(mtx, capsys):
    assert main(["info", mtx, "--format", "json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert (rep["n"], rep["nnz"], rep["max_row_nnz"], rep["class"]) == (9, 25, 3, "regular")
    assert main(["run", mtx, "--kernel", "cpu2", "--srs", "3", "--threads", "1"]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["schema_version"] == 1 and rec["passed"] and rec["tuning"]["srs"] == 3
    assert main(["run", mtx, "--kernel", "cuda35", "--block-dims", "4,8,12", "--warmups",
                 "0", "--reps", "2", "--format", "csv"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0].startswith("schema_version,matrix_id,kernel")
    assert main(["tune", mtx, "--device", "volta"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert (out["params"]["ssrs"], out["params"]["srs"]) == (8, 9)
    assert out["params"]["kernel_variant"] == "gpu3-emu"
    assert main(["compare", mtx, "--targets", "ref", "cpu3", "cuda3", "gpu35-emu",
                 "--warmups", "0", "--reps", "1"]) == 0
    cmp_ = json.loads(capsys.readouterr().out)
    by = {r["kernel"]: r for r in cmp_["results"]}
    assert by["ref"]["speedup"] == 1.0 and all(r["passed"] for r in cmp_["results"])
    assert main(["tune", mtx, "--device", "b200", "--grid", "--grid-reps", "1"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert len(out["table"]) == 64


@pytest.mark.parametrize("field,symmetry", [("real", "general"), ("integer", "symmetric"),
                                            ("pattern", "general"), ("real", "skew-symmetric")])
def test_native_matrix_market_body_equals_python_loop(tmp_path, monkeypatch, field, symmetry):
    """csrk_mm_parse (all host cores) parses large bodies to exactly what the
    reference's line loop yields (io.py:96-206), comments and blank lines
    included, and irregular lines fall back to the loop's exact errors."""
    from paper_2203_05096_b200 import format as F
    from paper_2203_05096_b200 import io as mio
    monkeypatch.setattr(F, "DEVICE_COO_MIN", 1 << 62)  # host canonicalisation here
    rng = np.random.default_rng(len(field) + len(symmetry))
    n, m = 3000, 30000
    r = rng.integers(1, n + 1, m).tolist()
    c = rng.integers(1, n + 1, m).tolist()
    if symmetry == "skew-symmetric":
        c = [(ci % n) + 1 if ci == ri else ci for ri, ci in zip(r, c)]
    v = (rng.standard_normal(m) * 10.0 ** rng.uniform(-30, 30, m)).tolist()
    if field == "integer":
        v = rng.integers(-9, 10, m).tolist()

    def entry(k):
        if field == "pattern":
            return f"{r[k]} {c[k]}"
        return f"  {r[k]}\t{c[k]}  {v[k]!r} " if k % 7 == 0 else f"{r[k]} {c[k]} {v[k]!r}"

    body = [entry(k) for k in range(m)]
    body.insert(10, "% a comment")
    body.insert(2000, "")
    body.insert(20000, "   % indented comment")
    text = "\n".join([f"%%MatrixMarket matrix coordinate {field} {symmetry}", "% header",
                      f"{n} {n} {m}"] + body) + "\n"
    path = tmp_path / "a.mtx"
    path.write_text(text)

    def both():
        out = []
        for threshold in (1, 1 << 62):
            monkeypatch.setattr(mio, "NATIVE_MIN_ENTRIES", threshold)
            try:
                a = mio.read_matrix_market(str(path))
                out.append((a.row_ptr.tobytes(), a.col_idx.tobytes(), a.vals.tobytes()))
            except mio.MatrixMarketError as e:
                out.append(str(e))
        return out

    native, python = both()
    assert native == python and not isinstance(native, str)
    for k, bad in ((7000, f"{n + 1} 1 1.0"), (15000, "1 2 3 4"), (25000, "1 2 nan(7)")):
        lines = text.split("\n")
        lines[k] = bad
        path.write_text("\n".join(lines))
        native, python = both()
        assert native == python
        assert isinstance(native, str) and native.startswith(f"line {k + 1}:")


def _mm_golden():
    import json
    import os
    import sys

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    import mm_cases
    with open(os.path.join(here, "mm.json")) as fh:
        return mm_cases, json.load(fh)


def _sha(b: bytes) -> str:
    import hashlib
    return hashlib.sha256(b).hexdigest()


def _check_mm_case(tmp_path, name, mm_cases, want):
    import io as _io

    from paper_2203_05096_b200 import io as mio
    path = tmp_path / f"{name}.mtx"
    path.write_text(mm_cases.mm_text(name))
    a = mio.read_matrix_market(str(path))
    assert (a.n_rows, a.n_cols, a.nnz) == (want["n_rows"], want["n_cols"], want["nnz"])
    assert _sha(np.ascontiguousarray(a.row_ptr, dtype="<u4").tobytes()) == want["row_ptr"]
    assert _sha(np.ascontiguousarray(a.col_idx, dtype="<u4").tobytes()) == want["col_idx"]
    assert _sha(np.ascontiguousarray(a.vals, dtype="<f8").tobytes()) == want["vals"]
    w = _io.StringIO()
    mio.write_matrix_market(a, w)
    assert _sha(w.getvalue().encode()) == want["written"]
    pf = _io.StringIO()
    mio.write_permutation_file(ck.Permutation.from_forward(mm_cases.perm_of(a.n_rows)), pf)
    assert _sha(pf.getvalue().encode()) == want["perm_file"]


@pytest.mark.parametrize("native", [False, True])
def test_matrix_market_ingest_equals_reference_goldens(tmp_path, monkeypatch, native):
    """Matrix Market -> canonical CSR (symmetric / skew / pattern expansion,
    duplicates summed), the writer and permutation files: digests the
    unmodified reference wrote (tests/golden/mm.json, make_golden.py mm).
    The body is parsed by the native parser (csrk_mm_parse, all host
    cores) or the line loop; canonicalisation on the host here."""
    from paper_2203_05096_b200 import format as F
    from paper_2203_05096_b200 import io as mio
    monkeypatch.setattr(F, "DEVICE_COO_MIN", 1 << 62)
    monkeypatch.setattr(mio, "NATIVE_MIN_ENTRIES", 1 if native else 1 << 62)
    mm_cases, gold = _mm_golden()
    for name in mm_cases.CASES:
        _check_mm_case(tmp_path, name, mm_cases, gold[name])


@pytest.mark.gpu
def test_matrix_market_ingest_on_device_equals_reference_goldens(tmp_path):
    """The same with the default thresholds: the large cases canonicalise
    on the GPU (csrk_coo_to_csr, >= 64 K triplets after expansion)."""
    mm_cases, gold = _mm_golden()
    for name in mm_cases.CASES:
        _check_mm_case(tmp_path, name, mm_cases, gold[name])


def test_packaged_manifest_equals_reference():
    """load_manifest() with no argument reads the packaged manifest of the
    paper's 64 matrices (data/manifest.csv, generated from PAPER.md's
    benchmark-suite table by tools/make_manifest.py): entry for entry what
    the reference's load_manifest() returns (digest in mm.json)."""
    import hashlib

    from paper_2203_05096_b200 import io as mio
    _, gold = _mm_golden()
    ents = mio.load_manifest()
    assert len(ents) == gold["_manifest"]["count"] == 64
    got = hashlib.sha256(repr([tuple(e.__dict__.values()) for e in ents]).encode()).hexdigest()
    assert got == gold["_manifest"]["entries"]
    assert sum(e.matrix_class == "regular" for e in ents) == 35
