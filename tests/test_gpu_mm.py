"""Matrix Market ingestion against the UNMODIFIED reference's
mm_read / mm_read_vector (oracle/_ref): same CSR bits (duplicates summed in
input order, symmetric storage expanded, columns sorted) and the same error
texts; FileSequence feeding the device reuse driver."""
import numpy as np
import pytest

from oracle import problems as P
from oracle import ref

pytestmark = pytest.mark.gpu
amg = pytest.importorskip("paper_2108_02054_b200")


def _bits(x):
    return np.asarray(x, np.float64).view(np.int64)


def _write(path, text):
    path.write_text(text)
    return path


CASES = {
    "general_dups": "%%MatrixMarket matrix coordinate real general\n% comment\n\n4 5 7\n"
                    "1 1 2.5\n3 2 -1e-3\n1 1 0.1\n  4 5 7 \n% mid comment\n2 2 1e300\n1 1 -0.0\n3 2 3\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 4\n2 1 -1\n3 2 -1.5\n3 3 2\n",
    "integer_crlf": "%%MatrixMarket matrix coordinate integer general\r\n2 2 3\r\n1 2 7\r\n2 1 -3\r\n2 2 5\r\n",
    "mixed_case_banner": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 1\n2 2 1.5\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n3 3 0\n",
    "extra_lines": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 junk here\n",
    "signed_hex_inf": "%%MatrixMarket matrix coordinate real general\n2 2 3\n+1 1 0x1p3\n2 2 inf\n1 2 -nan\n",
    "istream_split": "%%MatrixMarket matrix coordinate real general\n2 2 2\n2 2.5 1\n1 +2 -.25e1\n",
}

ERRORS = {
    "no_banner": "%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n% c\n3 x 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "malformed": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 x 1\n",
    "two_tokens": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "istream_exponent": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1e3 7\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n",
    "non_numeric": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 1.5x\n",
    "overflow": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e999\n",
    "eof": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n",
    "empty_file": "",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_mm_read_matches_reference(ctx, tmp_path, name):
    f = _write(tmp_path / f"{name}.mtx", CASES[name])
    rp, ci, v, ncols = ref.mm_read(f)
    M = amg.mm_read(f, ctx)
    grp, gci, gv = M.to_host()
    assert (M.nrows, M.ncols) == (len(rp) - 1, ncols)
    np.testing.assert_array_equal(grp, rp)
    np.testing.assert_array_equal(gci, ci)
    np.testing.assert_array_equal(_bits(gv), _bits(v))


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_mm_read_errors_match_reference(ctx, tmp_path, name):
    f = _write(tmp_path / f"{name}.mtx", ERRORS[name])
    with pytest.raises(ref.RefError) as r:
        ref.mm_read(f)
    with pytest.raises(amg.RuntimeFailure) as g:
        amg.mm_read(f, ctx)
    assert str(g.value) == str(r.value)


def test_mm_read_large_multithreaded_matches_reference(ctx, tmp_path):
    """~0.5M entries (several parse chunks) with duplicates, in random order."""
    rng = np.random.default_rng(11)
    n, m = 20000, 500000
    rows = rng.integers(1, n + 1, m)
    cols = rng.integers(1, n + 1, m)
    vals = rng.standard_normal(m) * 10.0 ** rng.integers(-5, 5, m)
    lines = ["%%MatrixMarket matrix coordinate real general", f"{n} {n} {m}"]
    lines += [f"{a} {b} {float(x)!r}" for a, b, x in zip(rows, cols, vals)]
    f = _write(tmp_path / "big.mtx", "\n".join(lines) + "\n")
    rp, ci, v, _ = ref.mm_read(f)
    grp, gci, gv = amg.mm_read(f, ctx).to_host()
    np.testing.assert_array_equal(grp, rp)
    np.testing.assert_array_equal(gci, ci)
    np.testing.assert_array_equal(_bits(gv), _bits(v))


def test_mm_read_vector_matches_reference(ctx, tmp_path):
    f = _write(tmp_path / "v.mtx", "%%MatrixMarket matrix array real general\n% rhs\n3 1\n1.5\n-2e-7\n  4 \n")
    np.testing.assert_array_equal(_bits(amg.mm_read_vector(f, ctx)), _bits(ref.mm_read_vector(f)))
    bad = _write(tmp_path / "w.mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n")
    with pytest.raises(ref.RefError) as r:
        ref.mm_read_vector(bad)
    with pytest.raises(amg.RuntimeFailure) as g:
        amg.mm_read_vector(bad, ctx)
    assert str(g.value) == str(r.value)


def _write_mm(path, A, symmetric=False):
    rp, ci, v = A
    n = len(rp) - 1
    lines = ["%%MatrixMarket matrix coordinate real general", f"{n} {n} {len(ci)}"]
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            lines.append(f"{i + 1} {ci[k] + 1} {float(v[k])!r}")
    path.write_text("\n".join(lines) + "\n")


def test_file_sequence_feeds_the_device_reuse_driver(ctx, tmp_path):
    """A FileSequence of dam-break steps on disk gives the same run as the
    in-memory sequence (the reader reproduces the matrices bit for bit)."""
    from paper_2108_02054_b200 import reuse as R

    g, steps = 12, 3
    mats = [P.grid3d_values("dambreak", g, k) for k in range(steps)]
    for k, A in enumerate(mats):
        _write_mm(tmp_path / f"step_{k:04d}.mtx", A)
    rhs = P.rhs(g ** 3)
    (tmp_path / "step_0001.rhs.mtx").write_text(
        "%%MatrixMarket matrix array real general\n" + f"{g ** 3} 1\n" + "\n".join(repr(float(x)) for x in rhs) + "\n")
    seq = R.FileSequence(tmp_path, ctx)
    assert seq.size() == steps

    class Mem:
        def size(self):
            return steps

        def step(self, k):
            return mats[k], (rhs if k == 1 else np.ones(g ** 3))

    cfg = R.StrategyConfig(R.StrategyKind.partial)
    a = R.run_sequence(seq, cfg, ctx=ctx)
    b = R.run_sequence(Mem(), cfg, ctx=ctx)
    assert [s.iterations for s in a.report.steps] == [s.iterations for s in b.report.steps]
    for ua, ub in zip(a.solutions, b.solutions):
        np.testing.assert_array_equal(_bits(ua), _bits(ub))
