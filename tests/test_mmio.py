"""Matrix Market files against the compiled reference.

The library's reader (csrc/mmio.cu: multi-threaded parse, sort-and-fold in
place of the reference's std::map passes) must give the reference's
read_matrix_market_file + assemble_problem result bit for bit -- CSR, the
Laplacian/adjacency decision and the warnings -- and fail with the same
message on every malformed input; the writer must produce the reference's
bytes. Host only (no GPU).
"""
import os

import numpy as np
import pytest

from paper_1108_1310_b200 import graphs as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MM_REF = os.path.join(ROOT, "oracle", "_ref", "mm_ref")
pytestmark = pytest.mark.skipif(not os.path.exists(MM_REF), reason="oracle/_ref/mm_ref not built")


class RefFailure(Exception):
    def __init__(self, msg):
        super().__init__(msg)
        self.msg = msg


def _ref_read(path, kind, policy, tmp):
    """The unmodified reference reader (oracle/_ref/mm_ref, a separate process)."""
    import struct
    import subprocess
    out = str(tmp) + ".bin"
    subprocess.run([MM_REF, str(path), str(kind), str(int(policy)), out], check=True, timeout=120)
    buf = open(out, "rb").read()
    st = struct.unpack_from("<i", buf, 0)[0]
    if st != 0:
        raise RefFailure(buf[4:].decode())
    n, m, lap, nw = struct.unpack_from("<iqii", buf, 4)
    off = 24
    warnings = []
    for _ in range(nw):
        ln = struct.unpack_from("<i", buf, off)[0]
        warnings.append(buf[off + 4:off + 4 + ln].decode())
        off += 4 + ln

    def take(dt, cnt):
        nonlocal off
        a = np.frombuffer(buf, dtype=dt, count=cnt, offset=off).copy()
        off += a.nbytes
        return a
    rp = take(np.int64, n + 1)
    col = take(np.int32, 2 * m)
    val = take(np.float64, 2 * m)
    diag = take(np.float64, n)
    return G.SparseLaplacian(n, m, rp, col, val, diag), bool(lap), warnings


def _same(a, b):
    assert (a.n, a.m) == (b.n, b.m)
    for f in ("row_ptr", "col", "val", "diag"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _random_file(rng, n, nnz, field, symmetry, laplacian, dup_frac=0.1, crlf=False, comments=True):
    lines = [f"%%MatrixMarket matrix coordinate {field} {symmetry}"]
    if comments:
        lines += ["% generated", "%"]
    ent = []
    if laplacian:
        a = G.random_connected(n, 1.5, int(rng.integers(1 << 30)))
        for u in range(n):
            ent.append((u, u, a.diag[u]))
            for k in range(a.row_ptr[u], a.row_ptr[u + 1]):
                v = int(a.col[k])
                if symmetry == "general" or v < u:
                    ent.append((u, v, a.val[k]))
    else:
        for _ in range(nnz):
            u, v = int(rng.integers(n)), int(rng.integers(n))
            ent.append((u, v, float(rng.normal()) * 10 ** float(rng.uniform(-3, 3))))
        for _ in range(int(dup_frac * nnz)):
            ent.append(ent[int(rng.integers(len(ent)))])
        rng.shuffle(ent)
    lines.append(f"{n} {n} {len(ent)}")
    for u, v, w in ent:
        lines.append(f"{u + 1} {v + 1}" + ("" if field == "pattern" else f" {float(w)!r}"))
    sep = "\r\n" if crlf else "\n"
    return sep.join(lines) + sep


@pytest.mark.parametrize("case", range(12))
def test_reader_matches_reference(tmp_path, case):
    from paper_1108_1310_b200 import lamg as L
    rng = np.random.default_rng(100 + case)
    field = ["real", "pattern"][case % 2]
    symmetry = ["general", "symmetric"][(case // 2) % 2]
    laplacian = field == "real" and case % 3 == 0
    n = int(rng.integers(5, 400))
    text = _random_file(rng, n, int(rng.integers(1, 3 * n)), field, symmetry, laplacian, crlf=case % 5 == 4)
    path = _write(tmp_path, f"c{case}.mtx", text)
    for kind, kname in ((0, "auto"), (1, "adjacency"), (2, "laplacian")):
        for pol in (True, False):
            try:
                want = _ref_read(path, kind, pol, tmp_path / f"r{kind}{pol}")
            except RefFailure as e:
                with pytest.raises(L.Error) as ei:
                    L.read_matrix_market(path, kname, pol)
                assert str(ei.value) == f"{ei.value.kind}: {e.msg}"
                continue
            got = L.read_matrix_market(path, kname, pol)
            _same(got[0], want[0])
            assert got[1] == want[1] and got[2] == want[2], (got[1:], want[1:])


BAD = {
    "empty": ("", None),
    "banner": ("%%MatrixMarkey matrix coordinate real general\n2 2 1\n1 2 1\n", None),
    "object": ("%%MatrixMarket vector coordinate real general\n2 2 1\n1 2 1\n", None),
    "array": ("%%MatrixMarket matrix array real general\n2 2\n1\n", None),
    "integer": ("%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 2 1\n", None),
    "field": ("%%MatrixMarket matrix coordinate quaternion general\n2 2 1\n1 2 1\n", None),
    "symmetry": ("%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 2 1\n", None),
    "size": ("%%MatrixMarket matrix coordinate real general\n% c\n2 x 1\n1 2 1\n", None),
    "norows": ("%%MatrixMarket matrix coordinate real general\n0 0 0\n", None),
    "square": ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 2 1\n", None),
    "entry": ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1\n1 x 1\n", None),
    "value": ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1\n2 3\n", None),
    "bounds": ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1\n4 1 1\n", None),
    "eof": ("%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 1\n\n% c\n2 3 1\n", None),
    "after_nnz": ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1\n2 3 1\ngarbage\n", None),
    "asym_lap": ("%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 1\n2 2 1\n1 2 -1\n2 1 -2\n", None),
    "selfloops": ("%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 2\n1 2 1\n2 3 -5\n3 3 1\n", None),
}


@pytest.mark.parametrize("name", list(BAD))
def test_edge_cases_match_reference(tmp_path, name):
    from paper_1108_1310_b200 import lamg as L
    path = _write(tmp_path, name + ".mtx", BAD[name][0])
    for kind, kname in ((0, "auto"), (1, "adjacency"), (2, "laplacian")):
        try:
            want = _ref_read(path, kind, True, tmp_path / f"r{kind}")
        except RefFailure as e:
            with pytest.raises(L.Error) as ei:
                L.read_matrix_market(path, kname, True)
            assert str(ei.value) == f"{ei.value.kind}: {e.msg}", (str(ei.value), e.msg)
            continue
        got = L.read_matrix_market(path, kname, True)
        _same(got[0], want[0])
        assert got[1:] == want[1:]


def _write_restated(a, lap):
    """write_matrix_market (matrix_market.cpp:196-216) restated: one triangle,
    row index >= column index, %.17g values."""
    out = ["%%MatrixMarket matrix coordinate real symmetric", f"{a.n} {a.n} {a.m + a.n if lap else a.m}"]
    for u in range(a.n):
        if lap:
            out.append(f"{u + 1} {u + 1} {'%.17g' % a.diag[u]}")
        for k in range(a.row_ptr[u], a.row_ptr[u + 1]):
            v = int(a.col[k])
            if v >= u:
                out.append(f"{v + 1} {u + 1} {'%.17g' % (a.val[k] if lap else -a.val[k])}")
    return "\n".join(out) + "\n"


def test_missing_file_and_writer(tmp_path):
    from paper_1108_1310_b200 import lamg as L
    with pytest.raises(L.IoError) as ei:
        L.read_matrix_market(str(tmp_path / "nope.mtx"))
    with pytest.raises(RefFailure) as er:
        _ref_read(tmp_path / "nope.mtx", 0, True, tmp_path / "nope")
    assert str(ei.value) == f"IoError: {er.value.msg}"
    a = G.random_connected(60, 2.0, 9)
    for lap in (False, True):
        p1 = str(tmp_path / f"ours{lap}.mtx")
        L.write_matrix_market(p1, a, lap)
        assert open(p1).read() == _write_restated(a, lap)
        back, was_lap, _ = L.read_matrix_market(p1)
        _same(back, a)
        assert was_lap == lap
        want = _ref_read(p1, 0, True, tmp_path / f"w{lap}")
        _same(want[0], a)
