"""File containers (reference io.hpp:25-41, io.cpp:80-207):
the product's host readers / writers and the oracle's numpy restatement
against fixtures written by the reference library itself
(tests/golden/make_golden_io.py), against the reference's own readers /
writers where oracle/_ref is built, and the cases of the reference's
test_io.cpp.  No GPU needed (the device loaders: test_io_gpu.py)."""
import os

import numpy as np
import pytest

import gspmm_testutil  # noqa: F401
import paper_2007_06354_b200 as P
from oracle import oracle as O

GOLD = os.path.join(gspmm_testutil.ROOT, "tests", "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def expected():
    return dict(np.load(os.path.join(GOLD, "io_expected.npz")))


def _same(a, b):
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("seed", [1, 8])
@pytest.mark.parametrize("tag,orient", [("src", P.SRC_MAJOR), ("dst", P.DST_MAJOR)])
def test_csr1_fixture_read_and_rewrite(expected, tmp_path, seed, tag, orient):
    path = os.path.join(GOLD, f"io_graph{seed}_{tag}.csr")
    n = int(expected[f"g{seed}_n"][0])
    want = [expected[f"g{seed}_{tag}_{k}"] for k in ("indptr", "indices", "eids")]
    for reader in (P.load_csr, O.read_csr1):
        o, r, c, *arrs = reader(path)
        assert (o, r, c) == (orient, n, n)
        assert all(_same(np.asarray(a, np.uint32), w) for a, w in zip(arrs, want))
    # the writers reproduce the reference's file byte for byte
    P.save_csr(tmp_path / "p.csr", orient, n, n, *want)
    O.write_csr1(tmp_path / "o.csr", orient, n, n, *want)
    ref_bytes = open(path, "rb").read()
    assert open(tmp_path / "p.csr", "rb").read() == ref_bytes
    assert open(tmp_path / "o.csr", "rb").read() == ref_bytes


def test_fmat1_fixture_read_and_rewrite(expected, tmp_path):
    path = os.path.join(GOLD, "io_feats.fmat")
    x = expected["feats"]
    assert _same(P.load_feature_matrix(path), x)
    assert _same(O.read_fmat1(path), x)
    P.save_feature_matrix(tmp_path / "p.fmat", x)
    O.write_fmat1(tmp_path / "o.fmat", x)
    ref_bytes = open(path, "rb").read()
    assert open(tmp_path / "p.fmat", "rb").read() == ref_bytes
    assert open(tmp_path / "o.fmat", "rb").read() == ref_bytes
    # a strided host matrix (column slice) writes only its own columns
    wide = np.zeros((37, 9), np.float32)
    wide[:, 2:7] = x
    P.save_feature_matrix(tmp_path / "s.fmat", wide[:, 2:7])
    assert open(tmp_path / "s.fmat", "rb").read() == ref_bytes


@pytest.mark.parametrize("seed", [1, 8])
def test_edge_list_fixture(expected, tmp_path, seed):
    path = os.path.join(GOLD, f"io_graph{seed}.txt")
    n, src, dst = P.load_edge_list(path)
    assert n == int(expected[f"g{seed}_n"][0])
    assert _same(src, expected[f"g{seed}_src"]) and _same(dst, expected[f"g{seed}_dst"])
    P.save_edge_list(tmp_path / "e.txt", n, src, dst)
    assert open(tmp_path / "e.txt", "rb").read() == open(path, "rb").read()
    # text -> canonical CSR == the reference's CSR1 of the same graph
    csr = P.build_csr(n, src, dst, P.DST_MAJOR)
    assert all(_same(a, expected[f"g{seed}_dst_{k}"])
               for a, k in zip(csr, ("indptr", "indices", "eids")))


# ---- the reference's own cases (test_io.cpp) --------------------------------
def test_edge_list_text_parsing(tmp_path):  # test_io.cpp:44-52
    (tmp_path / "e.txt").write_text("0 2\n1 2\n")
    n, src, dst = P.load_edge_list(tmp_path / "e.txt")
    assert n == 3 and src.tolist() == [0, 1] and dst.tolist() == [2, 2]


def test_edge_list_header_and_comments(tmp_path):  # test_io.cpp:54-60
    (tmp_path / "e.txt").write_text("# a comment\n%nodes 10\n0 1   # trailing\n\n")
    n, src, dst = P.load_edge_list(tmp_path / "e.txt")
    assert n == 10 and src.tolist() == [0] and dst.tolist() == [1]


@pytest.mark.parametrize("text,line,what", [
    ("0 x\n", 1, "expected 'src dst'"),                   # test_io.cpp:62-71
    ("0 1\n%nodes 2\n5 1\n", 3, "node id >= %nodes"),      # test_io.cpp:73-81
    ("0 1\n%edges 4\n", 2, "unknown '%' directive"),
    ("%nodes x\n", 1, "bad %nodes value"),
    ("%nodes 99999999999\n", 1, "%nodes overflows id width"),
    ("0 1 2\n", 1, "trailing garbage after edge"),
    ("0 4294967295\n", 1, "node id overflows id width"),
    ("1 2\r\n3\r\n", 2, "expected 'src dst'"),
])
def test_edge_list_parse_errors_carry_the_line(tmp_path, text, line, what):
    path = tmp_path / "bad.txt"
    path.write_bytes(text.encode())
    with pytest.raises(P.ParseError) as ei:
        P.load_edge_list(path)
    assert f"{path}:{line}: {what}" in str(ei.value)
    if O.ref_available():  # the reference fails the same way, same message
        with pytest.raises(O.OracleError) as ri:
            O.ref_load_edge_list(str(path))
        assert ri.value.status == O.PARSE_ERROR and f"{path}:{line}: {what}" in str(ri.value)


def test_edge_list_round_trip_keeps_isolated_nodes(tmp_path):  # test_io.cpp:83-91
    src, dst = np.array([0, 5, 3], np.uint32), np.array([5, 0, 3], np.uint32)
    P.save_edge_list(tmp_path / "rt.txt", 9, src, dst)
    n, s, d = P.load_edge_list(tmp_path / "rt.txt")
    assert n == 9 and _same(s, src) and _same(d, dst)


def test_edge_list_crlf_and_empty(tmp_path):
    (tmp_path / "crlf.txt").write_bytes(b"0 1\r\n2 3\r\n")
    n, s, d = P.load_edge_list(tmp_path / "crlf.txt")
    assert n == 4 and s.tolist() == [0, 2] and d.tolist() == [1, 3]
    (tmp_path / "empty.txt").write_text("# nothing\n")
    n, s, d = P.load_edge_list(tmp_path / "empty.txt")
    assert n == 0 and len(s) == 0 and len(d) == 0


def test_corrupt_containers_are_rejected(tmp_path):  # test_io.cpp:117-123
    (tmp_path / "bogus.bin").write_text("definitely not a matrix")
    with pytest.raises(P.IoError, match="not a FMAT1 file"):
        P.load_feature_matrix(tmp_path / "bogus.bin")
    with pytest.raises(P.IoError, match="not a CSR1 file"):
        P.load_csr(tmp_path / "bogus.bin")
    with pytest.raises(P.IoError, match="cannot open"):
        P.load_feature_matrix("/nonexistent/path")
    with pytest.raises(P.IoError, match="cannot open"):
        P.load_csr("/nonexistent/path")
    with pytest.raises(P.IoError, match="cannot open"):
        P.load_edge_list("/nonexistent/path")


def _csr_bytes(orient, rows, cols, indptr, indices, eids):
    return (b"CSR1" + bytes([orient]) + np.array([rows, cols, len(indices)], "<u8").tobytes() +
            b"".join(np.asarray(a, "<u8").tobytes() for a in (indptr, indices, eids)))


BAD_PAYLOADS = [
    # (indptr, indices, eids, validate() message, csr.cpp:111-156)
    ([1, 2, 3], [0, 1, 2], [0, 1, 2], "indptr[0] != 0"),
    ([0, 2, 1, 3], [0, 1, 2], [0, 1, 2], "indptr not monotone at row 2"),
    ([0, 1, 2], [0, 1, 2], [0, 1, 2], "indices/edge_ids length != indptr[num_rows] = 2"),
    ([0, 2, 3], [0, 7, 2], [0, 1, 2], "index out of range at nonzero 1"),
    ([0, 2, 3], [0, 1, 2], [0, 0, 2], "edge_ids not a permutation (at nonzero 1)"),
    ([0, 2, 3], [0, 1, 2], [0, 1, 5], "edge_ids not a permutation (at nonzero 2)"),
    ([0, 3, 3], [1, 0, 2], [0, 1, 2], "row 0 not sorted at nonzero 1"),
    ([0, 1, 3], [1, 2, 2], [0, 2, 1], "row 1 not sorted at nonzero 2"),
]


@pytest.mark.parametrize("indptr,indices,eids,why", BAD_PAYLOADS)
def test_invalid_csr_payload_message(tmp_path, indptr, indices, eids, why):
    path = tmp_path / "bad.csr"
    path.write_bytes(_csr_bytes(1, len(indptr) - 1, 3, indptr, indices, eids))
    with pytest.raises(P.IoError) as ei:
        P.load_csr(path)
    assert f"{path}: invalid CSR payload: {why}" in str(ei.value)
    if O.ref_available() and "length" not in why:  # the reference reads by the header's count
        with pytest.raises(O.OracleError) as ri:
            O.ref_load_csr(str(path))
        assert ri.value.status == O.IO_ERROR and why in str(ri.value)


def test_truncated_and_oversized_containers(tmp_path):
    good = _csr_bytes(1, 2, 3, [0, 2, 3], [0, 1, 2], [0, 1, 2])
    (tmp_path / "t.csr").write_bytes(good[:-4])
    with pytest.raises(P.IoError, match="truncated file"):
        P.load_csr(tmp_path / "t.csr")
    (tmp_path / "h.csr").write_bytes(good[:20])
    with pytest.raises(P.IoError, match="truncated file"):
        P.load_csr(tmp_path / "h.csr")
    wide = _csr_bytes(1, 2, 3, [0, 2, 3], [0, 1 << 32, 2], [0, 1, 2])
    (tmp_path / "w.csr").write_bytes(wide)
    with pytest.raises(P.IoError, match="id does not fit the configured id width"):
        P.load_csr(tmp_path / "w.csr")
    fm = b"FMAT1" + np.array([3, 4], "<u8").tobytes() + np.zeros(11, "<f4").tobytes()
    (tmp_path / "t.fmat").write_bytes(fm)
    with pytest.raises(P.IoError, match="truncated data section"):
        P.load_feature_matrix(tmp_path / "t.fmat")
    # trailing bytes are ignored, as by the reference
    (tmp_path / "x.csr").write_bytes(good + b"tail")
    assert P.load_csr(tmp_path / "x.csr")[1] == 2
    # empty graph / empty matrix
    P.save_csr(tmp_path / "e.csr", 0, 0, 0, np.zeros(1, np.uint32), [], [])
    o, r, c, ip, ix, ei = P.load_csr(tmp_path / "e.csr")
    assert (o, r, c, ip.tolist(), len(ix), len(ei)) == (0, 0, 0, [0], 0, 0)
    P.save_feature_matrix(tmp_path / "e.fmat", np.zeros((0, 7), np.float32))
    assert P.load_feature_matrix(tmp_path / "e.fmat").shape == (0, 7)


@needs_ref
@pytest.mark.parametrize("seed", [2, 5, 11])
def test_round_trip_against_the_reference(tmp_path, seed):
    """Files written by either side are read identically by the other."""
    src, dst = O.gen_rmat(300, 4000, 0.45, 0.25, 0.2, 0.1, seed)
    for orient in (P.SRC_MAJOR, P.DST_MAJOR):
        csr = P.build_csr(300, src, dst, orient)
        P.save_csr(tmp_path / "p.csr", orient, 300, 300, *csr)
        O.ref_save_csr(str(tmp_path / "r.csr"), orient, 300, 300, *csr)
        assert open(tmp_path / "p.csr", "rb").read() == open(tmp_path / "r.csr", "rb").read()
        got = O.ref_load_csr(str(tmp_path / "p.csr"))
        mine = P.load_csr(tmp_path / "r.csr")
        assert got[:3] == mine[:3] == (orient, 300, 300)
        assert all(_same(a, b) and _same(a, c) for a, b, c in zip(got[3:], mine[3:], csr))
    x = P.synth_normal(123, 17, seed)
    P.save_feature_matrix(tmp_path / "p.fmat", x)
    assert _same(O.ref_load_feature_matrix(str(tmp_path / "p.fmat")), x)
    O.ref_save_feature_matrix(str(tmp_path / "r.fmat"), x)
    assert _same(P.load_feature_matrix(tmp_path / "r.fmat"), x)
    P.save_edge_list(tmp_path / "p.txt", 300, src, dst)
    n, s, d = O.ref_load_edge_list(str(tmp_path / "p.txt"))
    assert n == 300 and _same(s, src) and _same(d, dst)
