"""Device loaders of the reference's containers:
gspmm_graph_load_csr1 (pinned ring -> narrow kernel -> device validate ->
handle), gspmm_fmat1_read_device, gspmm_validate_csr_device -- against the
reference-written fixtures, the host loaders and the oracle."""
import os

import numpy as np
import pytest

import gspmm_testutil  # noqa: F401
import paper_2007_06354_b200 as P
from oracle import oracle as O
from test_io import BAD_PAYLOADS, GOLD, _csr_bytes

pytestmark = pytest.mark.gpu


def _run_all(g, x, w):
    """Outputs that depend on every CSR array: indices (gather), edge ids
    (edge operand + arg_edge), indptr (row extents)."""
    import torch
    xs, ws = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    src_major = g.orientation == P.SRC_MAJOR
    cfg = (P.V, P.E, P.MUL, P.SUM, P.U) if src_major else (P.U, P.E, P.MUL, P.SUM, P.V)
    kw = dict(v=xs) if src_major else dict(u=xs)
    out = P.binary_reduce(g, cfg, e=ws, **kw)
    cmax = (P.V, P.NONE, P.COPY, P.MAX, P.U) if src_major else (P.U, P.NONE, P.COPY, P.MAX, P.V)
    mx, ao, ae = P.binary_reduce(g, cmax, want_arg_other=True, want_arg_edge=True, **kw)
    return [t.cpu().numpy() for t in (out, mx, ao, ae)]


@pytest.mark.parametrize("seed", [1, 8])
@pytest.mark.parametrize("tag", ["src", "dst"])
def test_load_csr1_fixture_to_device(seed, tag):
    path = os.path.join(GOLD, f"io_graph{seed}_{tag}.csr")
    o, r, c, indptr, indices, eids = P.load_csr(path)
    g_file = P.Graph.load(path)
    assert (g_file.orientation, g_file.num_rows, g_file.num_cols, g_file.num_edges) == \
        (o, r, c, len(indices))
    g_host = P.Graph(indptr, indices, eids, num_rows=r, num_cols=c, orientation=o)
    x = P.synth_uniform(c, 12, 5)
    w = P.synth_uniform(len(indices), 1, 6)
    for a, b in zip(_run_all(g_file, x, w), _run_all(g_host, x, w)):
        assert a.tobytes() == b.tobytes()
    # and the oracle on the edge list the reference wrote the file from
    exp = np.load(os.path.join(GOLD, "io_expected.npz"))
    og = O.Graph(r, exp[f"g{seed}_src"], exp[f"g{seed}_dst"])
    cfg = (O.V, O.E, O.MUL, O.SUM, O.U) if o == P.SRC_MAJOR else (O.U, O.E, O.MUL, O.SUM, O.V)
    want = O.binary_reduce(og, cfg, **({"v": x} if o == P.SRC_MAJOR else {"u": x}), e=w)
    assert _run_all(g_file, x, w)[0].tobytes() == want.tobytes()


def test_load_csr1_streams_several_ring_chunks(tmp_path):
    """9M edges: each 72 MB id array crosses the 32 MB ring slots twice."""
    import torch
    n, m = 200_000, 9_000_000
    src, dst = P.synth_rmat(n, m, 0.5, 0.2, 0.2, 0.1, 4)
    csr = P.build_csr(n, src, dst, P.DST_MAJOR)
    P.save_csr(tmp_path / "big.csr", P.DST_MAJOR, n, n, *csr)
    g = P.Graph.load(tmp_path / "big.csr")
    h = P.Graph(*csr, orientation=P.DST_MAJOR)
    x = torch.from_numpy(P.synth_uniform(n, 8, 1)).cuda()
    w = torch.from_numpy(P.synth_uniform(m, 1, 2)).cuda()
    cfg = (P.U, P.E, P.MUL, P.SUM, P.V)
    assert torch.equal(P.binary_reduce(g, cfg, u=x, e=w), P.binary_reduce(h, cfg, u=x, e=w))
    a = P.binary_reduce(g, (P.U, P.NONE, P.COPY, P.MAX, P.V), u=x, want_arg_edge=True)
    b = P.binary_reduce(h, (P.U, P.NONE, P.COPY, P.MAX, P.V), u=x, want_arg_edge=True)
    assert all(torch.equal(s, t) for s, t in zip(a, b) if s is not None)


@pytest.mark.parametrize("indptr,indices,eids,why", BAD_PAYLOADS)
def test_device_loader_rejects_invalid_payload(tmp_path, indptr, indices, eids, why):
    """The device checks report the reference's validate() message: the lowest
    offending nonzero, as its sequential scan does (csr.cpp:111-156)."""
    path = tmp_path / "bad.csr"
    path.write_bytes(_csr_bytes(1, len(indptr) - 1, 3, indptr, indices, eids))
    with pytest.raises(P.IoError) as ei:
        P.Graph.load(path)
    assert f"{path}: invalid CSR payload: {why}" in str(ei.value)


def test_device_loader_io_errors(tmp_path):
    good = _csr_bytes(1, 2, 3, [0, 2, 3], [0, 1, 2], [0, 1, 2])
    (tmp_path / "t.csr").write_bytes(good[:-4])
    with pytest.raises(P.IoError, match="truncated file"):
        P.Graph.load(tmp_path / "t.csr")
    (tmp_path / "w.csr").write_bytes(_csr_bytes(1, 2, 3, [0, 2, 3], [0, 1, 2], [0, 1 << 32, 2]))
    with pytest.raises(P.IoError, match="id does not fit the configured id width"):
        P.Graph.load(tmp_path / "w.csr")
    with pytest.raises(P.IoError, match="cannot open"):
        P.Graph.load("/nonexistent/path")
    (tmp_path / "bogus").write_text("definitely not a matrix")
    with pytest.raises(P.IoError, match="not a CSR1 file"):
        P.Graph.load(tmp_path / "bogus")
    with pytest.raises(P.IoError, match="not a FMAT1 file"):
        P.load_feature_matrix(tmp_path / "bogus", device=0)
    P.save_csr(tmp_path / "e.csr", 0, 0, 0, np.zeros(1, np.uint32), [], [])
    e = P.Graph.load(tmp_path / "e.csr")
    assert (e.num_rows, e.num_edges, e.orientation) == (0, 0, P.SRC_MAJOR)


def test_validate_csr_device_random_corruptions():
    """One corrupted element of a valid CSR: the device validation and the
    host validation (the reference's rules) agree on the message."""
    import torch
    rng = np.random.default_rng(7)
    n, m = 500, 6000
    src, dst = O.gen_rmat(n, m, 0.45, 0.25, 0.2, 0.1, 9)
    indptr, indices, eids = P.build_csr(n, src, dst, P.DST_MAJOR)
    dev = lambda a: torch.from_numpy(a.astype(np.int64)).to(torch.int32).cuda() \
        if a.max(initial=0) < 2**31 else torch.from_numpy(a.view(np.int32).copy()).cuda()  # noqa: E731
    P.validate_csr_device(n, n, dev(indptr), dev(indices), dev(eids))  # valid: no error
    for _ in range(40):
        ix, ei = indices.copy(), eids.copy()
        j = int(rng.integers(0, m))
        kind = int(rng.integers(0, 4))
        if kind == 0:
            ix[j] = n + int(rng.integers(0, 5))
        elif kind == 1:
            ei[j] = ei[int(rng.integers(0, m))]
        elif kind == 2:
            ei[j] = m + int(rng.integers(0, 9))
        else:
            k = int(rng.integers(0, m))
            ix[j], ix[k] = ix[k], ix[j]
        try:
            P.Graph(indptr, ix, ei, num_rows=n, num_cols=n, validate=True).close()
            want = None
        except P.StructureError as e:
            want = str(e).split(": ", 1)[1]
        try:
            P.validate_csr_device(n, n, dev(indptr), dev(ix), dev(ei))
            got = None
        except P.StructureError as e:
            got = str(e).split(": ", 1)[1]
        assert got == want, (kind, j)


@pytest.mark.parametrize("ld", [0, 8, 604])
def test_fmat1_to_device(tmp_path, ld):
    import torch
    path = os.path.join(GOLD, "io_feats.fmat")
    want = P.load_feature_matrix(path)
    if ld and ld < want.shape[1]:
        ld = want.shape[1] + 3
    got = P.load_feature_matrix(path, device=0, ld=ld)
    assert got.shape == want.shape and got.stride(0) == (ld or want.shape[1])
    assert got.cpu().numpy().tobytes() == want.tobytes()
    # a matrix larger than one ring slot (40 MB), padded rows
    x = P.synth_normal(17_000, 602, 3)
    P.save_feature_matrix(tmp_path / "big.fmat", x)
    d = P.load_feature_matrix(tmp_path / "big.fmat", device=0, ld=604)
    assert d.stride(0) == 604 and torch.equal(d.cpu(), torch.from_numpy(x))
