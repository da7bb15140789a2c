"""Device-side canonical CSR build / transpose against the
host builder (itself pinned bit-identical to the reference's build_csr /
transpose, test_abi / test_oracle_pins): duplicates, self-loops, empty rows,
both orientations; and a handle made from device arrays computing the same
aggregation as one made from host arrays."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("kind", ["rmat", "er", "dups"])
def test_build_and_transpose_match_host(kind):
    import paper_2007_06354_b200 as P
    n = 5000
    if kind == "rmat":
        src, dst = P.synth_rmat(n, 80000, seed=3)
    elif kind == "er":
        src, dst = P.synth_er(n, 40000, -1.0, 4)
    else:  # heavy duplicates, self-loops, isolated nodes
        rng = np.random.default_rng(5)
        src = rng.integers(0, 50, 30000).astype(np.uint32)
        dst = rng.integers(0, 50, 30000).astype(np.uint32)
    s_d = torch.from_numpy(src.view(np.int32)).cuda()
    d_d = torch.from_numpy(dst.view(np.int32)).cuda()
    for orient in (P.DST_MAJOR, P.SRC_MAJOR):
        want = P.build_csr(n, src, dst, orient)
        got = P.build_csr_device(n, s_d, d_d, orient)
        for w, g in zip(want, got):
            assert np.array_equal(w, _u32(g))
        tw = P.transpose(n, n, *want)
        tg = P.transpose_device(n, n, *got)
        for w, g in zip(tw, tg):
            assert np.array_equal(w, _u32(g))


def test_empty_graph_device_build():
    import paper_2007_06354_b200 as P
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    ip, ix, ei = P.build_csr_device(10, e, e)
    assert _u32(ip).tolist() == [0] * 11 and ix.numel() == 0 and ei.numel() == 0


def test_graph_from_device_arrays_aggregates_identically():
    import paper_2007_06354_b200 as P
    n = 20000
    src, dst = P.synth_rmat(n, 300000, seed=7)
    host = P.Graph(*P.build_csr(n, src, dst, P.DST_MAJOR))
    dcsr = P.build_csr_device(n, torch.from_numpy(src.view(np.int32)).cuda(),
                              torch.from_numpy(dst.view(np.int32)).cuda())
    dev = P.Graph.from_device(*dcsr)
    assert dev.num_long_rows == host.num_long_rows
    x = torch.randn(n, 64, device="cuda")
    a = P.binary_reduce(host, "u_copy_add_v", u=x)
    b = P.binary_reduce(dev, "u_copy_add_v", u=x)
    assert torch.equal(a, b)
