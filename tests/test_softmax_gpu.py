"""Fused GAT edge softmax through the C-ABI: forward
against the f64 composite (oracle.softmax_attention), backward against the
f64 formula, rows summing to one, determinism, both edge orders, warp rows
and CTA (hub) rows, non-power-of-two head counts, and the errors."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _graph(seed=0):
    # R-MAT plus one 5000-edge hub so both the warp and the CTA kernels run
    n = 3000
    src, dst = O.gen_rmat(n, 30000, seed=seed)
    rng = np.random.default_rng(seed)
    hub = rng.integers(0, n, 5000).astype(np.uint32)
    src = np.concatenate([src, hub])
    dst = np.concatenate([dst, np.full(len(hub), 11, np.uint32)])
    return n, src, dst


@pytest.fixture(scope="module")
def G():
    import paper_2007_06354_b200 as P
    n, src, dst = _graph()
    ip, ix, ei = P.build_csr(n, src, dst, P.DST_MAJOR)
    g = P.Graph(ip, ix, ei, orientation=P.DST_MAJOR)
    assert np.diff(ip.astype(np.int64)).max() > 1024
    return P, g, n, src, dst, ei


@pytest.mark.parametrize("heads", [1, 3, 8, 32])
@pytest.mark.parametrize("by_pos", [False, True])
def test_edge_softmax_forward_backward(G, heads, by_pos):
    P, g, n, src, dst, ei = G
    rng = np.random.default_rng(heads)
    lg = (rng.standard_normal((len(src), heads)) * 3).astype(np.float32)
    ga = rng.standard_normal((len(src), heads)).astype(np.float32)
    want = O.softmax_attention(n, dst, lg)
    order = P.EDGE_BY_POS if by_pos else P.EDGE_BY_ID
    perm = ei.astype(np.int64) if by_pos else np.arange(len(src))  # row j <- edge eids[j]
    lg_d = torch.from_numpy(lg[perm]).cuda()
    a = P.edge_softmax(g, lg_d, e_order=order)
    a2 = P.edge_softmax(g, lg_d, e_order=order)
    assert torch.equal(a, a2)  # deterministic
    got = np.empty_like(lg)
    got[perm] = a.cpu().numpy()
    assert np.abs(got - want).max() <= 2e-6
    sums = np.zeros((n, heads))
    np.add.at(sums, dst, got.astype(np.float64))
    has = np.bincount(dst, minlength=n) > 0
    assert np.abs(sums[has] - 1.0).max() <= 1e-5
    # backward on the kernel's own a
    gl = P.edge_softmax_backward(g, a, torch.from_numpy(ga[perm]).cuda(), e_order=order)
    got_b = np.empty_like(lg)
    got_b[perm] = gl.cpu().numpy()
    want_b = O.softmax_attention_backward(n, dst, got, ga)
    err = np.abs(got_b - want_b) / np.maximum(np.abs(want_b), 1.0)
    assert err.max() <= 1e-5


def test_edge_softmax_errors(G):
    P, g, n, src, dst, ei = G
    with pytest.raises(P.ShapeError):
        P.edge_softmax(g, torch.zeros((len(src), 33), device="cuda"))
    with pytest.raises(P.ShapeError):
        P.edge_softmax(g, torch.zeros((len(src) - 1, 2), device="cuda"))
    ip, ix, ei2 = P.build_csr(n, src, dst, P.SRC_MAJOR)
    gs = P.Graph(ip, ix, ei2, orientation=P.SRC_MAJOR)
    with pytest.raises(P.ShapeError):
        P.edge_softmax(gs, torch.zeros((len(src), 2), device="cuda"))


def test_edge_softmax_autograd(G):
    from paper_2007_06354_b200 import autograd as A
    P, g, n, src, dst, ei = G
    ops = A.GraphOps(n, src, dst)
    torch.manual_seed(0)
    lg = torch.randn(len(src), 4, device="cuda", requires_grad=True)
    a = A.edge_softmax(ops, lg)
    da = torch.randn_like(a)
    (a * da).sum().backward()
    lr = lg.detach().double().requires_grad_(True)
    d = torch.from_numpy(dst.astype(np.int64)).cuda()
    mx = torch.full((n, 4), float("-inf"), dtype=torch.float64, device="cuda").scatter_reduce(
        0, d.unsqueeze(1).expand(-1, 4), lr, reduce="amax", include_self=True)
    ex = torch.exp(lr - mx[d])
    z = torch.zeros((n, 4), dtype=torch.float64, device="cuda").index_add_(0, d, ex)
    ar = ex / z[d]
    (ar * da.double()).sum().backward()
    assert (a.detach().double() - ar.detach()).abs().max().item() <= 2e-6
    assert ((lg.grad.double() - lr.grad).abs() / lr.grad.abs().clamp(min=1)).max().item() <= 1e-5
