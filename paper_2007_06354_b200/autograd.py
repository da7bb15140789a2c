"""torch.autograd binding of the aggregation ops.

DGL-style message-passing ops whose forward AND backward run on the
library's sm_100a kernels (no torch compute on the hot path):

  op                  forward (dst-major)          backward
  copy_u_sum(x)       u_copy_add_v                 grad_x = v_copy_add_u(dy)           (src-major)
  copy_u_mean(x)      u_copy_add_v / deg           grad_x = v_copy_add_u(dy * 1/deg)   (src-major, fused scale)
  copy_u_max(x)       u_copy_max_v + argmax        grad_x = scatter of dy through the argmax
  copy_e_sum(w)       e_copy_add_v                 grad_w[e] = dy[dst(e)]              (out = E)
  u_mul_e_sum(x, w)   u_mul_e_add_v (w [E] or      grad_x = v_mul_e_add_u(dy, w)        (src-major)
                      [E, H] per head)             grad_w = u_dot_v_copy_e(x, dy)       (out = E, per head)
  u_add_v_sum(x, y)   u_add_v_add_v                grad_x = v_copy_add_u(dy); grad_y = v_copy_add_v(dy)
  u_mul_v_sum(x, y)   u_mul_v_add_v                grad_x = v_copy_add_u(dy * y);  grad_y = u_mul_v_add_v(x, dy)
  edge_softmax(l)     fused max/exp/sum/div        grad_l = a * (da - sum_row(a * da))  (fused)

u_mul_v's grad_x[u] = sum_v dy[v] * y[v] needs the product of two V rows per
edge, which the operator set cannot express in one call (lhs != rhs,
br_config.cpp:83-94); the binding forms dy*y with one torch elementwise
multiply (N x F, negligible next to the E x F gather) and aggregates it.

Inputs are fp32 CUDA tensors; the graph is given as (src, dst) edge lists and
both CSR orientations are built and uploaded once (`GraphOps`).  Forward
results are bit-identical to the reference's RowParallelSpmm; gradients are
the composed reference calls of SURVEY 8(a) a17.3-a17.5.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api as P

__all__ = ["GraphOps", "copy_u_sum", "copy_u_mean", "copy_u_max", "copy_e_sum", "u_mul_e_sum",
           "u_add_v_sum", "u_mul_v_sum", "edge_softmax"]


class GraphOps:
    """Both orientations of a square graph on one device, plus 1/in-degree."""

    def __init__(self, num_nodes, src, dst, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", 0)
        idx = dev.index if dev.index is not None else 0
        self.device = dev
        self.n = int(num_nodes)
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        self.m = len(src)
        dcsr = P.build_csr(self.n, src, dst, P.DST_MAJOR)
        scsr = P.transpose(self.n, self.n, *dcsr)
        self.fwd = P.Graph(*dcsr, orientation=P.DST_MAJOR, device=idx)
        self.bwd = P.Graph(*scsr, orientation=P.SRC_MAJOR, device=idx)
        deg = np.diff(dcsr[0].astype(np.int64)).astype(np.float32)
        inv = np.zeros(self.n, np.float32)
        nz = deg > 0
        inv[nz] = np.float32(1.0) / deg[nz]
        self.inv_deg = torch.from_numpy(inv).to(dev)


def _c(t):
    return t if t.is_contiguous() else t.contiguous()


class _CopyUSum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, x, mean):
        ctx.g, ctx.mean = g, mean
        cfg = (P.U, P.NONE, P.COPY, P.MEAN if mean else P.SUM, P.V)
        return P.binary_reduce(g.fwd, cfg, u=_c(x))

    @staticmethod
    def backward(ctx, dy):
        g = ctx.g
        kw = {"other_scale": g.inv_deg} if ctx.mean else {}
        gx = P.binary_reduce(g.bwd, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=_c(dy), **kw)
        return None, gx, None


class _CopyUMax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, x):
        out, arg, _ = P.binary_reduce(g.fwd, "u_copy_max_v", u=_c(x), want_arg_other=True)
        ctx.g, ctx.rows = g, x.shape[0]
        ctx.save_for_backward(arg)
        ctx.mark_non_differentiable(arg)
        return out

    @staticmethod
    def backward(ctx, dy):
        (arg,) = ctx.saved_tensors
        return None, P.argmax_backward(arg, _c(dy), ctx.rows)


class _CopyESum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, w):
        ctx.g = g
        return P.binary_reduce(g.fwd, (P.E, P.NONE, P.COPY, P.SUM, P.V), e=_c(w))

    @staticmethod
    def backward(ctx, dy):
        g = ctx.g
        gw = P.binary_reduce(g.fwd, (P.V, P.NONE, P.COPY, P.COPY_LAST, P.E), v=_c(dy))
        return None, gw


class _UMulESum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, x, w):
        w2 = w.reshape(w.shape[0], -1)
        heads = w2.shape[1]
        ctx.g, ctx.heads, ctx.wshape = g, heads, w.shape
        ctx.save_for_backward(x, w2)
        return P.binary_reduce(g.fwd, "u_mul_e_add_v", u=_c(x), e=_c(w2), heads=heads)

    @staticmethod
    def backward(ctx, dy):
        g, heads = ctx.g, ctx.heads
        x, w2 = ctx.saved_tensors
        dy = _c(dy)
        gx = gw = None
        if ctx.needs_input_grad[1]:
            gx = P.binary_reduce(g.bwd, "v_mul_e_add_u", v=dy, e=_c(w2), heads=heads)
        if ctx.needs_input_grad[2]:
            gw = P.binary_reduce(g.fwd, (P.U, P.V, P.DOT, P.COPY_LAST, P.E), u=_c(x), v=dy,
                                 heads=heads).reshape(ctx.wshape)
        return None, gx, gw


class _UAddVSum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, x, y):
        ctx.g = g
        return P.binary_reduce(g.fwd, "u_add_v_add_v", u=_c(x), v=_c(y))

    @staticmethod
    def backward(ctx, dy):
        g = ctx.g
        dy = _c(dy)
        gx = P.binary_reduce(g.bwd, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=dy)
        gy = P.binary_reduce(g.fwd, (P.V, P.NONE, P.COPY, P.SUM, P.V), v=dy)
        return None, gx, gy


class _UMulVSum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, x, y):
        ctx.g = g
        ctx.save_for_backward(x, y)
        return P.binary_reduce(g.fwd, "u_mul_v_add_v", u=_c(x), v=_c(y))

    @staticmethod
    def backward(ctx, dy):
        g = ctx.g
        x, y = ctx.saved_tensors
        dy = _c(dy)
        gx = P.binary_reduce(g.bwd, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=_c(dy * y))
        gy = P.binary_reduce(g.fwd, "u_mul_v_add_v", u=_c(x), v=dy)
        return None, gx, gy


class _EdgeSoftmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, logits):
        a = P.edge_softmax(g.fwd, _c(logits))
        ctx.g = g
        ctx.save_for_backward(a)
        return a

    @staticmethod
    def backward(ctx, da):
        (a,) = ctx.saved_tensors
        return None, P.edge_softmax_backward(ctx.g.fwd, a, _c(da))


def edge_softmax(g, logits):
    """GAT attention: softmax of logits [E, H] over the in-edges of each node."""
    return _EdgeSoftmax.apply(g, logits)


def copy_u_sum(g, x):
    return _CopyUSum.apply(g, x, False)


def copy_u_mean(g, x):
    return _CopyUSum.apply(g, x, True)


def copy_u_max(g, x):
    return _CopyUMax.apply(g, x)


def copy_e_sum(g, w):
    return _CopyESum.apply(g, w)


def u_mul_e_sum(g, x, w):
    """w: [E] / [E, 1] (scalar per edge) or [E, H] (per head; x width H*D)."""
    return _UMulESum.apply(g, x, w)


def u_add_v_sum(g, x, y):
    return _UAddVSum.apply(g, x, y)


def u_mul_v_sum(g, x, y):
    return _UMulVSum.apply(g, x, y)
