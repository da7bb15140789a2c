"""Python host API over the C-ABI, mirroring the reference's operator
interface (proj/include/gspmm/kernels.hpp): ``binary_reduce`` / ``copy_reduce``
with the same config names, operand roles, output shapes and error types.

Device tensors are torch CUDA tensors (torch is used for device memory and
streams only -- every byte of compute is the library's sm_100a kernels);
``*_host`` variants take numpy arrays and go through the C-ABI host entry.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi as A
from ._capi import (ADD, COPY, COPY_LAST, DIV, DOT, DST_MAJOR, E, EDGE_BY_ID, EDGE_BY_POS, MAX,
                    MEAN, MIN, MUL, NONE, PROD, SRC_MAJOR, SUB, SUM, U, V, check)

__all__ = [
    "Graph", "binary_reduce", "binary_reduce_host", "binary_reduce_host_async", "copy_reduce",
    "argmax_backward", "argmax_backward_host", "argmax_backward_host_async",
    "named_config", "validate_config", "required_orientation", "out_shape",
    "synth_rmat", "synth_er", "build_csr", "transpose", "synth_uniform", "synth_normal",
    "synth_gcn_weights", "synth_powerlaw", "launch_count", "edge_softmax", "edge_softmax_backward",
    "build_csr_device", "transpose_device",
    "load_feature_matrix", "save_feature_matrix", "load_csr", "save_csr", "load_graph",
    "validate_csr_device", "load_edge_list", "save_edge_list",
]


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a):
    return None if a is None else a.ctypes.data


# ------------------------------------------------------------------ config
def named_config(name):
    """named_config (br_config.cpp:96-131)."""
    cfg = A.Config()
    check(A.LIB.gspmm_named_config(name.encode(), C.byref(cfg)), f"named_config({name!r})")
    return cfg


def as_config(cfg):
    if isinstance(cfg, A.Config):
        return cfg
    if isinstance(cfg, str):
        return named_config(cfg)
    return A.Config(*cfg)


def validate_config(cfg):
    check(A.LIB.gspmm_validate_config(C.byref(as_config(cfg))), "validate_config")


def required_orientation(strategy, out):
    o = A.LIB.gspmm_required_orientation(strategy, out)
    if o < 0:
        raise A.ConfigError(A.last_error())
    return o


def launch_count():
    return A.LIB.gspmm_launch_count()


# ------------------------------------------------------------------- graph
class Graph:
    """Device-resident CsrGraph (csr.hpp:37-54) plus the device row plan.

    ``indptr/indices/edge_ids`` are host arrays in the reference's canonical
    CSR order; they are uploaded once.  ``orientation`` is DST_MAJOR (rows are
    destinations, the forward view) or SRC_MAJOR (the transposed view used by
    out=U configs and the backward)."""

    def __init__(self, indptr, indices, edge_ids, num_rows=None, num_cols=None,
                 orientation=DST_MAJOR, device=0, validate=False):
        indptr, indices, edge_ids = _u32(indptr), _u32(indices), _u32(edge_ids)
        self.num_rows = len(indptr) - 1 if num_rows is None else int(num_rows)
        self.num_cols = self.num_rows if num_cols is None else int(num_cols)
        self.orientation = orientation
        self.device = device
        self.num_edges = int(indptr[-1]) if len(indptr) else 0
        h = C.c_void_p()
        check(A.LIB.gspmm_graph_create(device, orientation, self.num_rows, self.num_cols,
                                       _ptr(indptr), _ptr(indices), _ptr(edge_ids),
                                       1 if validate else 0, C.byref(h)), "graph_create")
        self._h = h
        nl = C.c_uint32()
        check(A.LIB.gspmm_graph_info(h, None, None, None, None, C.byref(nl)))
        self.num_long_rows = nl.value

    @classmethod
    def from_device(cls, indptr, indices, edge_ids, num_rows=None, num_cols=None,
                    orientation=DST_MAJOR):
        """Handle over a canonical CSR held in CUDA tensors (int32 storage of
        the u32 arrays, e.g. from ``build_csr_device``): no host round trip
        except indptr for the row plan."""
        self = cls.__new__(cls)
        self.num_rows = indptr.numel() - 1 if num_rows is None else int(num_rows)
        self.num_cols = self.num_rows if num_cols is None else int(num_cols)
        self.orientation = orientation
        self.device = indptr.device.index or 0
        self.num_edges = int(indices.numel())
        h = C.c_void_p()
        check(A.LIB.gspmm_graph_create_device(self.device, orientation, self.num_rows, self.num_cols,
                                              indptr.data_ptr(), indices.data_ptr(),
                                              edge_ids.data_ptr(), C.byref(h)),
              "graph_create_device")
        self._h = h
        nl = C.c_uint32()
        check(A.LIB.gspmm_graph_info(h, None, None, None, None, C.byref(nl)))
        self.num_long_rows = nl.value
        return self

    @classmethod
    def load(cls, path, device=0):
        """load_csr (io.cpp:183-205) of a CSR1 container straight to a device
        handle: the payload streams through a pinned ring, is narrowed to
        32-bit ids and validated on the device (csr.cpp:111-156)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        check(A.LIB.gspmm_graph_load_csr1(_path(path), device, C.byref(h)), "load_csr")
        self._h = h
        o, r, c_, m, nl = C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint32()
        check(A.LIB.gspmm_graph_info(h, C.byref(o), C.byref(r), C.byref(c_), C.byref(m),
                                     C.byref(nl)))
        self.orientation, self.num_rows, self.num_cols = o.value, r.value, c_.value
        self.num_edges, self.num_long_rows, self.device = m.value, nl.value, device
        return self

    @property
    def handle(self):
        if self._h is None:
            raise A.ArgumentError("graph handle already closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None:
            A.LIB.gspmm_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def entity_rows(self, ent):
        src_major = self.orientation == SRC_MAJOR
        if ent == U:
            return self.num_rows if src_major else self.num_cols
        if ent == V:
            return self.num_cols if src_major else self.num_rows
        return self.num_edges

    def set_source_blocks(self, nblocks):
        """Source blocking (the paper's Alg. 3 / BlockPlan): 0 = automatic
        (default), 1 = never, >= 2 = that many neighbour-id blocks, folded
        pass by pass into the partial rows so each pass's gathered rows fit
        in L2.  Results are bit-identical either way."""
        check(A.LIB.gspmm_graph_set_source_blocks(self.handle, int(nblocks)), "set_source_blocks")
        return self

    def set_plan(self, seg_cost=0, long_threshold=0, unit_cols=0, kernel=0, long_ctas=0,
                 split_edges=0):
        """Rebuild the device plan (gspmm_graph_set_plan): segment-unit cost,
        a fixed long-row threshold, a fixed long-row unit width (multiple of
        4, <= 512), kernel=1 for the register kernel on every call (2: planned kernels with
        the segment kernel a programmatic dependent of the long-row kernel), long_ctas
        = N to run the long-row units concurrently with the segments on N
        CTAs.  0 = the default of each.  split_edges: 0 = long rows of max /
        min reductions are folded as chunks of 512 edges combined in chunk
        order (exact: the reference's bits), sums stay sequential; 1 = never
        split; N >= 16 = split every reduction at N.  Results never depend
        on the plan, except the sums of long rows under split_edges >= 16
        (deterministic, but up to ~1e-3 from the reference's sequential
        fold, whose own rounding is that large: outside the parity
        contract)."""
        p = A.Plan(seg_cost, long_threshold, unit_cols, kernel, long_ctas, split_edges)
        check(A.LIB.gspmm_graph_set_plan(self.handle, C.byref(p)), "set_plan")
        nl = C.c_uint32()
        check(A.LIB.gspmm_graph_info(self.handle, None, None, None, None, C.byref(nl)))
        self.num_long_rows = nl.value
        return self

    def permute_edges(self, e, stream=None):
        """Edge operand in edge-id order -> this handle's CSR position order
        (device, untimed setup like the reference's BlockPlan)."""
        import torch
        e2 = e.reshape(e.shape[0], -1)
        # one row per CSR position of this handle (a shard's edge ids index a
        # larger, global edge operand)
        out = torch.empty((self.num_edges, e2.shape[1]), dtype=e2.dtype, device=e2.device)
        check(A.LIB.gspmm_graph_permute_edges(self.handle, e2.data_ptr(), e2.shape[1],
                                              e2.stride(0), out.data_ptr(), out.stride(0),
                                              _stream(stream, e2)), "permute_edges")
        return out


# -------------------------------------------------------------- operands
def _stream(stream, ref_tensor=None):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    import torch
    dev = ref_tensor.device if ref_tensor is not None else None
    return torch.cuda.current_stream(dev).cuda_stream


def _dev_mat(t, edge_order=EDGE_BY_ID):
    if t is None:
        return None
    import torch
    if t.dtype != torch.float32 or not t.is_cuda:
        raise A.ShapeError("operands must be float32 CUDA tensors")
    t2 = t.reshape(t.shape[0], -1) if t.dim() != 2 else t
    if t2.shape[1] > 1 and t2.stride(1) != 1:
        raise A.ShapeError("operand rows must be contiguous")
    if t2.shape[0] > 1 and t2.stride(0) < t2.shape[1]:
        # an expanded / overlapping view (e.g. bias.expand(n, d), stride 0)
        # would be read as n distinct rows
        raise A.ShapeError("operand rows must not overlap (expanded views are not supported; "
                           "pass a width-1 operand to broadcast, or materialise it)")
    ld = t2.stride(0) if t2.shape[0] > 1 else t2.shape[1]
    m = A.Mat(t2.data_ptr(), t2.shape[0], t2.shape[1], ld, edge_order)
    m._keep = t2
    return m


def _host_mat(a, edge_order=EDGE_BY_ID):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    m = A.Mat(a.ctypes.data if a.size else 1, a.shape[0], a.shape[1], a.shape[1], edge_order)
    m._keep = a
    return m


def _opts(heads=1, arg_other=None, arg_edge=None, other_scale=None, arg_ld=0, out2=None,
          out2_ld=0, reduce2=SUM):
    o = A.Options()
    o.heads = heads
    o.arg_other = arg_other
    o.arg_edge = arg_edge
    o.arg_ld = arg_ld
    o.other_scale = other_scale
    o.out2 = out2
    o.out2_ld = out2_ld
    o.reduce2 = reduce2
    return o


def _ref(m):
    return C.byref(m) if m is not None else None


def out_shape(graph, cfg, u=None, v=None, e=None, heads=1, host=False):
    cfg = as_config(cfg)
    mk = _host_mat if host else _dev_mat
    mu, mv, me = mk(u), mk(v), mk(e)
    r, d = C.c_int64(), C.c_int64()
    check(A.LIB.gspmm_out_shape(graph.handle, C.byref(cfg), _ref(mu), _ref(mv), _ref(me),
                                C.byref(_opts(heads)), C.byref(r), C.byref(d)), "binary_reduce")
    return r.value, d.value


# ----------------------------------------------------------------- compute
def _check_out(t, rows, dim, dtype, dev, what):
    import torch
    if t.dtype != dtype or not t.is_cuda or t.device != dev:
        raise A.ShapeError(f"{what} must be a {dtype} tensor on {dev}")
    t2 = t if t.dim() == 2 else t.reshape(rows, -1)
    if tuple(t2.shape) != (rows, dim) or (dim > 1 and t2.stride(1) != 1) or \
            (rows > 1 and t2.stride(0) < dim):
        raise A.ShapeError(f"{what} must be a row-major {rows} x {dim} view "
                           f"(got shape {tuple(t.shape)}, strides {tuple(t.stride())})")
    return t2


def binary_reduce(graph, cfg, u=None, v=None, e=None, *, out=None, e_order=EDGE_BY_ID,
                  want_arg_other=False, want_arg_edge=False, heads=1, other_scale=None,
                  arg_other_out=None, arg_edge_out=None, out2=None, reduce2=SUM, stream=None):
    """binary_reduce (kernels.hpp:60-64) on device tensors.

    Returns ``out`` (allocated when not given) or ``(out, arg_other,
    arg_edge)`` when an argmax output is requested (``arg_*_out``: caller
    buffers for them).  ``out2``: a second output receiving the same config
    with reducer ``reduce2`` (SUM or MEAN), fused into the same gather for
    copy + max/min (config 3's max and mean forward)."""
    import torch
    cfg = as_config(cfg)
    mu, mv, me = _dev_mat(u), _dev_mat(v), _dev_mat(e, e_order)
    ref_t = next(t for t in (u, v, e) if t is not None) if any(
        t is not None for t in (u, v, e)) else None
    rows, dim = out_shape(graph, cfg, u, v, e, heads)
    dev = ref_t.device if ref_t is not None else torch.device("cuda", graph.device)
    if out is None:
        out = torch.empty((rows, dim), dtype=torch.float32, device=dev)
    o2 = _check_out(out, rows, dim, torch.float32, dev, "out")
    mo = A.Out(o2.data_ptr(), rows, dim, o2.stride(0) if rows > 1 else dim)
    want_arg_other = want_arg_other or arg_other_out is not None
    want_arg_edge = want_arg_edge or arg_edge_out is not None
    ao, ae = arg_other_out, arg_edge_out
    if want_arg_other and ao is None:
        ao = torch.empty((rows, dim), dtype=torch.int32, device=dev)
    if want_arg_edge and ae is None:
        ae = torch.empty((rows, dim), dtype=torch.int32, device=dev)
    for t, what in ((ao, "arg_other"), (ae, "arg_edge")):
        if t is not None and (not t.is_contiguous() or
                              _check_out(t, rows, dim, torch.int32, dev, what) is None):
            raise A.ShapeError(f"{what} must be a contiguous int32 {rows} x {dim} tensor")
    if other_scale is not None:
        if other_scale.dtype != torch.float32 or other_scale.device != dev or \
                not other_scale.is_contiguous():
            raise A.ShapeError("other_scale must be a contiguous float32 tensor on the "
                               "operands' device")
    o2 = None
    if out2 is not None:
        o2 = _check_out(out2, rows, dim, torch.float32, dev, "out2")
    opts = _opts(heads, ao.data_ptr() if ao is not None else None,
                 ae.data_ptr() if ae is not None else None,
                 other_scale.data_ptr() if other_scale is not None else None,
                 out2=o2.data_ptr() if o2 is not None else None,
                 out2_ld=(o2.stride(0) if rows > 1 else dim) if o2 is not None else 0,
                 reduce2=reduce2)
    check(A.LIB.gspmm_binary_reduce_ex(graph.handle, C.byref(cfg), _ref(mu), _ref(mv), _ref(me),
                                       C.byref(mo), C.byref(opts), _stream(stream, ref_t)),
          "binary_reduce")
    if want_arg_other or want_arg_edge:
        return out, ao, ae
    return out


def copy_reduce(graph, src, reduce, *, out=None, stream=None):
    """copy_reduce (kernels.hpp:71-73): source entity inferred from rows."""
    import torch
    ms = _dev_mat(src)
    rows = graph.entity_rows(V)
    if out is None:
        out = torch.empty((rows, ms.dim), dtype=torch.float32, device=src.device)
    mo = A.Out(out.data_ptr(), rows, ms.dim, out.stride(0))
    check(A.LIB.gspmm_copy_reduce(graph.handle, C.byref(ms), reduce, C.byref(mo),
                                  _stream(stream, src)), "copy_reduce")
    return out


def argmax_backward(arg, grad_out, src_rows, *, out=None, src_lo=0, stream=None):
    """grad_src[arg[r,f] - src_lo, f] += grad_out[r,f] for the source rows
    [src_lo, src_lo + src_rows) (f64 accumulate, fp32 result)."""
    import torch
    rows, dim = arg.shape
    if arg.dtype != torch.int32 or grad_out.dtype != torch.float32 or \
            tuple(grad_out.shape) != (rows, dim) or arg.stride(1) != 1 or grad_out.stride(1) != 1:
        raise A.ShapeError("argmax_backward: arg int32 and grad_out float32 [rows x dim] rows")
    if out is None:
        out = torch.empty((src_rows, dim), dtype=torch.float32, device=grad_out.device)
    _check_out(out, src_rows, dim, torch.float32, grad_out.device, "out")
    check(A.LIB.gspmm_argmax_backward_range(arg.data_ptr(), rows, dim, arg.stride(0),
                                            grad_out.data_ptr(), grad_out.stride(0),
                                            out.data_ptr(), src_lo, src_rows, out.stride(0),
                                            _stream(stream, grad_out)),
          "argmax_backward")
    return out


def argmax_backward_host(arg, grad_out, src_rows, *, out=None, device=0, stream=None):
    """argmax_backward on host arrays (gspmm_argmax_backward_host)."""
    arg = np.ascontiguousarray(arg, np.int32)
    grad_out = np.ascontiguousarray(grad_out, np.float32)
    rows, dim = arg.shape
    if out is None:
        out = np.empty((src_rows, dim), np.float32)
    check(A.LIB.gspmm_argmax_backward_host(arg.ctypes.data, rows, dim, grad_out.ctypes.data,
                                           out.ctypes.data, src_rows, device, stream or None),
          "argmax_backward_host")
    return out


def argmax_backward_host_async(arg, grad_out, src_rows, *, out, device=0, stream,
                               wait_event=None, upload_event=None):
    """Enqueue-only argmax_backward_host: pinned arrays, valid after `stream`
    synchronizes."""
    rows, dim = arg.shape
    if arg.dtype != np.int32 or grad_out.dtype != np.float32 or out.shape != (src_rows, dim) \
            or not (arg.flags.c_contiguous and grad_out.flags.c_contiguous and
                    out.flags.c_contiguous):
        raise A.ShapeError("argmax_backward_host_async: contiguous int32 / float32 arrays")
    ev = lambda x: None if x is None else (x if isinstance(x, int) else x.cuda_event)  # noqa: E731
    st = stream if isinstance(stream, int) else stream.cuda_stream
    check(A.LIB.gspmm_argmax_backward_host_async(arg.ctypes.data, rows, dim,
                                                 grad_out.ctypes.data, out.ctypes.data,
                                                 src_rows, device, st, ev(wait_event),
                                                 ev(upload_event)),
          "argmax_backward_host_async")
    return out


def edge_softmax(graph, logits, *, out=None, e_order=EDGE_BY_ID, stream=None):
    """Fused GAT edge softmax over in-edges (dst-major handle): logits [E, H]
    (H <= 32) in `e_order`; returns a [E, H] in the same order."""
    import torch
    lg = logits if logits.dim() == 2 else logits.reshape(-1, 1)
    if out is None:
        out = torch.empty(lg.shape, dtype=torch.float32, device=lg.device)
    o2 = out if out.dim() == 2 else out.reshape(-1, 1)
    mo = A.Out(o2.data_ptr(), o2.shape[0], o2.shape[1], o2.stride(0))
    check(A.LIB.gspmm_edge_softmax(graph.handle, C.byref(_dev_mat(lg, e_order)), C.byref(mo),
                                   _stream(stream, lg)), "edge_softmax")
    return out


def edge_softmax_backward(graph, a, grad_a, *, out=None, e_order=EDGE_BY_ID, stream=None):
    """grad_logits = a * (grad_a - sum over the row of a * grad_a)."""
    import torch
    a2 = a if a.dim() == 2 else a.reshape(-1, 1)
    g2 = grad_a if grad_a.dim() == 2 else grad_a.reshape(-1, 1)
    if out is None:
        out = torch.empty(a2.shape, dtype=torch.float32, device=a2.device)
    o2 = out if out.dim() == 2 else out.reshape(-1, 1)
    mo = A.Out(o2.data_ptr(), o2.shape[0], o2.shape[1], o2.stride(0))
    check(A.LIB.gspmm_edge_softmax_backward(graph.handle, C.byref(_dev_mat(a2, e_order)),
                                            C.byref(_dev_mat(g2, e_order)), C.byref(mo),
                                            _stream(stream, a2)), "edge_softmax_backward")
    return out


def binary_reduce_host(graph, cfg, u=None, v=None, e=None, *, out=None, want_arg_other=False,
                       want_arg_edge=False, heads=1, stream=None, e_order=EDGE_BY_ID):
    """The reference's synchronous call shape: numpy in, numpy out, through
    the C-ABI host entry (H2D, kernel, D2H)."""
    cfg = as_config(cfg)
    mu, mv, me = _host_mat(u), _host_mat(v), _host_mat(e, e_order)
    rows, dim = out_shape(graph, cfg, u, v, e, heads, host=True)
    if out is None:
        out = np.empty((rows, dim), np.float32)
    mo = A.Out(out.ctypes.data, rows, dim, dim)
    ao = np.empty((rows, dim), np.int32) if want_arg_other else None
    ae = np.empty((rows, dim), np.int32) if want_arg_edge else None
    opts = _opts(heads, _ptr(ao), _ptr(ae))
    check(A.LIB.gspmm_binary_reduce_host(graph.handle, C.byref(cfg), _ref(mu), _ref(mv), _ref(me),
                                         C.byref(mo), C.byref(opts), stream or None),
          "binary_reduce_host")
    if want_arg_other or want_arg_edge:
        return out, ao, ae
    return out


def binary_reduce_host_async(graph, cfg, u=None, v=None, e=None, *, out, heads=1, stream,
                             wait_event=None, upload_event=None, e_order=EDGE_BY_ID,
                             arg_other=None, other_scale=None, out2=None, reduce2=SUM):
    """Enqueue-only form of binary_reduce_host (gspmm_binary_reduce_host_async):
    pinned host arrays in and out (``arg_other``: an int32 output array for
    the argmax; ``other_scale``: a host float32 array over the gathered
    nodes), valid once `stream` synchronizes; uploads start after
    `wait_event` and `upload_event` is recorded when they are done
    (torch.cuda.Event objects or raw handles)."""
    cfg = as_config(cfg)
    mu, mv, me = _host_mat(u), _host_mat(v), _host_mat(e, e_order)
    rows, dim = out_shape(graph, cfg, u, v, e, heads, host=True)
    if out.shape != (rows, dim) or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise A.ShapeError(f"out must be a contiguous float32 {rows} x {dim} array")
    if arg_other is not None and (arg_other.shape != (rows, dim) or arg_other.dtype != np.int32
                                  or not arg_other.flags.c_contiguous):
        raise A.ShapeError(f"arg_other must be a contiguous int32 {rows} x {dim} array")
    if other_scale is not None and (other_scale.dtype != np.float32 or
                                    other_scale.shape != (graph.num_cols,) or
                                    not other_scale.flags.c_contiguous):
        raise A.ShapeError(f"other_scale must be a float32 array of {graph.num_cols}")
    if out2 is not None and (out2.shape != (rows, dim) or out2.dtype != np.float32 or
                             not out2.flags.c_contiguous):
        raise A.ShapeError(f"out2 must be a contiguous float32 {rows} x {dim} array")
    mo = A.Out(out.ctypes.data, rows, dim, dim)
    opts = _opts(heads, _ptr(arg_other), None, _ptr(other_scale), out2=_ptr(out2),
                 reduce2=reduce2)
    ev = lambda x: None if x is None else (x if isinstance(x, int) else x.cuda_event)  # noqa: E731
    st = stream if isinstance(stream, int) else stream.cuda_stream
    check(A.LIB.gspmm_binary_reduce_host_async(graph.handle, C.byref(cfg), _ref(mu), _ref(mv),
                                               _ref(me), C.byref(mo), C.byref(opts), st,
                                               ev(wait_event), ev(upload_event)),
          "binary_reduce_host_async")
    return out


# ------------------------------------------------- synthesis and CSR build
def synth_rmat(n, num_edges, a=0.57, b=0.19, c=0.19, d=0.05, seed=0, threads=0):
    src = np.empty(max(num_edges, 1), np.uint32)
    dst = np.empty(max(num_edges, 1), np.uint32)
    m = A.LIB.gspmm_synth_rmat(n, num_edges, a, b, c, d, seed, _ptr(src), _ptr(dst), threads)
    if m < 0:
        raise A.ConfigError("rmat: could not place an edge inside the node range")
    return src[:num_edges], dst[:num_edges]


def synth_er(n, num_edges=0, prob=-1.0, seed=0):
    ps, pd = C.c_void_p(), C.c_void_p()
    m = A.LIB.gspmm_synth_er(n, num_edges, prob, seed, C.byref(ps), C.byref(pd))
    cap = max(m, 1)
    src = np.ctypeslib.as_array(C.cast(ps, C.POINTER(C.c_uint32)), shape=(cap,))[:m].copy()
    dst = np.ctypeslib.as_array(C.cast(pd, C.POINTER(C.c_uint32)), shape=(cap,))[:m].copy()
    A.LIB.gspmm_free(ps)
    A.LIB.gspmm_free(pd)
    return src, dst


def build_csr(n, src, dst, orientation=DST_MAJOR, threads=0):
    src, dst = _u32(src), _u32(dst)
    m = len(src)
    indptr = np.empty(n + 1, np.uint32)
    indices = np.empty(max(m, 1), np.uint32)
    eids = np.empty(max(m, 1), np.uint32)
    check(A.LIB.gspmm_build_csr(n, m, _ptr(src), _ptr(dst), orientation, _ptr(indptr),
                                _ptr(indices), _ptr(eids), threads), "build_csr")
    return indptr, indices[:m], eids[:m]


def transpose(num_rows, num_cols, indptr, indices, eids, threads=0):
    indptr, indices, eids = _u32(indptr), _u32(indices), _u32(eids)
    m = int(indptr[-1])
    t_indptr = np.empty(num_cols + 1, np.uint32)
    t_indices = np.empty(max(m, 1), np.uint32)
    t_eids = np.empty(max(m, 1), np.uint32)
    check(A.LIB.gspmm_transpose(num_rows, num_cols, _ptr(indptr), _ptr(indices), _ptr(eids),
                                _ptr(t_indptr), _ptr(t_indices), _ptr(t_eids), threads),
          "transpose")
    return t_indptr, t_indices[:m], t_eids[:m]


def build_csr_device(n, src, dst, orientation=DST_MAJOR, stream=None):
    """Canonical CSR on the device from CUDA edge lists (int32/uint32 storage,
    edge-id order); returns (indptr, indices, edge_ids) as int32 CUDA
    tensors holding the u32 values.  Bit-identical to ``build_csr``."""
    import torch
    m = src.numel()
    dev = src.device
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    eids = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    check(A.LIB.gspmm_build_csr_device(n, m, src.data_ptr(), dst.data_ptr(), orientation,
                                       indptr.data_ptr(), indices.data_ptr(), eids.data_ptr(),
                                       _stream(stream, src)), "build_csr_device")
    return indptr, indices, eids


def transpose_device(num_rows, num_cols, indptr, indices, eids, stream=None):
    """Device transpose of a canonical CSR (int32 CUDA tensors)."""
    import torch
    m = indices.numel()
    dev = indptr.device
    t_indptr = torch.empty(num_cols + 1, dtype=torch.int32, device=dev)
    t_indices = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    t_eids = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    check(A.LIB.gspmm_transpose_device(num_rows, num_cols, m, indptr.data_ptr(),
                                       indices.data_ptr(), eids.data_ptr(), t_indptr.data_ptr(),
                                       t_indices.data_ptr(), t_eids.data_ptr(),
                                       _stream(stream, indptr)), "transpose_device")
    return t_indptr, t_indices, t_eids


def synth_uniform(rows, dim, seed, threads=0, out=None):
    out = np.empty((rows, dim), np.float32) if out is None else out
    A.LIB.gspmm_synth_uniform(rows * dim, seed, out.ctypes.data, threads)
    return out


def synth_normal(rows, dim, seed, threads=0, out=None):
    out = np.empty((rows, dim), np.float32) if out is None else out
    A.LIB.gspmm_synth_normal(rows * dim, seed, out.ctypes.data, threads)
    return out


def synth_powerlaw(n, d_min, d_max, seed=0, threads=0):
    """Power-law in-degree graph (cfg5, see gspmm_synth_powerlaw)."""
    m = A.LIB.gspmm_synth_powerlaw(n, d_min, d_max, seed, None, None, threads)
    if m < 0:
        raise A.ConfigError("powerlaw: bad parameters")
    src = np.empty(max(m, 1), np.uint32)
    dst = np.empty(max(m, 1), np.uint32)
    A.LIB.gspmm_synth_powerlaw(n, d_min, d_max, seed, _ptr(src), _ptr(dst), threads)
    return src[:m], dst[:m]


def synth_gcn_weights(n, src, dst, threads=0):
    src, dst = _u32(src), _u32(dst)
    w = np.empty((len(src), 1), np.float32)
    A.LIB.gspmm_synth_gcn_weights(n, len(src), _ptr(src), _ptr(dst), w.ctypes.data, threads)
    return w


# ------------------------------------------------- file containers (io.hpp)
def _path(path):
    import os
    return os.fsencode(path)


def load_feature_matrix(path, device=None, ld=0):
    """load_feature_matrix (io.cpp:149-166) of a FMAT1 container.  device None:
    a numpy array; else a CUDA tensor on that device, streamed through a
    pinned ring (``ld`` > dim pads the device rows, e.g. 604 for 602 columns;
    the view returned is [rows, dim])."""
    rows, dim = C.c_int64(), C.c_int64()
    check(A.LIB.gspmm_fmat1_info(_path(path), C.byref(rows), C.byref(dim)), "load_feature_matrix")
    rows, dim = rows.value, dim.value
    if device is None:
        out = np.empty((rows, dim), np.float32)
        check(A.LIB.gspmm_fmat1_read(_path(path), _ptr(out), 0), "load_feature_matrix")
        return out
    import torch
    ld = ld or dim
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    buf = torch.empty((rows, ld), dtype=torch.float32, device=dev)
    check(A.LIB.gspmm_fmat1_read_device(_path(path), dev.index or 0, buf.data_ptr(), ld,
                                        _stream(None, buf)), "load_feature_matrix")
    return buf[:, :dim]


def save_feature_matrix(path, a):
    """save_feature_matrix (io.cpp:137-147) from a 2-D float32 host array."""
    a = np.asarray(a, np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2:
        raise A.ArgumentError("save_feature_matrix: a 2-D matrix is required")
    if a.size and (a.strides[1] != 4 or a.strides[0] % 4 or a.strides[0] < 4 * a.shape[1]):
        a = np.ascontiguousarray(a)
    ld = a.strides[0] // 4 if a.shape[0] > 1 and a.size else a.shape[1]
    check(A.LIB.gspmm_fmat1_write(_path(path), _ptr(a), a.shape[0], a.shape[1], ld),
          "save_feature_matrix")


def load_csr(path):
    """load_csr (io.cpp:183-205) into host arrays: (orientation, num_rows,
    num_cols, indptr, indices, edge_ids), validated."""
    o, r, c_, m = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(A.LIB.gspmm_csr1_info(_path(path), C.byref(o), C.byref(r), C.byref(c_), C.byref(m)),
          "load_csr")
    indptr = np.empty(r.value + 1, np.uint32)
    indices = np.empty(max(m.value, 1), np.uint32)
    eids = np.empty(max(m.value, 1), np.uint32)
    check(A.LIB.gspmm_csr1_read(_path(path), _ptr(indptr), _ptr(indices), _ptr(eids)), "load_csr")
    return o.value, r.value, c_.value, indptr, indices[:m.value], eids[:m.value]


def save_csr(path, orientation, num_rows, num_cols, indptr, indices, edge_ids):
    """save_csr (io.cpp:168-181)."""
    indptr, indices, edge_ids = _u32(indptr), _u32(indices), _u32(edge_ids)
    check(A.LIB.gspmm_csr1_write(_path(path), orientation, num_rows, num_cols, _ptr(indptr),
                                 _ptr(indices), _ptr(edge_ids)), "save_csr")


def load_graph(path, device=0):
    """A CSR1 container as a device Graph (``Graph.load``)."""
    return Graph.load(path, device)


def validate_csr_device(num_rows, num_cols, indptr, indices, edge_ids, stream=None):
    """validate() (csr.cpp:111-156) of a device CSR (int32 CUDA tensors);
    raises StructureError with the reference's message."""
    check(A.LIB.gspmm_validate_csr_device(indptr.device.index or 0, num_rows, num_cols,
                                          indptr.data_ptr(), indices.data_ptr(),
                                          edge_ids.data_ptr(), _stream(stream, indptr)),
          "validate")


def load_edge_list(path):
    """load_edge_list (io.cpp:80-127): (num_nodes, src, dst)."""
    n, m, ps, pd = C.c_uint32(), C.c_uint64(), C.c_void_p(), C.c_void_p()
    check(A.LIB.gspmm_edge_list_read(_path(path), C.byref(n), C.byref(m), C.byref(ps),
                                     C.byref(pd)), "load_edge_list")
    cap = max(m.value, 1)
    src = np.ctypeslib.as_array(C.cast(ps, C.POINTER(C.c_uint32)), shape=(cap,))[:m.value].copy()
    dst = np.ctypeslib.as_array(C.cast(pd, C.POINTER(C.c_uint32)), shape=(cap,))[:m.value].copy()
    A.LIB.gspmm_free(ps)
    A.LIB.gspmm_free(pd)
    return n.value, src, dst


def save_edge_list(path, num_nodes, src, dst):
    """save_edge_list (io.cpp:129-135)."""
    src, dst = _u32(src), _u32(dst)
    check(A.LIB.gspmm_edge_list_write(_path(path), num_nodes, len(src), _ptr(src), _ptr(dst)),
          "save_edge_list")
