"""Python face of the parity oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module; the product package never does.

Two back ends:
  * ``C``   -- oracle/_build/libgspmm_oracle.so, the C restatement of the
              reference algorithm (oracle/gspmm_oracle.c), always built;
  * ``REF`` -- oracle/_ref/libgspmm_ref.so, the unmodified reference library
              compiled from /root/reference/proj/src (None when absent).

Ops the reference lacks (mean, argmax, max backward, multi-head, GCN weights,
softmax attention, self-loops, symmetrisation) are composed here from the
restated primitives exactly as SURVEY.md section 8(a) a17 specifies.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# enum values of the reference (ops.hpp:28,33; br_config.hpp Operand)
U, V, E, NONE = 0, 1, 2, 3
ADD, SUB, MUL, DIV, DOT, COPY = 0, 1, 2, 3, 4, 5
SUM, MAX, MIN, PROD, LAST = 0, 1, 2, 3, 4
SRC_MAJOR, DST_MAJOR = 0, 1
PUSH, PULL, BLOCKED, SPMM = 0, 1, 2, 3

OK, CONFIG, SHAPE, STRUCTURE = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


class Feat(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("dim", C.c_int64)]


def _feat(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    f = Feat(a.ctypes.data, a.shape[0], a.shape[1])
    f._keep = a
    return f


def _ptr(a):
    return None if a is None else a.ctypes.data


_u32p = C.POINTER(C.c_uint32)


def _load_c():
    path = os.path.join(_HERE, "_build", "libgspmm_oracle.so")
    if not os.path.exists(path):
        raise OSError(f"{path} missing: run `make -C oracle`")
    lib = C.CDLL(path)
    vp, i64, u32, u64, i32, dbl = C.c_void_p, C.c_int64, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    fp = C.POINTER(Feat)
    sig = {
        "or_splitmix64_at": (u64, [u64, u64]),
        "or_u01_at": (dbl, [u64, u64]),
        "or_unit_float_at": (C.c_float, [u64, u64]),
        "or_normal_at": (C.c_float, [u64, u64]),
        "or_gen_er": (i64, [u32, u64, dbl, u64, C.POINTER(_u32p), C.POINTER(_u32p)]),
        "or_gen_rmat": (i64, [u32, u64, dbl, dbl, dbl, dbl, u64, C.POINTER(_u32p), C.POINTER(_u32p)]),
        "or_gen_sbm": (i64, [u32, i32, dbl, dbl, u64, C.POINTER(_u32p), C.POINTER(_u32p)]),
        "or_free": (None, [vp]),
        "or_gen_powerlaw": (i64, [u32, u32, u32, u64, C.POINTER(_u32p), C.POINTER(_u32p)]),
        "or_random_features": (None, [i64, i64, u64, vp]),
        "or_normal_features": (None, [i64, u64, vp]),
        "or_normal_features_at": (None, [i64, i64, u64, vp]),
        "or_build_csr": (i32, [u32, i64, vp, vp, i32, vp, vp, vp]),
        "or_transpose": (i32, [u32, u32, vp, vp, vp, vp, vp, vp]),
        "or_validate": (i32, [u32, u32, i64, vp, i64, vp, vp]),
        "or_out_shape": (i32, [i32, u32, u32, i64, i32, i32, i32, i32, i32, fp, fp, fp,
                               C.POINTER(i64), C.POINTER(i64)]),
        "or_binary_reduce": (i32, [i32, u32, u32, vp, vp, vp, i32, i32, i32, i32, i32, fp, fp, fp, vp]),
        "or_oracle_aggregate": (i32, [u32, i64, vp, vp, i32, i32, i32, i32, i32, fp, fp, fp, vp]),
        "or_mean": (i32, [i32, u32, u32, vp, vp, vp, i32, fp, vp]),
        "or_copy_max_argmax": (i32, [u32, u32, vp, vp, vp, i32, fp, vp, vp, vp]),
        "or_argmax_backward": (None, [i64, i64, vp, vp, i64, vp]),
        "or_copy_max_argmax_mt": (i32, [u32, u32, vp, vp, vp, i32, fp, vp, vp, vp, i32]),
        "or_argmax_backward_mt": (None, [i64, i64, vp, vp, i64, vp, i32]),
        "or_max_rel_error": (dbl, [i64, vp, vp]),
        "or_bit_equal": (i32, [i64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def _load_ref():
    path = os.path.join(_HERE, "_ref", "libgspmm_ref.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    vp, i64, u32, u64, i32, dbl = C.c_void_p, C.c_int64, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    fp = C.POINTER(Feat)
    sig = {
        "ref_free": (None, [vp]),
        "ref_generate": (i64, [i32, u32, u64, dbl, i32, dbl, dbl, dbl, dbl, dbl, dbl, u64,
                               C.POINTER(_u32p), C.POINTER(_u32p)]),
        "ref_random_features": (None, [i64, i64, u64, vp]),
        "ref_build_csr": (i32, [u32, i64, vp, vp, i32, vp, vp, vp]),
        "ref_transpose": (i32, [i32, u32, u32, vp, vp, vp, vp, vp, vp]),
        "ref_binary_reduce": (i32, [i32, i32, u32, u32, vp, vp, vp, i32, i32, i32, i32, i32,
                                    fp, fp, fp, i32, vp, C.POINTER(i64), C.POINTER(i64)]),
        "ref_oracle_aggregate": (i32, [u32, i64, vp, vp, i32, i32, i32, i32, i32, fp, fp, fp, vp,
                                       C.POINTER(i64), C.POINTER(i64)]),
        "ref_views_create": (vp, [u32, i64, vp, vp]),
        "ref_views_free": (None, [vp]),
        "ref_views_csr": (i32, [vp, i32, vp, vp, vp]),
        "ref_feat_create": (vp, [i64, i64, vp]),
        "ref_feat_free": (None, [vp]),
        "ref_run": (dbl, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, i32, vp]),
        "ref_graph_create": (vp, [i32, u32, u32, vp, vp, vp]),
        "ref_graph_free": (None, [vp]),
        "ref_feat_create_strided": (vp, [i64, i64, vp, i64]),
        "ref_run_graph": (dbl, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, i32, vp, i64]),
        "ref_bench_case": (dbl, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, i32, i32, i32,
                                 C.POINTER(dbl), C.POINTER(dbl)]),
        "ref_bench_csv": (dbl, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, i32, i32, i32,
                                C.c_char_p, i32]),
        "ref_bench_csv_header": (C.c_char_p, []),
        "ref_io_error": (C.c_char_p, []),
        "ref_save_csr": (i32, [C.c_char_p, vp]),
        "ref_load_csr": (i32, [C.c_char_p, C.POINTER(vp), C.POINTER(i32), C.POINTER(u32),
                               C.POINTER(u32), C.POINTER(u64)]),
        "ref_graph_arrays": (None, [vp, vp, vp, vp]),
        "ref_save_feature_matrix": (i32, [C.c_char_p, vp]),
        "ref_load_feature_matrix": (i32, [C.c_char_p, C.POINTER(vp), C.POINTER(i64),
                                          C.POINTER(i64)]),
        "ref_feat_data": (None, [vp, vp]),
        "ref_save_edge_list": (i32, [C.c_char_p, u32, i64, vp, vp]),
        "ref_load_edge_list": (i32, [C.c_char_p, C.POINTER(u32), C.POINTER(i64),
                                     C.POINTER(_u32p), C.POINTER(_u32p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load_c()
REF = _load_ref()


def _check(st, what=""):
    if st != 0:
        raise OracleError(st, what)


# ------------------------------------------------------------------- rng
def splitmix64_at(seed, counter):
    return LIB.or_splitmix64_at(seed, counter)


def random_features(rows, dim, seed):
    """generate.cpp:256-266, U[-1,1)."""
    out = np.empty((rows, dim), np.float32)
    LIB.or_random_features(rows, dim, seed, out.ctypes.data)
    return out


def normal_features(rows, dim, seed, threads=1):
    """Builder-defined N(0,1), Box-Muller.  threads > 1 splits the
    counter stream into chunks (ctypes releases the GIL)."""
    out = np.empty((rows, dim), np.float32)
    total = rows * dim
    if threads <= 1 or total < (1 << 20):
        LIB.or_normal_features(total, seed, out.ctypes.data)
        return out
    from concurrent.futures import ThreadPoolExecutor
    flat = out.reshape(-1)
    bounds = np.linspace(0, total, threads + 1).astype(np.int64)

    def work(k):
        b, e = int(bounds[k]), int(bounds[k + 1])
        LIB.or_normal_features_at(b, e - b, seed, flat[b:].ctypes.data)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return out


# ------------------------------------------------------------ generators
def _take_edges(m, ps, pd, free):
    if m < 0:
        raise OracleError(-m, "generator")
    src = np.ctypeslib.as_array(ps, shape=(max(m, 1),))[:m].copy()
    dst = np.ctypeslib.as_array(pd, shape=(max(m, 1),))[:m].copy()
    free(C.cast(ps, C.c_void_p))
    free(C.cast(pd, C.c_void_p))
    return src, dst


def gen_er(n, num_edges=0, prob=-1.0, seed=0):
    ps, pd = _u32p(), _u32p()
    m = LIB.or_gen_er(n, num_edges, prob, seed, C.byref(ps), C.byref(pd))
    return _take_edges(m, ps, pd, LIB.or_free)


def gen_rmat(n, num_edges, a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
    ps, pd = _u32p(), _u32p()
    m = LIB.or_gen_rmat(n, num_edges, a, b, c, d, seed, C.byref(ps), C.byref(pd))
    return _take_edges(m, ps, pd, LIB.or_free)


def gen_sbm(n, blocks, p_in, p_out, seed=0):
    ps, pd = _u32p(), _u32p()
    m = LIB.or_gen_sbm(n, blocks, p_in, p_out, seed, C.byref(ps), C.byref(pd))
    return _take_edges(m, ps, pd, LIB.or_free)


def gen_powerlaw(n, d_min, d_max, seed=0):
    """Builder-defined power-law in-degree graph (cfg5)."""
    ps, pd = _u32p(), _u32p()
    m = LIB.or_gen_powerlaw(n, d_min, d_max, seed, C.byref(ps), C.byref(pd))
    return _take_edges(m, ps, pd, LIB.or_free)


def random_small_graph(seed):
    """test_util.hpp:30-61: n <= 200, m <= 2000, kind picked by seed."""
    pick = splitmix64_at(seed, 9000)
    n = 8 + splitmix64_at(seed, 9001) % 193
    degree = 1.0 + float(splitmix64_at(seed, 9002) % 10)
    kind = pick % 3
    if kind == 0:
        src, dst = gen_er(n, 0, min(1.0, degree / (n - 1.0)), seed)
    elif kind == 1:
        m = min(2000, int(degree * n))
        src, dst = gen_rmat(n, m, 0.40, 0.25, 0.25, 0.10, seed)
    else:
        blocks = 1 + int(splitmix64_at(seed, 9004) % 4)
        p_in = min(1.0, degree * blocks / float(n))
        src, dst = gen_sbm(n, blocks, p_in, p_in / 20.0, seed)
    return int(n), src, dst


# ------------------------------------------------------------ graph core
def build_csr(n, src, dst, orientation=DST_MAJOR):
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    m = len(src)
    indptr = np.empty(n + 1, np.uint32)
    indices = np.empty(max(m, 1), np.uint32)
    eids = np.empty(max(m, 1), np.uint32)
    _check(LIB.or_build_csr(n, m, _ptr(src), _ptr(dst), orientation, _ptr(indptr),
                            _ptr(indices), _ptr(eids)), "build_csr")
    return indptr, indices[:m], eids[:m]


def transpose(num_rows, num_cols, indptr, indices, eids):
    m = int(indptr[-1])
    t_indptr = np.empty(num_cols + 1, np.uint32)
    t_indices = np.empty(max(m, 1), np.uint32)
    t_eids = np.empty(max(m, 1), np.uint32)
    indices = np.ascontiguousarray(indices, np.uint32)
    eids = np.ascontiguousarray(eids, np.uint32)
    LIB.or_transpose(num_rows, num_cols, _ptr(np.ascontiguousarray(indptr, np.uint32)),
                     _ptr(indices), _ptr(eids), _ptr(t_indptr), _ptr(t_indices), _ptr(t_eids))
    return t_indptr, t_indices[:m], t_eids[:m]


def validate(num_rows, num_cols, indptr, indices, eids):
    indptr = np.ascontiguousarray(indptr, np.uint32)
    indices = np.ascontiguousarray(indices, np.uint32)
    eids = np.ascontiguousarray(eids, np.uint32)
    if len(indptr) != num_rows + 1:
        return 1
    if len(indices) != len(eids):
        return 4
    return LIB.or_validate(num_rows, num_cols, len(indptr), _ptr(indptr), len(indices),
                           _ptr(indices), _ptr(eids))


class Graph:
    """Both orientations of one edge list (make_views, bench.cpp:48-53)."""

    def __init__(self, n, src, dst):
        self.n = int(n)
        self.src = np.ascontiguousarray(src, np.uint32)
        self.dst = np.ascontiguousarray(dst, np.uint32)
        self.m = len(self.src)
        self.dst_major = build_csr(self.n, self.src, self.dst, DST_MAJOR)
        self.src_major = transpose(self.n, self.n, *self.dst_major)

    def csr(self, orientation):
        return self.dst_major if orientation == DST_MAJOR else self.src_major


# ---------------------------------------------------------- config names
_OPS = {"u": U, "v": V, "e": E}
_BIN = {"add": ADD, "sub": SUB, "mul": MUL, "div": DIV, "dot": DOT}
_RED = {"add": SUM, "max": MAX, "min": MIN, "mul": PROD, "copy": LAST}


def named_config(name):
    """named_config, br_config.cpp:96-131 -> (lhs, rhs, binop, reduce, out)."""
    t = name.split("_")
    if len(t) == 4:
        if t[0] not in ("u", "e") or t[1] != "copy" or t[2] not in _RED or t[3] != "v":
            raise OracleError(CONFIG, name)
        return (_OPS[t[0]], NONE, COPY, _RED[t[2]], V)
    if len(t) == 5:
        if t[0] not in _OPS or t[1] not in _BIN or t[2] not in _OPS or t[3] not in _RED \
                or t[4] not in _OPS:
            raise OracleError(CONFIG, name)
        cfg = (_OPS[t[0]], _OPS[t[2]], _BIN[t[1]], _RED[t[3]], _OPS[t[4]])
        if cfg[4] == E:
            cfg = cfg[:3] + (LAST, E)
        if cfg[0] == cfg[1]:
            raise OracleError(CONFIG, name)
        return cfg
    raise OracleError(CONFIG, name)


APPLICATION_CONFIGS = [  # br_config.cpp:148-161
    "u_copy_add_v", "u_dot_v_add_e", "u_mul_e_add_v", "e_copy_add_v", "e_copy_max_v",
    "u_add_v_copy_e", "e_sub_v_copy_e", "e_div_v_copy_e", "v_mul_e_copy_e",
]


# ----------------------------------------------------------- aggregation
def out_shape(orientation, num_rows, num_cols, m, cfg, u=None, v=None, e=None):
    fu, fv, fe = _feat(u), _feat(v), _feat(e)
    r, d = C.c_int64(), C.c_int64()
    st = LIB.or_out_shape(orientation, num_rows, num_cols, m, *cfg, fu, fv, fe,
                          C.byref(r), C.byref(d))
    _check(st, "out_shape")
    return r.value, d.value


def binary_reduce(g, cfg, u=None, v=None, e=None, orientation=None):
    """binary_reduce(RowParallelSpmm, g.oriented(required), cfg, u, v, e)."""
    if orientation is None:
        orientation = SRC_MAJOR if cfg[4] == U else DST_MAJOR
    indptr, indices, eids = g.csr(orientation)
    fu, fv, fe = _feat(u), _feat(v), _feat(e)
    r, d = C.c_int64(), C.c_int64()
    _check(LIB.or_out_shape(orientation, g.n, g.n, g.m, *cfg, fu, fv, fe, C.byref(r),
                            C.byref(d)), "binary_reduce")
    out = np.empty((r.value, d.value), np.float32)
    _check(LIB.or_binary_reduce(orientation, g.n, g.n, _ptr(indptr), _ptr(indices), _ptr(eids),
                                *cfg, fu, fv, fe, out.ctypes.data), "binary_reduce")
    return out


def oracle_aggregate(g, cfg, u=None, v=None, e=None):
    fu, fv, fe = _feat(u), _feat(v), _feat(e)
    orientation = SRC_MAJOR if cfg[4] == U else DST_MAJOR
    r, d = C.c_int64(), C.c_int64()
    _check(LIB.or_out_shape(orientation, g.n, g.n, g.m, *cfg, fu, fv, fe, C.byref(r),
                            C.byref(d)), "oracle_aggregate")
    out = np.empty((r.value, d.value), np.float32)
    _check(LIB.or_oracle_aggregate(g.n, g.m, _ptr(g.src), _ptr(g.dst), *cfg, fu, fv, fe,
                                   out.ctypes.data), "oracle_aggregate")
    return out


def mean(g, src_feats, lhs=U, orientation=DST_MAJOR):
    """a17.1: copy-sum / (float)in-degree, 0 for empty rows."""
    indptr, indices, eids = g.csr(orientation)
    f = _feat(src_feats)
    out = np.empty((g.n, f.dim), np.float32)
    _check(LIB.or_mean(orientation, g.n, g.n, _ptr(indptr), _ptr(indices), _ptr(eids), lhs,
                       f, out.ctypes.data), "mean")
    return out


def copy_max_argmax(g, src_feats, lhs=U):
    """a17.2: max value (== binary_reduce u_copy_max_v) + first-position argmax."""
    indptr, indices, eids = g.dst_major
    f = _feat(src_feats)
    out = np.empty((g.n, f.dim), np.float32)
    arg_u = np.empty((g.n, f.dim), np.int32)
    arg_e = np.empty((g.n, f.dim), np.int32)
    _check(LIB.or_copy_max_argmax(g.n, g.n, _ptr(indptr), _ptr(indices), _ptr(eids), lhs, f,
                                  out.ctypes.data, arg_u.ctypes.data, arg_e.ctypes.data))
    return out, arg_u, arg_e


def copy_max_argmax_csr(csr, num_rows, num_cols, src_feats, lhs=U, threads=0):
    """a17.2 on a given dst-major CSR, threaded (BASELINE sizes): identical to
    copy_max_argmax (or_copy_max_argmax_mt)."""
    indptr, indices, eids = (np.ascontiguousarray(a, np.uint32) for a in csr)
    f = _feat(src_feats)
    out = np.empty((num_rows, f.dim), np.float32)
    arg_u = np.empty((num_rows, f.dim), np.int32)
    arg_e = np.empty((num_rows, f.dim), np.int32)
    _check(LIB.or_copy_max_argmax_mt(num_rows, num_cols, _ptr(indptr), _ptr(indices),
                                     _ptr(eids), lhs, f, out.ctypes.data, arg_u.ctypes.data,
                                     arg_e.ctypes.data, threads))
    return out, arg_u, arg_e


def argmax_backward_mt(arg, grad_out, src_rows, threads=0):
    """a17.4, threaded over source-row ranges (same per-entry order)."""
    arg = np.ascontiguousarray(arg, np.int32)
    grad_out = np.ascontiguousarray(grad_out, np.float32)
    out = np.empty((src_rows, arg.shape[1]), np.float32)
    LIB.or_argmax_backward_mt(arg.shape[0], arg.shape[1], arg.ctypes.data,
                              grad_out.ctypes.data, src_rows, out.ctypes.data, threads)
    return out


def argmax_backward(arg, grad_out, src_rows):
    """a17.4: scatter grad_out through the argmax, f64 accumulation."""
    arg = np.ascontiguousarray(arg, np.int32)
    grad_out = np.ascontiguousarray(grad_out, np.float32)
    out = np.empty((src_rows, arg.shape[1]), np.float32)
    LIB.or_argmax_backward(arg.shape[0], arg.shape[1], arg.ctypes.data, grad_out.ctypes.data,
                           src_rows, out.ctypes.data)
    return out


def sum_backward(g, grad_out, e=None):
    """a17.3 grad_u of copy_u/u_mul_e + sum: binary_reduce on the src-major
    graph with v_mul_e_add_u (or {V, None, Copy, Sum, U} without e)."""
    if e is None:
        return binary_reduce(g, (V, NONE, COPY, SUM, U), v=grad_out)
    return binary_reduce(g, (V, E, MUL, SUM, U), v=grad_out, e=e)


def edge_grad(g, x, grad_out):
    """a17.3 grad_e: binary_reduce(dst_major, u_dot_v_copy_e, u=x, v=grad_out)."""
    return binary_reduce(g, (U, V, DOT, LAST, E), u=x, v=grad_out)


def in_degree(g):
    return np.diff(g.dst_major[0].astype(np.int64))


def mean_backward(g, grad_out):
    """a17.3 for mean: v_mul_e_add_u with e = 1/(float)deg_in(dst(e))."""
    deg = in_degree(g)
    inv = np.zeros(g.n, np.float32)
    nz = deg > 0
    inv[nz] = np.float32(1.0) / deg[nz].astype(np.float32)
    e = inv[g.dst].reshape(-1, 1)
    return binary_reduce(g, (V, E, MUL, SUM, U), v=grad_out, e=e)


def multihead_u_mul_e_sum(g, x, a, heads):
    """a17.5: per head h, binary_reduce(u_mul_e_add_v) on the contiguous
    head slice x[:, h*D:(h+1)*D] with scalar edge weight a[:, h]."""
    n, width = x.shape
    d = width // heads
    out = np.empty((g.n, width), np.float32)
    for h in range(heads):
        xh = np.ascontiguousarray(x[:, h * d:(h + 1) * d])
        ah = np.ascontiguousarray(a[:, h:h + 1])
        out[:, h * d:(h + 1) * d] = binary_reduce(g, (U, E, MUL, SUM, V), u=xh, e=ah)
    return out


def multihead_backward(g, x, a, grad_out, heads):
    """a17.5 backward: grad_x per head on the src-major graph, grad_a per head
    as u_dot_v_copy_e of the head slices."""
    n, width = x.shape
    d = width // heads
    grad_x = np.empty_like(x)
    grad_a = np.empty((g.m, heads), np.float32)
    for h in range(heads):
        gh = np.ascontiguousarray(grad_out[:, h * d:(h + 1) * d])
        ah = np.ascontiguousarray(a[:, h:h + 1])
        xh = np.ascontiguousarray(x[:, h * d:(h + 1) * d])
        grad_x[:, h * d:(h + 1) * d] = binary_reduce(g, (V, E, MUL, SUM, U), v=gh, e=ah)
        grad_a[:, h] = binary_reduce(g, (U, V, DOT, LAST, E), u=xh, v=gh)[:, 0]
    return grad_x, grad_a


# ------------------------------------------------- input synthesis pieces
def add_self_loops(n, src, dst):
    """cfg2: append (i, i) for every node after the generated edges."""
    loop = np.arange(n, dtype=np.uint32)
    return np.concatenate([src, loop]), np.concatenate([dst, loop])


def symmetrize(src, dst):
    """cfg3: append the reverse of every edge (edge m+i = reverse of edge i)."""
    return np.concatenate([src, dst]), np.concatenate([dst, src])


def gcn_weights(n, src, dst):
    """cfg2: w_e = 1/sqrt(deg_out(u) * deg_in(v)), f64 then rounded, edge-id order."""
    dout = np.bincount(src, minlength=n).astype(np.float64)
    din = np.bincount(dst, minlength=n).astype(np.float64)
    w = 1.0 / np.sqrt(dout[src] * din[dst])
    return w.astype(np.float32).reshape(-1, 1)


def softmax_attention(n, dst, logits):
    """cfg4: a[e,h] = softmax over the in-edges of dst(e) of logits[:, h],
    computed in f64 and rounded to fp32."""
    lg = logits.astype(np.float64)
    m, heads = lg.shape
    mx = np.full((n, heads), -np.inf)
    np.maximum.at(mx, dst, lg)
    ex = np.exp(lg - mx[dst])
    den = np.zeros((n, heads))
    np.add.at(den, dst, ex)
    return (ex / den[dst]).astype(np.float32)


def softmax_attention_backward(n, dst, a, grad_a):
    """Edge-softmax backward (f64): grad_l = a * (grad_a - sum_row(a * grad_a))."""
    a64, g64 = a.astype(np.float64), grad_a.astype(np.float64)
    s = np.zeros((n, a.shape[1]))
    np.add.at(s, dst, a64 * g64)
    return a64 * (g64 - s[dst])


# ----------------------------------------------------------- comparisons
def max_rel_error(got, want):
    got = np.ascontiguousarray(got, np.float32)
    want = np.ascontiguousarray(want, np.float32)
    if got.shape != want.shape:
        return float("inf")
    return LIB.or_max_rel_error(got.size, got.ctypes.data, want.ctypes.data)


def bit_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    if a.shape != b.shape:
        return False
    return bool(LIB.or_bit_equal(a.size, a.ctypes.data, b.ctypes.data))


def is_exact_reduce(reduce):
    """compare.hpp:58-61."""
    return reduce in (MAX, MIN, LAST)


# ------------------------------------------------ the reference library
def ref_available():
    return REF is not None


def ref_generate(kind, n, num_edges=0, prob=-1.0, blocks=2, p_in=0.0, p_out=0.0,
                 a=0.57, b=0.19, c=0.19, d=0.05, seed=0):
    ps, pd = _u32p(), _u32p()
    m = REF.ref_generate(kind, n, num_edges, prob, blocks, p_in, p_out, a, b, c, d, seed,
                         C.byref(ps), C.byref(pd))
    return _take_edges(m, ps, pd, REF.ref_free)


def ref_random_features(rows, dim, seed):
    out = np.empty((rows, dim), np.float32)
    REF.ref_random_features(rows, dim, seed, out.ctypes.data)
    return out


def ref_build_csr(n, src, dst, orientation=DST_MAJOR):
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    m = len(src)
    indptr = np.empty(n + 1, np.uint32)
    indices = np.empty(max(m, 1), np.uint32)
    eids = np.empty(max(m, 1), np.uint32)
    _check(REF.ref_build_csr(n, m, _ptr(src), _ptr(dst), orientation, _ptr(indptr),
                             _ptr(indices), _ptr(eids)), "ref_build_csr")
    return indptr, indices[:m], eids[:m]


def ref_transpose(orientation, num_rows, num_cols, indptr, indices, eids):
    m = int(indptr[-1])
    t_indptr = np.empty(num_cols + 1, np.uint32)
    t_indices = np.empty(max(m, 1), np.uint32)
    t_eids = np.empty(max(m, 1), np.uint32)
    _check(REF.ref_transpose(orientation, num_rows, num_cols,
                             _ptr(np.ascontiguousarray(indptr, np.uint32)),
                             _ptr(np.ascontiguousarray(indices, np.uint32)),
                             _ptr(np.ascontiguousarray(eids, np.uint32)),
                             _ptr(t_indptr), _ptr(t_indices), _ptr(t_eids)))
    return t_indptr, t_indices[:m], t_eids[:m]


def ref_binary_reduce(g, cfg, u=None, v=None, e=None, strategy=SPMM, threads=0):
    orientation = SRC_MAJOR if cfg[4] == U else DST_MAJOR
    if strategy == PUSH:
        orientation = 1 - orientation
    indptr, indices, eids = g.csr(orientation)
    fu, fv, fe = _feat(u), _feat(v), _feat(e)
    r, d = C.c_int64(), C.c_int64()
    st = REF.ref_binary_reduce(strategy, orientation, g.n, g.n, _ptr(indptr), _ptr(indices),
                               _ptr(eids), *cfg, fu, fv, fe, threads, None, C.byref(r),
                               C.byref(d))
    _check(st, "ref_binary_reduce")
    out = np.empty((r.value, d.value), np.float32)
    _check(REF.ref_binary_reduce(strategy, orientation, g.n, g.n, _ptr(indptr), _ptr(indices),
                                 _ptr(eids), *cfg, fu, fv, fe, threads, out.ctypes.data,
                                 C.byref(r), C.byref(d)), "ref_binary_reduce")
    return out


def ref_oracle_aggregate(g, cfg, u=None, v=None, e=None):
    fu, fv, fe = _feat(u), _feat(v), _feat(e)
    r, d = C.c_int64(), C.c_int64()
    _check(REF.ref_oracle_aggregate(g.n, g.m, _ptr(g.src), _ptr(g.dst), *cfg, fu, fv, fe, None,
                                    C.byref(r), C.byref(d)), "ref_oracle_aggregate")
    out = np.empty((r.value, d.value), np.float32)
    _check(REF.ref_oracle_aggregate(g.n, g.m, _ptr(g.src), _ptr(g.dst), *cfg, fu, fv, fe,
                                    out.ctypes.data, C.byref(r), C.byref(d)))
    return out


class RefGraph:
    """The reference library (oracle/_ref) on a canonical CSR handed in
    directly: binary_reduce(strategy, ...) with all host threads, for
    whole-output parity at the BASELINE sizes.  run() returns the output;
    run_timed() also the reference's own steady_clock seconds."""

    def __init__(self, orientation, num_rows, num_cols, indptr, indices, eids):
        if REF is None:
            raise OSError("oracle/_ref/libgspmm_ref.so not built")
        self._keep = [np.ascontiguousarray(a, np.uint32) for a in (indptr, indices, eids)]
        self.orientation, self.num_rows, self.num_cols = orientation, num_rows, num_cols
        self.h = REF.ref_graph_create(orientation, num_rows, num_cols,
                                      *(a.ctypes.data for a in self._keep))
        if not self.h:
            raise OracleError(9, "ref_graph_create")

    @staticmethod
    def feat(a):
        """FeatureMatrix from a 2-D float32 array (a column slice is fine)."""
        if a is None:
            return None
        a = np.asarray(a, np.float32)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        if a.strides[1] != 4:
            a = np.ascontiguousarray(a)
        return REF.ref_feat_create_strided(a.shape[0], a.shape[1], a.ctypes.data,
                                           a.strides[0] // 4)

    def run_timed(self, cfg, u=None, v=None, e=None, strategy=SPMM, threads=0, out=None):
        fs = [self.feat(x) for x in (u, v, e)]
        try:
            if out is None:
                rows = self.num_rows if cfg[4] != E else int(self._keep[0][-1])
                w = (1 if cfg[2] == DOT else
                     max(x.shape[1] if x.ndim > 1 else 1 for x in (u, v, e) if x is not None)
                     if cfg[2] != COPY else (u if cfg[0] == U else v if cfg[0] == V else e).shape[1])
                out = np.empty((rows, w), np.float32)
            assert out.strides[1] == 4
            t = REF.ref_run_graph(self.h, strategy, *cfg, *fs, threads, out.ctypes.data,
                                  out.strides[0] // 4)
            if t < 0:
                raise OracleError(int(-t), "ref_run_graph")
            return out, t
        finally:
            for f in fs:
                if f:
                    REF.ref_feat_free(f)

    def run(self, cfg, u=None, v=None, e=None, strategy=SPMM, threads=0, out=None):
        return self.run_timed(cfg, u, v, e, strategy, threads, out)[0]

    def close(self):
        if self.h:
            REF.ref_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------ file containers
# numpy restatement of the reference's binary containers (io.hpp:29-41,
# io.cpp:137-205) and thin wrappers over the reference's own readers /
# writers (oracle/_ref), for the loader round-trip tests.
IO_ERROR, PARSE_ERROR = 6, 7


def write_fmat1(path, a):
    """save_feature_matrix (io.cpp:137-147)."""
    a = np.ascontiguousarray(a, np.float32)
    with open(path, "wb") as f:
        f.write(b"FMAT1")
        f.write(np.array(a.shape, "<u8").tobytes())
        f.write(a.astype("<f4", copy=False).tobytes())


def read_fmat1(path):
    """load_feature_matrix (io.cpp:149-166); OracleError(IO_ERROR) on a bad file."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise OracleError(IO_ERROR, "cannot open " + path)
    if raw[:5] != b"FMAT1":
        raise OracleError(IO_ERROR, path + ": not a FMAT1 file")
    if len(raw) < 21:
        raise OracleError(IO_ERROR, path + ": truncated file")
    rows, dim = (int(v) for v in np.frombuffer(raw, "<u8", 2, 5))
    if len(raw) - 21 < rows * dim * 4:
        raise OracleError(IO_ERROR, path + ": truncated data section")
    return np.frombuffer(raw, "<f4", rows * dim, 21).reshape(rows, dim).copy()


def write_csr1(path, orientation, num_rows, num_cols, indptr, indices, eids):
    """save_csr (io.cpp:168-181): every element as a 64-bit little-endian word."""
    with open(path, "wb") as f:
        f.write(b"CSR1")
        f.write(bytes([1 if orientation == DST_MAJOR else 0]))
        f.write(np.array([num_rows, num_cols, int(indptr[num_rows])], "<u8").tobytes())
        for a in (indptr[:num_rows + 1], indices[:int(indptr[num_rows])],
                  eids[:int(indptr[num_rows])]):
            f.write(np.asarray(a).astype("<u8").tobytes())


def read_csr1(path):
    """load_csr (io.cpp:183-205) -> (orientation, num_rows, num_cols, indptr,
    indices, eids) as uint32 arrays; the payload is validated (csr.cpp:111-156)."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise OracleError(IO_ERROR, "cannot open " + path)
    if raw[:4] != b"CSR1":
        raise OracleError(IO_ERROR, path + ": not a CSR1 file")
    if len(raw) < 29:
        raise OracleError(IO_ERROR, path + ": truncated file")
    orientation = DST_MAJOR if raw[4] else SRC_MAJOR
    rows, cols, m = (int(v) for v in np.frombuffer(raw, "<u8", 3, 5))
    if len(raw) - 29 < 8 * (rows + 1 + 2 * m):
        raise OracleError(IO_ERROR, path + ": truncated file")
    arrs, off = [], 29
    for count in (rows + 1, m, m):
        a = np.frombuffer(raw, "<u8", count, off)
        off += 8 * count
        if count and int(a.max()) > 0xffffffff:
            raise OracleError(IO_ERROR, path + ": id does not fit the configured id width")
        arrs.append(a.astype(np.uint32))
    bad = validate(rows, cols, *arrs)
    if bad:
        raise OracleError(IO_ERROR, path + ": invalid CSR payload: " + bad)
    return (orientation, rows, cols, *arrs)


def _ref_io(st, what):
    if st:
        raise OracleError(st, what + ": " + REF.ref_io_error().decode(errors="replace"))


def ref_save_csr(path, orientation, num_rows, num_cols, indptr, indices, eids):
    g = RefGraph(orientation, num_rows, num_cols, indptr, indices, eids)
    try:
        _ref_io(REF.ref_save_csr(os.fsencode(path), g.h), "save_csr")
    finally:
        g.close()


def ref_load_csr(path):
    h, o, r, c, m = C.c_void_p(), C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint64()
    _ref_io(REF.ref_load_csr(os.fsencode(path), C.byref(h), C.byref(o), C.byref(r), C.byref(c),
                             C.byref(m)), "load_csr")
    indptr = np.empty(r.value + 1, np.uint32)
    indices = np.empty(max(m.value, 1), np.uint32)
    eids = np.empty(max(m.value, 1), np.uint32)
    REF.ref_graph_arrays(h, indptr.ctypes.data, indices.ctypes.data, eids.ctypes.data)
    REF.ref_graph_free(h)
    return o.value, r.value, c.value, indptr, indices[:m.value], eids[:m.value]


def ref_save_feature_matrix(path, a):
    a = np.ascontiguousarray(a, np.float32)
    f = REF.ref_feat_create(a.shape[0], a.shape[1], a.ctypes.data)
    try:
        _ref_io(REF.ref_save_feature_matrix(os.fsencode(path), f), "save_feature_matrix")
    finally:
        REF.ref_feat_free(f)


def ref_load_feature_matrix(path):
    f, r, d = C.c_void_p(), C.c_int64(), C.c_int64()
    _ref_io(REF.ref_load_feature_matrix(os.fsencode(path), C.byref(f), C.byref(r), C.byref(d)),
            "load_feature_matrix")
    out = np.empty((r.value, d.value), np.float32)
    REF.ref_feat_data(f, out.ctypes.data)
    REF.ref_feat_free(f)
    return out


def ref_save_edge_list(path, n, src, dst):
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    _ref_io(REF.ref_save_edge_list(os.fsencode(path), n, len(src), _ptr(src), _ptr(dst)),
            "save_edge_list")


def ref_load_edge_list(path):
    n, m, ps, pd = C.c_uint32(), C.c_int64(), _u32p(), _u32p()
    _ref_io(REF.ref_load_edge_list(os.fsencode(path), C.byref(n), C.byref(m), C.byref(ps),
                                   C.byref(pd)), "load_edge_list")
    src, dst = _take_edges(m.value, ps, pd, REF.ref_free)
    return n.value, src, dst
