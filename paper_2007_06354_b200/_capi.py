"""ctypes binding of the C-ABI (include/gspmm_b200.h).

Loads the in-tree ``_lib/libgspmm_b200.so`` (built by ``make -C
paper_2007_06354_b200`` / ``__graft_entry__.build()``) and fails loudly when it
is missing: there is no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libgspmm_b200.so")

# status codes
OK, ERR_CONFIG, ERR_SHAPE, ERR_STRUCTURE, ERR_CUDA, ERR_ARG, ERR_IO, ERR_PARSE = 0, 1, 2, 3, 4, 5, 6, 7
# enums (reference numeric values)
U, V, E, NONE = 0, 1, 2, 3
ADD, SUB, MUL, DIV, DOT, COPY = 0, 1, 2, 3, 4, 5
SUM, MAX, MIN, PROD, COPY_LAST, MEAN = 0, 1, 2, 3, 4, 5
SRC_MAJOR, DST_MAJOR = 0, 1
PUSH, PULL, BLOCKED, SPMM = 0, 1, 2, 3
EDGE_BY_ID, EDGE_BY_POS = 0, 1


class GspmmError(RuntimeError):
    status = -1


class ConfigError(GspmmError):
    status = ERR_CONFIG


class ShapeError(GspmmError):
    status = ERR_SHAPE


class StructureError(GspmmError):
    status = ERR_STRUCTURE


class DeviceError(GspmmError):
    status = ERR_CUDA


class ArgumentError(GspmmError):
    status = ERR_ARG


class IoError(GspmmError):
    status = ERR_IO


class ParseError(GspmmError):
    status = ERR_PARSE


_ERRORS = {ERR_CONFIG: ConfigError, ERR_SHAPE: ShapeError, ERR_STRUCTURE: StructureError,
           ERR_CUDA: DeviceError, ERR_ARG: ArgumentError, ERR_IO: IoError, ERR_PARSE: ParseError}


class Config(C.Structure):
    _fields_ = [("lhs", C.c_int32), ("rhs", C.c_int32), ("binary", C.c_int32),
                ("reduce", C.c_int32), ("out", C.c_int32)]

    def astuple(self):
        return (self.lhs, self.rhs, self.binary, self.reduce, self.out)


class Mat(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("dim", C.c_int64),
                ("ld", C.c_int64), ("edge_order", C.c_int32)]


class Out(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("dim", C.c_int64),
                ("ld", C.c_int64)]


class Plan(C.Structure):
    _fields_ = [("seg_cost", C.c_uint32), ("long_threshold", C.c_uint32),
                ("unit_cols", C.c_uint32), ("kernel", C.c_int32), ("long_ctas", C.c_uint32),
                ("split_edges", C.c_uint32)]


class Options(C.Structure):
    _fields_ = [("arg_other", C.c_void_p), ("arg_edge", C.c_void_p), ("arg_ld", C.c_int64),
                ("heads", C.c_int32), ("other_scale", C.c_void_p), ("source_blocks", C.c_int32),
                ("out2", C.c_void_p), ("out2_ld", C.c_int64), ("reduce2", C.c_int32)]


# Every symbol include/gspmm_b200.h declares, with its prototype.
_vp, _i64, _u32, _u64, _i32, _dbl = C.c_void_p, C.c_int64, C.c_uint32, C.c_uint64, C.c_int, C.c_double
_P = C.POINTER
SIGNATURES = {
    "gspmm_last_error": (C.c_char_p, []),
    "gspmm_abi_version": (_i32, []),
    "gspmm_validate_config": (_i32, [_P(Config)]),
    "gspmm_named_config": (_i32, [C.c_char_p, _P(Config)]),
    "gspmm_required_orientation": (_i32, [_i32, _i32]),
    "gspmm_graph_create": (_i32, [_i32, _i32, _u32, _u32, _vp, _vp, _vp, _i32, _P(_vp)]),
    "gspmm_graph_create_device": (_i32, [_i32, _i32, _u32, _u32, _vp, _vp, _vp, _P(_vp)]),
    "gspmm_graph_destroy": (_i32, [_vp]),
    "gspmm_graph_info": (_i32, [_vp, _P(_i32), _P(_u32), _P(_u32), _P(_u64), _P(_u32)]),
    "gspmm_graph_device_csr": (_i32, [_vp, _P(_vp), _P(_vp), _P(_vp)]),
    "gspmm_graph_permute_edges": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "gspmm_graph_set_source_blocks": (_i32, [_vp, _i32]),
    "gspmm_graph_set_plan": (_i32, [_vp, _P(Plan)]),
    "gspmm_binary_reduce": (_i32, [_vp, _P(Config), _P(Mat), _P(Mat), _P(Mat), _P(Out), _vp]),
    "gspmm_binary_reduce_ex": (_i32, [_vp, _P(Config), _P(Mat), _P(Mat), _P(Mat), _P(Out),
                                      _P(Options), _vp]),
    "gspmm_copy_reduce": (_i32, [_vp, _P(Mat), _i32, _P(Out), _vp]),
    "gspmm_argmax_backward": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "gspmm_argmax_backward_range": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64,
                                           _i64, _vp]),
    "gspmm_argmax_backward_host": (_i32, [_vp, _i64, _i64, _vp, _vp, _i64, _i32, _vp]),
    "gspmm_argmax_backward_host_async": (_i32, [_vp, _i64, _i64, _vp, _vp, _i64, _i32, _vp,
                                                _vp, _vp]),
    "gspmm_edge_softmax": (_i32, [_vp, _P(Mat), _P(Out), _vp]),
    "gspmm_edge_softmax_backward": (_i32, [_vp, _P(Mat), _P(Mat), _P(Out), _vp]),
    "gspmm_binary_reduce_host": (_i32, [_vp, _P(Config), _P(Mat), _P(Mat), _P(Mat), _P(Out),
                                        _P(Options), _vp]),
    "gspmm_binary_reduce_host_async": (_i32, [_vp, _P(Config), _P(Mat), _P(Mat), _P(Mat),
                                              _P(Out), _P(Options), _vp, _vp, _vp]),
    "gspmm_out_shape": (_i32, [_vp, _P(Config), _P(Mat), _P(Mat), _P(Mat), _P(Options),
                               _P(_i64), _P(_i64)]),
    "gspmm_launch_count": (_u64, []),
    "gspmm_synth_rmat": (_i64, [_u32, _u64, _dbl, _dbl, _dbl, _dbl, _u64, _vp, _vp, _i32]),
    "gspmm_synth_er": (_i64, [_u32, _u64, _dbl, _u64, _P(_vp), _P(_vp)]),
    "gspmm_free": (None, [_vp]),
    "gspmm_build_csr": (_i32, [_u32, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _i32]),
    "gspmm_transpose": (_i32, [_u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _i32]),
    "gspmm_build_csr_device": (_i32, [_u32, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "gspmm_transpose_device": (_i32, [_u32, _u32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gspmm_synth_uniform": (None, [_i64, _u64, _vp, _i32]),
    "gspmm_synth_normal": (None, [_i64, _u64, _vp, _i32]),
    "gspmm_synth_gcn_weights": (None, [_u32, _i64, _vp, _vp, _vp, _i32]),
    "gspmm_synth_powerlaw": (_i64, [_u32, _u32, _u32, _u64, _vp, _vp, _i32]),
    "gspmm_fmat1_info": (_i32, [C.c_char_p, _P(_i64), _P(_i64)]),
    "gspmm_fmat1_read": (_i32, [C.c_char_p, _vp, _i64]),
    "gspmm_fmat1_read_device": (_i32, [C.c_char_p, _i32, _vp, _i64, _vp]),
    "gspmm_fmat1_write": (_i32, [C.c_char_p, _vp, _i64, _i64, _i64]),
    "gspmm_csr1_info": (_i32, [C.c_char_p, _P(_i32), _P(_u64), _P(_u64), _P(_u64)]),
    "gspmm_csr1_read": (_i32, [C.c_char_p, _vp, _vp, _vp]),
    "gspmm_csr1_write": (_i32, [C.c_char_p, _i32, _u32, _u32, _vp, _vp, _vp]),
    "gspmm_graph_load_csr1": (_i32, [C.c_char_p, _i32, _P(_vp)]),
    "gspmm_validate_csr_device": (_i32, [_i32, _u32, _u32, _vp, _vp, _vp, _vp]),
    "gspmm_edge_list_read": (_i32, [C.c_char_p, _P(_u32), _P(_u64), _P(_vp), _P(_vp)]),
    "gspmm_edge_list_write": (_i32, [C.c_char_p, _u32, _u64, _vp, _vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__; __graft_entry__.build()'); "
            "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def last_error():
    return LIB.gspmm_last_error().decode(errors="replace")


def check(status, what=""):
    if status != OK:
        cls = _ERRORS.get(status, GspmmError)
        raise cls(f"{what}: {last_error()}" if what else last_error())
    return status
