"""B200-native (sm_100a) Copy-Reduce / Binary-Reduce over CSR graphs.

The hot path of arXiv 2007.06354 (DGL's CPU aggregation primitives, as
re-implemented by the reference's gspmm::binary_reduce / copy_reduce),
rebuilt as hand-written CUDA kernels behind a C-ABI (include/gspmm_b200.h).
See DESIGN.md.
"""
from . import _capi
from ._capi import (ADD, COPY, COPY_LAST, DIV, DOT, DST_MAJOR, E, EDGE_BY_ID, EDGE_BY_POS, MAX,
                    MEAN, MIN, MUL, NONE, PROD, PULL, PUSH, BLOCKED, SPMM, SRC_MAJOR, SUB, SUM,
                    U, V, ArgumentError, ConfigError, DeviceError, GspmmError, IoError, ParseError,
                    ShapeError, StructureError)
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all

LIB_PATH = _capi.LIB_PATH
__all__ = list(_api_all)
