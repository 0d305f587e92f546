"""ctypes binding of libgfb.so (include/gfb.h).

The product path: every call goes to the sm_100a kernels in
``paper_2212_08200_b200/lib/libgfb.so``.  There is no CPU fallback; a missing
library raises at import/first use.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFB_LIB") or os.path.join(HERE, "lib", "libgfb.so")

GFB_OK, GFB_EINVAL, GFB_ERANGE, GFB_ELOGIC, GFB_ECUDA, GFB_ENOMEM, GFB_ENCCL, GFB_EPARSE = range(8)
W_U32, W_F32, W_F64 = 0, 1, 2
DIR_PUSH, DIR_PULL, DIR_AUTO = 0, 1, 2
SPARSE, DENSE = 0, 1
OP_RELAX_MIN, OP_RECORD, OP_ALWAYS = 0, 1, 2
NIL = 0xFFFFFFFF

# (C ABI function, argtypes) -- every symbol include/gfb.h declares.
_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64
_pu64 = C.POINTER(C.c_uint64)
_int = C.c_int


class SsspOpts(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("direction", C.c_int32), ("pull_alpha", C.c_float),
                ("device_loop", C.c_int32), ("delta", C.c_double), ("compute_pred", C.c_int32),
                ("loop", C.c_int32), ("relabel", C.c_int32), ("defer_pct", C.c_int32),
                ("advance_tile", C.c_int32), ("trace", C.c_int32), ("tail_edges", C.c_int32),
                ("reserved", C.c_int32 * 1)]


class SsspStats(C.Structure):
    _fields_ = [("supersteps", C.c_uint64), ("relaxations", C.c_uint64), ("n_reach", C.c_uint64),
                ("m_reach", C.c_uint64), ("push_steps", C.c_uint64), ("pull_steps", C.c_uint64),
                ("pred_fallback", C.c_uint64), ("device_ms", C.c_double),
                ("advance_ms", C.c_double), ("advance_launches", C.c_uint64),
                ("kernel_launches", C.c_uint64)]


SIGNATURES = {
    "gfb_version": ([], C.c_int),
    "gfb_last_error": ([], C.c_char_p),
    "gfb_ctx_create": ([_int, C.POINTER(_vp)], _int),
    "gfb_ctx_destroy": ([_vp], _int),
    "gfb_ctx_num_sms": ([_vp, C.POINTER(_int)], _int),
    "gfb_graph_upload": ([_vp, _u64, _u64, _vp, _vp, _vp, _int, _int, _int, C.POINTER(_vp)], _int),
    "gfb_graph_refill": ([_vp, _vp, _vp, _vp, _int], _int),
    "gfb_graph_free": ([_vp], _int),
    "gfb_graph_info": ([_vp, _pu64, _pu64, C.POINTER(_int), C.POINTER(_int)], _int),
    "gfb_graph_download": ([_vp, _vp, _vp, _vp], _int),
    "gfb_debug_relabel": ([_vp, _vp, _vp, _vp], _int),
    "gfb_graph_relabel_ranges": ([_vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp], _int),
    "gfb_graph_generate_rmat": ([_vp, _int, _int, _u64, _int, _int, C.POINTER(_vp)], _int),
    "gfb_graph_generate_grid": ([_vp, _u32, _u64, _int, C.POINTER(_vp)], _int),
    "gfb_frontier_create": ([_vp, _u64, _int, C.POINTER(_vp)], _int),
    "gfb_frontier_free": ([_vp], _int),
    "gfb_frontier_assign": ([_vp, _vp, _u64], _int),
    "gfb_frontier_size": ([_vp, _pu64], _int),
    "gfb_frontier_read": ([_vp, _vp, _u64, _pu64], _int),
    "gfb_frontier_repr": ([_vp, C.POINTER(_int)], _int),
    "gfb_dist_create": ([_vp, _vp, C.POINTER(_vp)], _int),
    "gfb_dist_free": ([_vp], _int),
    "gfb_dist_init": ([_vp, _u32], _int),
    "gfb_dist_read": ([_vp, _vp, _pu64], _int),
    "gfb_record_create": ([_vp, _u64, C.POINTER(_vp)], _int),
    "gfb_record_free": ([_vp], _int),
    "gfb_record_read": ([_vp, _vp, _vp, _vp, _u64, _pu64], _int),
    "gfb_advance_push": ([_vp, _vp, _vp, _vp, _int, _vp], _int),
    "gfb_advance_pull": ([_vp, _vp, _vp, _vp, _int, _vp], _int),
    "gfb_filter_unique": ([_vp, _vp, _vp], _int),
    "gfb_filter": ([_vp, _vp, _vp, _int, _vp, C.c_double], _int),
    "gfb_mm_parse": ([C.c_char_p, C.c_size_t, _int, _int, C.POINTER(_vp)], _int),
    "gfb_edge_list_info": ([_vp, _pu64, _pu64], _int),
    "gfb_edge_list_read": ([_vp, _vp, _vp, _vp], _int),
    "gfb_edge_list_free": ([_vp], _int),
    "gfb_last_error_line": ([], C.c_uint64),
    "gfb_graph_from_edges": ([_vp, _u64, _u64, _vp, _vp, _vp, _int, _int, C.POINTER(_vp)], _int),
    "gfb_graph_from_edge_list": ([_vp, _vp, _int, _int, C.POINTER(_vp)], _int),
    "gfb_mg_create_ex": ([_int, _vp, _int, C.POINTER(_vp)], _int),
    "gfb_mg_uses_nccl": ([_vp, C.POINTER(_int)], _int),
    "gfb_sssp_opts_default": ([C.POINTER(SsspOpts)], None),
    "gfb_sssp": ([_vp, _vp, _u32, C.POINTER(SsspOpts), _vp, _vp, C.POINTER(SsspStats)], _int),
    "gfb_sssp_read": ([_vp, _vp, _vp, _vp], _int),
    "gfb_bfs": ([_vp, _vp, _u32, _int, _vp, _pu64, _pu64], _int),
    "gfb_part_create": ([_vp, _u64, _u32, _u32, _u64, _vp, _vp, _vp, _int, _int,
                         C.POINTER(_vp)], _int),
    "gfb_part_free": ([_vp], _int),
    "gfb_part_init": ([_vp, _u32], _int),
    "gfb_part_advance": ([_vp, _vp, _u64, _vp, _int, _vp, _pu64], _int),
    "gfb_part_apply": ([_vp, _vp, _u64], _int),
    "gfb_part_pending": ([_vp, _pu64], _int),
    "gfb_part_read": ([_vp, _vp, _pu64, _pu64], _int),
    "gfb_part_pred": ([_vp, _vp, _vp, _vp, _u32], _int),
    "gfb_peer_create": ([_vp, _int, _int, _vp, _u64, _vp, _vp, _vp, _int, _int, C.POINTER(_vp)],
                        _int),
    "gfb_peer_export": ([_vp, _vp], _int),
    "gfb_peer_link": ([_vp, _vp], _int),
    "gfb_peer_sssp": ([_vp, _u32, C.POINTER(SsspOpts), C.POINTER(SsspStats)], _int),
    "gfb_peer_read": ([_vp, _vp, _vp, _vp], _int),
    "gfb_peer_free": ([_vp], _int),
    "gfb_mg_create": ([_int, _vp, C.POINTER(_vp)], _int),
    "gfb_mg_graph_upload": ([_vp, _u64, _u64, _vp, _vp, _vp, _int, _int], _int),
    "gfb_mg_ranges": ([_vp, _vp], _int),
    "gfb_mg_sssp": ([_vp, _u32, C.POINTER(SsspOpts), _vp, _vp, C.POINTER(SsspStats)], _int),
    "gfb_mg_destroy": ([_vp], _int),
}

PEER_HANDLE_BYTES = 64

_LIB = None


def load():
    """Load libgfb.so (raises if it was never built: no fallback path)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


class GfbError(RuntimeError):
    code = GFB_ECUDA


def _exc(code, msg):
    """Map a gfb_status to the exception type the reference throws."""
    if code == GFB_EINVAL:
        e = ValueError(msg)          # std::invalid_argument
    elif code == GFB_ERANGE:
        e = IndexError(msg)          # std::out_of_range
    elif code == GFB_ELOGIC:
        e = GfbLogicError(msg)       # std::logic_error
    elif code == GFB_EPARSE:
        e = ParseError(msg, int(load().gfb_last_error_line()))  # graflow::ParseError
    else:
        e = GfbError(msg)            # std::runtime_error
    e.gfb_code = code
    return e


class GfbLogicError(RuntimeError):
    pass


class ParseError(RuntimeError):
    """graflow::ParseError (io.hpp:27-36): message "line N: ...", .line."""

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


def check(code):
    if code != GFB_OK:
        raise _exc(code, load().gfb_last_error().decode(errors="replace"))
