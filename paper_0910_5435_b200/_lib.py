"""Loader for libbfly_b200.so (the C ABI declared in include/bfly_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_0910_5435_b200/csrc``).  There is no fallback: if the library
is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BFLY_LIB") or os.path.join(HERE, "libbfly_b200.so")  # BFLY_LIB: tuning builds

BFLY_OK, BFLY_EINVAL, BFLY_ERUNTIME, BFLY_ESERIAL, BFLY_ECUDA, BFLY_ENCCL, BFLY_EOTHER = range(7)

# Every symbol include/bfly_b200.h declares: name -> (restype, argtypes)
_vp, _i64, _i32, _dbl, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_size_t
_dp = C.POINTER(C.c_double)
_pp = C.POINTER(C.c_void_p)
SIGNATURES = {
    "bfly_last_error": (C.c_char_p, []),
    "bfly_version": (C.c_char_p, []),
    "bfly_plan_from_bfly1": (_i32, [C.c_char_p, _sz, _pp]),
    "bfly_plan_to_bfly1": (_i32, [_vp, C.c_char_p, _sz, C.POINTER(_sz)]),
    "bfly_plan_build_glrow": (_i32, [_i32, _i32, _i32, _dbl, _i32, _pp]),
    "bfly_plan_build_dense": (_i32, [_dp, _i64, _i64, _dbl, _i32, _pp]),
    "bfly_plan_info": (_i32, [_vp, C.POINTER(_i64), _dp]),
    "bfly_plan_destroy": (None, [_vp]),
    "bfly_dev_planset_create": (_i32, [_pp, _i32, _i32, _pp]),
    "bfly_dev_apply": (_i32, [_vp, _i32, _vp, _i64, _vp, _i64, _i32, _vp]),
    "bfly_host_apply": (_i32, [_vp, _i32, _dp, _i64, _dp, _i64, _i32]),
    "bfly_dev_planset_info": (_i32, [_vp, C.POINTER(_i64)]),
    "bfly_dev_planset_destroy": (None, [_vp]),
    "bfly_sht_create": (_i32, [_i32, _dbl, _i32, _i32, _i32, _pp]),
    "bfly_sht_create_from_plans": (_i32, [_i32, _pp, _i32, _dp, _i32, _pp]),
    "bfly_sht_create_rule": (_i32, [_i32, _dbl, _i32, _i32, _dp, _dp, _i32, _pp]),
    "bfly_sht_synthesize": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_analyze": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_legendre_synthesize": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_legendre_analyze": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_phi_synthesize": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_synthesize_real": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_analyze_real": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_phi_analyze": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_synthesize_host": (_i32, [_vp, _dp, _dp, _i32]),
    "bfly_sht_analyze_host": (_i32, [_vp, _dp, _dp, _i32]),
    "bfly_sht_info": (_i32, [_vp, C.POINTER(_i64)]),
    "bfly_sht_program_info": (_i32, [_vp, C.POINTER(_i64)]),
    "bfly_sht_rule": (_i32, [_vp, _dp, _dp]),
    "bfly_sht_trace": (_i32, [_vp, _i32]),
    "bfly_sht_debug": (_i32, [_vp, _i32]),
    "bfly_sht_engine_time": (_i32, [_vp, _i32, _dp, C.POINTER(_i64)]),
    "bfly_sht_trace_read": (_i32, [_vp, _vp, _i32]),
    "bfly_sht_destroy": (None, [_vp]),
    "bfly_sht_save": (_i32, [_vp, C.c_char_p]),
    "bfly_sht_load": (_i32, [C.c_char_p, _i32, _pp]),
    "bfly_glrow_planset_build": (_i32, [_i32, _i32, _i32, _dbl, _i32, _i32, _pp, _i32,
                                        C.POINTER(_i32)]),
    "bfly_glrow_planset_build_rule": (_i32, [_i32, _i32, _i32, _dbl, _i32, _i32, _dp, _dp, _pp, _i32,
                                             C.POINTER(_i32)]),
    "bfly_gl_rule": (_i32, [_i32, _dp, _dp]),
    "bfly_phi_time": (_i32, [_i32, _i32, _i32, _dp]),
    "bfly_shard_last_error": (C.c_char_p, []),
    "bfly_shard_layout": (_i32, [_i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "bfly_shard_tables": (_i32, [_i32, _i32, _i32, _i32, C.POINTER(_i64), C.POINTER(C.c_int32), C.POINTER(_i64),
                                 C.POINTER(_i64), C.POINTER(_i64)]),
    "bfly_shard_nccl_id": (_i32, [_vp]),
    "bfly_shard_create": (_i32, [_i32, _dbl, _i32, _i32, _i32, _i32, _vp, _i32, _pp]),
    "bfly_shard_info": (_i32, [_vp, C.POINTER(_i64)]),
    "bfly_shard_sht": (_i32, [_vp, _pp]),
    "bfly_shard_synthesize": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_shard_analyze": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "bfly_shard_destroy": (None, [_vp]),
    "bfly_pack_inspect": (_i32, [_pp, _i32, _vp, _vp, _vp, _vp, C.POINTER(_i64)]),
    "bfly_waves_inspect": (_i32, [_pp, _i32, C.POINTER(_i64), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bfly_pack_inspect_split": (_i32, [_pp, _i32, C.POINTER(_i32), _i32, _vp, _vp, _vp, _vp, C.POINTER(_i64),
                                       _vp, _vp]),
    "bfly_sht_create_range": (_i32, [_i32, _i32, _i32, _pp, _i32, _dp, _i32, _pp]),
    "bfly_sht_shard_supported": (_i32, [_vp, _vp]),
    "bfly_sht_shard_synthesize": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "bfly_sht_shard_phi": (_i32, [_vp, _i32, _vp, _vp, _vp, _i32, _i32, _vp]),
    "bfly_sht_shard_analyze": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _vp]),
}


class BflyError(RuntimeError):
    """A BFLY_E* status from the library."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class BflyInvalidArgument(BflyError, ValueError):
    """BFLY_EINVAL — the reference's std::invalid_argument."""


class BflySerializationError(BflyError):
    """BFLY_ESERIAL — the reference's bfly::SerializationError."""


class BflyCudaError(BflyError):
    """BFLY_ECUDA."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == BFLY_OK:
        return
    msg = lib().bfly_last_error().decode()
    cls = {BFLY_EINVAL: BflyInvalidArgument, BFLY_ESERIAL: BflySerializationError,
           BFLY_ECUDA: BflyCudaError}.get(rc, BflyError)
    raise cls(rc, msg)


def dptr(a):
    """ctypes double* of a C-contiguous float64 numpy array."""
    return a.ctypes.data_as(_dp)
