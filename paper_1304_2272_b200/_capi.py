"""ctypes binding of libgwasgls_b200.so (the C-ABI in include/gwasgls_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA device is present,
``lib()`` / ``device()`` raise ``DeviceError`` loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError, DimensionMismatch

HERE = os.path.dirname(os.path.abspath(__file__))
# GG_LIB_PATH: load another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("GG_LIB_PATH") or os.path.join(HERE, "libgwasgls_b200.so")

GG_OK, GG_ENOTPD, GG_EDIM, GG_ECUDA, GG_ENCCL, GG_EARG = 0, 1, 2, 3, 4, 5
GG_TILE = 128
GG_PMAX = 20

_vp, _i, _ll, _d, _sz = C.c_void_p, C.c_int, C.c_longlong, C.c_double, C.c_size_t
_ull = C.c_ulonglong
_ip = C.POINTER(C.c_int)

# name -> (restype, argtypes); every entry point of include/gwasgls_b200.h
SIGNATURES = {
    "gg_version": (C.c_char_p, []),
    "gg_last_error": (C.c_char_p, []),
    "gg_pad": (_i, [_i]),
    "gg_potrf_workspace_bytes": (_sz, [_i]),
    "gg_potrf_f64": (_i, [_i, _vp, _i, _i, _vp, _vp, _i, _vp, _ip, _vp]),
    "gg_trtri_workspace_bytes": (_sz, [_i]),
    "gg_trtri_lower_f64": (_i, [_i, _vp, _i, _vp, _i, _vp, _vp]),
    "gg_trsm_lower_blocked_workspace_bytes": (_sz, [_i, _i]),
    "gg_trsm_lower_blocked_f64": (_i, [_i, _i, _vp, _i, _vp, _i, _vp, _i, _vp, _vp]),
    "gg_trsm_lower_f64": (_i, [_i, _i, _vp, _i, _vp, _i, _vp, _i, _vp]),
    "gg_trsm_lower_rm_f64": (_i, [_i, _i, _vp, _i, _vp, _i, _vp, _i, _vp]),
    "gg_packed_lower_bytes": (_sz, [_i]),
    "gg_pack_lower_f64": (_i, [_i, _vp, _i, _i, _vp, _vp]),
    "gg_pack_lower_blockcyclic_f64": (_i, [_i, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "gg_trsm_lower_packed_f64": (_i, [_i, _i, _vp, _vp, _i, _vp, _i, _vp]),
    "gg_i8_slices": (_i, []),
    "gg_i8_value_bound": (_i, [_i]),
    "gg_slice_packed_inverse_i8": (_i, [_i, _vp, _vp, _vp, _vp]),
    "gg_row_exponents_blockcyclic": (_i, [_i, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "gg_slice_blockcyclic_i8": (_i, [_i, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp, _vp]),
    "gg_inverse_slices_bytes": (_sz, [_i]),
    "gg_slice_meta_ints": (_sz, [_i]),
    "gg_slice_meta_i8": (_i, [_i, _vp, _vp, _vp]),
    "gg_slice_inverse_i8": (_i, [_i, _vp, _i, _vp, _vp, _vp]),
    "gg_narrow_f64_i8": (_i, [_i, _i, _vp, _ll, _vp, _ll, _vp, _vp]),
    "gg_trsm_i8_workspace_bytes": (_sz, []),
    "gg_trsm_lower_i8": (_i, [_i, _i, _vp, _vp, _vp, _ll, _vp, _i, _vp, _vp]),
    "gg_partials_bytes": (_sz, [_i, _i, _i]),
    "gg_trsm_lower_i8_partials": (_i, [_i, _i, _vp, _vp, _vp, _ll, _i, _vp, _vp, _vp, _vp, _i,
                                       _vp, _i, _vp, _vp]),
    "gg_gls_reduce_solve_f64": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gg_transpose_f64": (_i, [_i, _vp, _i, _vp, _i, _vp]),
    "gg_dgemm_f64": (_i, [_i, _i, _i, _d, _vp, _i, _vp, _i, _i, _d, _vp, _i, _vp]),
    "gg_gemm_ozaki_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "gg_gemm_ozaki_f64": (_i, [_i, _i, _i, _vp, _ll, _ll, _vp, _ll, _ll, _vp, _ll, _d, _d, _i,
                               _vp, _sz, _vp]),
    "gg_widen_i8_f64": (_i, [_i, _i, _vp, _ll, _vp, _i, _vp]),
    "gg_gls_dots_f64": (_i, [_i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _vp, _vp]),
    "gg_small_spd_solve_f64": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "gg_gls_epilogue_f64": (_i, [_i, _i, _i, _vp, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp]),
    "gg_gls_block_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "gg_gls_block_f64": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _ll,
                              _vp, _vp, _vp, _vp, _vp]),
    "gg_memcpy2d_async": (_i, [_vp, _sz, _vp, _sz, _sz, _sz, _i, _vp]),
    "gg_gen_genotypes_i8": (_i, [_ull, _i, _i, _i, _ll, _ll, _i, _d, _d, _vp, _ll, _vp, _i,
                                 _vp]),
    # distributed Cholesky + inverse (csrc/dist_native.cu)
    "gg_dist_nccl_unique_id": (_i, [_vp]),
    "gg_dist_comms_nccl": (_i, [_i, _i, _i, _i, _vp, _vp]),
    "gg_dist_comms_callbacks": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "gg_dist_comms_free": (_i, [_vp]),
    "gg_dist_local_dims": (_i, [_i, _i, _vp, _ip, _ip]),
    "gg_dist_potrf_workspace_bytes": (_sz, [_i, _i, _vp]),
    "gg_dist_potrf_f64": (_i, [_i, _i, _vp, _ll, _vp, _ll, _vp, _vp, _sz, _ip, _vp]),
    "gg_dist_trsm_workspace_bytes": (_sz, [_i, _i, _i, _vp]),
    "gg_dist_trsm_f64": (_i, [_i, _i, _i, _vp, _ll, _vp, _ll, _vp, _vp, _sz, _vp]),
}
# callback types of gg_dist_comms_callbacks (group 0 world, 1 process row, 2 process column)
DIST_BCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_int)
DIST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t)

_lock = threading.Lock()
_lib = None


def load_library(path=LIB_PATH):
    """Load the shared library and bind every exported symbol (no GPU needed)."""
    if not os.path.exists(path):
        raise DeviceError(
            f"native library {path} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _CheckedLib:
    """Arity-checked view of the library: ctypes forwards surplus arguments to a C function
    silently (the last one would be taken as the stream); refuse them instead."""

    def __init__(self, cdll):
        self._cdll = cdll

    def __getattr__(self, name):
        fn = getattr(self._cdll, name)
        want = len(SIGNATURES[name][1]) if name in SIGNATURES else None

        def call(*args):
            if want is not None and len(args) != want:
                raise TypeError(f"{name} takes {want} arguments ({len(args)} given)")
            return fn(*args)

        call.__name__ = name
        setattr(self, name, call)
        return call


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = _CheckedLib(load_library())
    return _lib


def last_error():
    msg = lib().gg_last_error()
    return msg.decode() if msg else ""


def check(rc, what):
    """Map a C-ABI status to the package's exceptions."""
    if rc == GG_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == GG_EDIM:
        raise DimensionMismatch(msg)
    if rc == GG_EARG:
        raise ValueError(msg)
    raise DeviceError(msg)


def pad(n):
    return ((int(n) + GG_TILE - 1) // GG_TILE) * GG_TILE


def device():
    """The CUDA device the product path runs on (current torch device)."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the gwasgls B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    import torch

    return _vp(torch.cuda.current_stream().cuda_stream)


def i8_work(device=None):
    """A fresh workspace for one gg_trsm_lower_i8* launch (its tile counter), from torch's
    caching allocator on the current device."""
    import torch

    n = int(lib().gg_trsm_i8_workspace_bytes())
    return torch.empty(n, dtype=torch.uint8, device=device or _dev_now())


def _dev_now():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def ptr(t):
    """Raw device pointer of a torch tensor (or None)."""
    return None if t is None else _vp(t.data_ptr())
