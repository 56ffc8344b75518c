"""ctypes binding of libmgp.so (include/megopolis_b200.h).

The library is built in-tree (``python -m paper_2109_13504_b200.build`` or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or no CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmgp.so")

MGP_F32, MGP_F64 = 0, 1
RNG = {"megores": 0, "philox": 1}
KIND = {"metropolis": 0, "c1": 1, "c2": 2, "megopolis": 3, "multinomial": 4, "systematic": 5}
MGP_EINVAL, MGP_EUNSUPPORTED = -1, -2
FLAG_NONZERO = 1
FLAG_NO_STAGE = 2

_lib = None
_lock = threading.Lock()

_u64, _i64, _i32, _vp, _dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double

# name -> (restype, argtypes); mirrors include/megopolis_b200.h one to one
SIGNATURES = {
    "mgp_abi_version": (_i32, []),
    "mgp_last_error": (ctypes.c_char_p, []),
    "mgp_release_cached_memory": (_i32, [_i32]),
    "mgp_check_host_weights": (_i32, [_vp, _i32, _i64, _vp]),
    "mgp_weight_stats": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "mgp_compute_iterations": (_i32, [_dbl, _dbl, _dbl, _vp]),
    "mgp_offsets_host": (_i32, [_u64, _i64, _i32, _i32, _vp]),
    "mgp_offsets": (_i32, [_u64, _i64, _i32, _i32, _vp, _vp]),
    "mgp_megopolis": (_i32, [_vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _vp, _vp]),
    "mgp_metropolis": (_i32, [_vp, _i32, _i64, _i32, _u64, _i32, _i32, _vp, _vp]),
    "mgp_metropolis_c1": (_i32, [_vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "mgp_metropolis_c2": (_i32, [_vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "mgp_resample_range": (_i32, [_i32, _vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _vp,
                                   _vp]),
    "mgp_resample_gather": (_i32, [_i32, _vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _i32, _i32, _i64, _i64,
                                    _vp, _i32, _i64, _i64, _vp, _vp, _vp]),
    "mgp_resample_multi": (_i32, [_i32, _vp, _i32, _i64, _i32, _dbl, _u64, _i32, _i32, _i32, _i32, _i32, _vp, _vp,
                                  _vp]),
    "mgp_resample_stripes": (_i32, [_i32, _vp, _i32, _i64, _i32, _u64, _i32, _i32, _i32, _i32, _i32, _i64, _i64,
                                     _vp, _vp]),
    "mgp_resample_host": (_i32, [_i32, _vp, _i32, _i64, _i32, _dbl, _u64, _i32, _i32, _i32, _i32, _vp, _vp, _i32]),
    "mgp_resample_host_batch": (_i32, [_i32, _vp, _i32, _i64, _i32, _i32, _dbl, _vp, _i32, _i32, _i32, _i32, _vp, _vp,
                                       _i32]),
    "mgp_offspring": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "mgp_expected_offspring": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp]),
    "mgp_expected_offspring_slice": (_i32, [_vp, _i32, _i64, _i64, _dbl, _vp, _vp]),
    "mgp_quality_add": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "mgp_quality_finalize": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "mgp_quality_runs": (_i32, [_i32, _vp, _i32, _i64, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                 _vp, _vp]),
    "mgp_squared_error": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "mgp_gather": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "mgp_gather_peers": (_i32, [_vp, _i32, _i64, _i64, _vp, _i64, _vp, _vp]),
    "mgp_comparison_indices": (_i32, [_i32, _i64, _i32, _u64, _i32, _i32, _i32, _vp, _vp]),
    "mgp_traffic_report": (_i32, [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _vp]),
    "mgp_ipc_export": (_i32, [_vp, _vp, _vp]),
    "mgp_ipc_open": (_i32, [_vp, _i64, _vp]),
    "mgp_ipc_close": (_i32, [_vp, _i64]),
    "mgp_mean": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "mgp_pf_init": (_i32, [_i64, _u64, _dbl, _vp, _vp]),
    "mgp_pf_predict_update": (_i32, [_vp, _i64, _dbl, _dbl, _u64, _dbl, _dbl, _i32, _vp, _vp, _vp, _vp]),
    "mgp_estimate_ratio_stats": (_i32, [_vp, _i32, _i64, _i64, _u64, _vp, _vp]),
    "mgp_gen_gaussian": (_i32, [_dbl, _i64, _u64, _i32, _vp, _vp]),
    "mgp_gen_gamma": (_i32, [_dbl, _dbl, _i64, _u64, _i32, _vp, _vp]),
    "mgp_cumsum": (_i32, [_vp, _i32, _i64, _vp, _vp]),
    "mgp_multinomial": (_i32, [_vp, _i32, _i64, _u64, _vp, _vp]),
    "mgp_systematic": (_i32, [_vp, _i32, _i64, _u64, _vp, _vp]),
    "mgp_systematic_oracle": (_i32, [_vp, _i32, _i64, _dbl, _vp, _vp]),
    "mgp_philox_selftest": (_i32, [_u64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _i64, _vp]),
    "mgp_debug_megores_fallbacks": (_i32, [_vp, ctypes.c_int]),
    "mgp_debug_px_prof": (_i32, [_vp, ctypes.c_int]),
    "mgp_debug_offspring_mode": (_i32, [ctypes.c_int]),
}


class MgpError(RuntimeError):
    """A CUDA-side failure reported by libmgp.so."""


def lib():
    """Load libmgp.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_2109_13504_b200.build` "
                        "(there is no CPU fallback)"
                    )
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a libmgp return code onto the reference's exception types."""
    if rc == 0:
        return
    msg = lib().mgp_last_error().decode("utf-8", "replace")
    if rc == MGP_EINVAL:
        raise ValueError(msg)
    if rc == MGP_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise MgpError(msg)
