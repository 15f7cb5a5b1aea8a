"""ctypes binding of libmonoiga_b200.so (the C ABI in include/monoiga_b200.h).

There is no CPU fallback: if the library cannot be loaded or a call fails,
an ExtensionError (or the reference exception the status maps to) is raised.
"""

import ctypes
import os

from .errors import ExtensionError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmonoiga_b200.so")

MI_OK, MI_ERR_ARG, MI_ERR_CUDA, MI_ERR_STATE = 0, 1, 2, 3

_c_int, _c_ll, _c_dbl, _vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)

_SIGS = {
    "mi_version": ([], _c_int),
    "mi_last_error": ([], ctypes.c_char_p),
    "mi_diag_fp64_peak": ([_c_int, _c_int, _vp, _vp], _c_int),
    "mi_ctx_create": ([_c_int, _c_int, _vp, _c_int, _c_int, _c_int, ctypes.POINTER(_vp)], _c_int),
    "mi_ctx_destroy": ([_vp], _c_int),
    "mi_ctx_set_stream": ([_vp, _vp], _c_int),
    "mi_ctx_set_zslab": ([_vp, _c_int, _c_int, _c_int, _c_int], _c_int),
    "mi_prof_enable": ([_vp, _c_int], _c_int),
    "mi_prof_read": ([_vp, _vp, _vp, _c_int], _c_int),
    "mi_op_setup": ([_vp, _c_int], _c_int),
    "mi_op_set_time_bands": ([_vp, _vp], _c_int),
    "mi_op_set_kron_channel": ([_vp, _c_int, _c_int, _vp, _vp], _c_int),
    "mi_op_set_su_channel": ([_vp, _c_int, _vp, _vp, _c_int], _c_int),
    "mi_op_apply": ([_vp, _vp, _vp], _c_int),
    "mi_op_apply_from_host": ([_vp, _vp, _vp, _vp, _c_int], _c_int),
    "mi_op_set_reaction": ([_vp, _vp, _vp, _c_dbl, _c_dbl, _c_dbl, _vp, _vp, _vp, _vp], _c_int),
    "mi_op_clear_reaction": ([_vp], _c_int),
    "mi_op_set_lift": ([_vp, _vp, _vp], _c_int),
    "mi_op_finalize": ([_vp, _c_int], _c_int),
    "mi_op_apply_lift": ([_vp, _vp], _c_int),
    "mi_theta_set_lift": ([_vp, _vp], _c_int),
    "mi_op_set_reaction_weight": ([_vp, _vp], _c_int),
    "mi_op_set_reaction_store": ([_vp, _c_int], _c_int),
    "mi_op_set_reaction_kernel": ([_vp, _c_int], _c_int),
    "mi_op_set_quad_channel": ([_vp, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp], _c_int),
    "mi_op_set_quad_channel_k": ([_vp, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp], _c_int),
    "mi_op_set_channel_stencil": ([_vp, _c_int, _vp], _c_int),
    "mi_op_get_channel_stencil": ([_vp, _c_int, _vp], _c_int),
    "mi_op_set_reaction_rows": ([_vp, _c_int], _c_int),
    "mi_pc_setup": ([_vp, _vp, _vp, _c_dbl, _c_dbl, _vp, _vp, _vp, _vp, _vp, _vp, _c_dbl], _c_int),
    "mi_pc_apply": ([_vp, _vp, _vp], _c_int),
    "mi_pc_apply_spatial": ([_vp, _vp, _vp, _c_ll, _c_int], _c_int),
    "mi_pc_apply_time": ([_vp, _vp, _c_ll, _c_ll], _c_int),
    "mi_pc_apply_time_yslab": ([_vp, _vp, _c_int, _c_int], _c_int),
    "mi_pc_mode": ([_vp, _c_int, _c_int, _vp, _vp, _c_ll, _c_ll], _c_int),
    "mi_pc_fold": ([_vp, _c_int], _c_int),
    "mi_pc_mode_mapped": ([_vp, _c_int, _c_int, _vp, _vp, _c_ll, _c_ll, _vp, _vp], _c_int),
    "mi_ws_setup": ([_vp, _vp, _vp, _vp], _c_int),
    "mi_ws_time": ([_vp, _vp, _vp], _c_int),
    "mi_ws_mass": ([_vp, _vp, _vp, _c_ll, _c_int], _c_int),
    "mi_rowdots": ([_vp, _c_ll, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_row_axpy": ([_vp, _c_ll, _c_ll, _vp, _c_dbl, _vp, _vp], _c_int),
    "mi_row_xpby": ([_vp, _c_ll, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_dots": ([_vp, _c_ll, _c_int, _vp, _c_ll, _vp, _vp], _c_int),
    "mi_sub_combination": ([_vp, _c_ll, _c_int, _vp, _c_ll, _vp, _vp], _c_int),
    "mi_combination": ([_vp, _c_ll, _c_int, _vp, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_scale_inv": ([_vp, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_normalize": ([_vp, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_cgs_pass": ([_vp, _c_ll, _c_int, _vp, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_cgs_norm_pass": ([_vp, _c_ll, _c_int, _vp, _c_ll, _vp, _vp, _vp], _c_int),
    "mi_theta_setup": ([_vp, _vp, _vp, _vp, _vp, _vp, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_dbl], _c_int),
    "mi_theta_elements": ([_vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _vp], _c_int),
    "mi_theta_mapped_elements": ([_vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _vp, _vp], _c_int),
    "mi_window_max": ([_vp, _vp, _vp, _c_ll, _c_int, _c_int, _c_ll, _vp, _vp], _c_int),
    "mi_theta_ratio": ([_vp, _vp, _vp, _c_ll, _c_dbl], _c_int),
}

EXPORTED = tuple(_SIGS)

PROF_SLOTS = ("op_stencil", "op_time_filter", "op_reaction", "pc_spatial", "pc_time", "pc_arrowhead",
              "krylov", "setup")

_lib = None


def load():
    """Load (once) and return the ctypes library; raise ExtensionError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionError("libmonoiga_b200.so not built (%s); run "
                             "`python -m paper_2311_17500_b200.build`" % LIB_PATH)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise ExtensionError("cannot load %s: %s" % (LIB_PATH, exc)) from exc
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc, what=""):
    if rc == MI_OK:
        return
    msg = load().mi_last_error().decode(errors="replace")
    if rc == MI_ERR_ARG:
        raise ValueError("%s: %s" % (what, msg) if what else msg)
    raise ExtensionError("%s failed (status %d): %s" % (what, rc, msg))


def call(name, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
