"""ctypes binding of libmoep_b200.so (the C ABI in include/moep_b200.h).

The product path has no fallback: if the library is missing or no CUDA device
is present, every compute entry point raises. Struct layouts below mirror the
header field for field.
"""

from __future__ import annotations

import ctypes as C
import os

from .exceptions import ConfigurationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoep_b200.so")

MOEP_OK, MOEP_ESHAPE, MOEP_EALIGN, MOEP_EUNSUPPORTED, MOEP_ELAUNCH, MOEP_EARG = 0, -1, -2, -3, -4, -5
MOEP_BF16, MOEP_F64, MOEP_F32 = 1, 2, 3
MAX_BOUNDS = 4

EXPORTED = (
    "moep_predict_bf16", "moep_predict_fp64", "moep_eval_logits", "moep_topk_logits",
    "moep_counters_reduce", "moep_rank_order", "moep_input_norm", "moep_num_sms", "moep_version",
    "moep_labels", "moep_loss", "moep_act_backward", "moep_optim_step", "moep_forward_train",
    "moep_prefetch_plan", "moep_gather_rows",
)

vp = C.c_void_p
i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double


class PredictArgs(C.Structure):
    _fields_ = [
        ("n_tokens", i64), ("d", i32), ("hidden", i32), ("n_experts", i32), ("arch", i32),
        ("x", vp), ("w1", vp), ("b1", vp), ("act_alpha", vp), ("act_beta", vp), ("w2", vp), ("b2", vp),
        ("m_sel", i32), ("n_bounds", i32), ("bounds", i32 * MAX_BOUNDS),
        ("tau_abs", f32), ("tau_rel", f32), ("w2_norm", f32),
        ("ids", vp), ("logits", vp), ("flags", vp), ("flag_list", vp), ("flag_count", vp),
        ("truth", vp), ("k", i32), ("n_m", i32), ("m_list", i32 * MAX_BOUNDS), ("partials", vp),
    ]


class Fp64Args(C.Structure):
    _fields_ = [
        ("n_tokens", i64), ("d", i32), ("hidden", i32), ("n_experts", i32), ("arch", i32),
        ("x_dtype", i32), ("w_dtype", i32),
        ("x", vp), ("w1", vp), ("b1", vp), ("bn_scale", vp), ("bn_shift", vp), ("bn_mean", vp),
        ("bn_var", vp), ("bn_eps", f64), ("w2", vp), ("b2", vp),
        ("rows", vp), ("row_count", vp), ("m_sel", i32), ("ids", vp), ("logits64", vp), ("logits32", vp),
        ("truth", vp), ("k", i32), ("n_m", i32), ("m_list", i32 * MAX_BOUNDS), ("partials", vp),
    ]


_lib = None


def lib():
    """Load the library once; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2511_10676_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.moep_predict_bf16.argtypes = [C.POINTER(PredictArgs), vp]
        L.moep_predict_fp64.argtypes = [C.POINTER(Fp64Args), vp]
        L.moep_eval_logits.argtypes = [vp, i32, i64, i32, vp, i32, i32, vp, vp, vp]
        L.moep_topk_logits.argtypes = [vp, i32, i64, i32, i32, vp, vp]
        L.moep_rank_order.argtypes = [vp, i32, i64, i32, vp, vp]
        L.moep_counters_reduce.argtypes = [vp, i32, i32, vp, vp]
        L.moep_input_norm.argtypes = [vp, i32, i64, i32, i32, vp, vp, f64, vp, vp, vp]
        L.moep_num_sms.argtypes = []
        L.moep_version.restype = C.c_char_p
        for name in EXPORTED:
            if hasattr(L, name):
                getattr(L, name).restype = getattr(L, name).restype if name == "moep_version" else i32
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == MOEP_OK:
        return
    if rc in (MOEP_ESHAPE, MOEP_EALIGN):
        raise ConfigurationError(f"{what}: shape/alignment rejected by the kernel (code {rc})")
    if rc in (MOEP_EUNSUPPORTED, MOEP_EARG):
        raise ValueError(f"{what}: unsupported argument (code {rc})")
    raise RuntimeError(f"{what}: CUDA launch failed (code {rc})")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
