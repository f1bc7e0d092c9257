"""ctypes binding of libmoep_b200.so (the C ABI in include/moep_b200.h).

The product path has no fallback: if the library is missing or no CUDA device
is present, every compute entry point raises. Struct layouts below mirror the
header field for field (tests/test_capi.py checks sizes and offsets against a
C compiler).
"""

from __future__ import annotations

import ctypes as C
import os

from .exceptions import ConfigurationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOEP_LIB: alternative build of the same library (tools/variant_lib.py, tools/k1_prof.py)
LIB_PATH = os.environ.get("MOEP_LIB") or os.path.join(_HERE, "libmoep_b200.so")

MOEP_OK, MOEP_ESHAPE, MOEP_EALIGN, MOEP_EUNSUPPORTED, MOEP_ELAUNCH, MOEP_EARG = 0, -1, -2, -3, -4, -5
MOEP_BF16, MOEP_F64, MOEP_F32 = 1, 2, 3
MAX_BOUNDS = 4

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
        ("a_out", vp), ("split_scratch", vp), ("split_scratch_floats", i64), ("status", vp), ("kernel", i32), ("probs", vp),
    ]


MOEP_K1_AUTO, MOEP_K1_ONE_SM, MOEP_K1_PAIR_V2, MOEP_K1_PAIR_V4, MOEP_K1_QUAD_V5 = 0, 1, 2, 4, 5


class Fp64Args(C.Structure):
    _fields_ = [
        ("n_tokens", i64), ("d", i32), ("hidden", i32), ("n_experts", i32), ("arch", i32),
        ("x_dtype", i32), ("w_dtype", i32),
        ("x", vp), ("w1", vp), ("b1", vp), ("bn_scale", vp), ("bn_shift", vp), ("bn_mean", vp),
        ("bn_var", vp), ("bn_eps", f64), ("w2", vp), ("w2t", vp), ("b2", vp),
        ("rows", vp), ("row_count", vp), ("m_sel", i32), ("ids", vp), ("logits64", vp), ("logits32", vp),
        ("truth", vp), ("k", i32), ("n_m", i32), ("m_list", i32 * MAX_BOUNDS), ("partials", vp),
        ("a_out", vp), ("row_begin", i64),
    ]


class LossArgs(C.Structure):
    _fields_ = [
        ("family", i32),
        ("top_weight", f64), ("mid_weight", f64), ("rest_weight", f64), ("ranking_lambda", f64),
        ("margin", f64), ("focal_gamma", f64), ("focal_alpha", f64),
        ("normalize_ranking", i32), ("n", i64), ("n_global", i64), ("n_experts", i32), ("dtype", i32),
        ("logits", vp), ("scores", vp), ("rank_of", vp), ("topk_mask", vp), ("dz", vp), ("dz_hinge", vp),
        ("partials", vp), ("n_blocks", i32),
    ]


class OptimArgs(C.Structure):
    _fields_ = [
        ("kind", i32), ("dtype", i32), ("n", i64), ("params", vp), ("grads", vp), ("m", vp), ("v", vp),
        ("lr", f64), ("beta1", f64), ("beta2", f64), ("eps", f64), ("momentum", f64), ("t", i64),
        ("shadow_bf16", vp), ("n_shadow", i64), ("nonfinite", vp),
    ]


# name -> argtypes (restype int32 unless listed in _RESTYPES)
_SIGS = {
    "moep_predict_bf16": [C.POINTER(PredictArgs), vp],
    "moep_predict_fp64": [C.POINTER(Fp64Args), vp],
    "moep_fixup_fp64": [C.POINTER(Fp64Args), vp, i64, vp, vp],
    "moep_decode_fp64": [C.POINTER(Fp64Args), vp, vp],
    "moep_predict_split_floats": [i64, i32, i32],
    "moep_eval_logits": [vp, i32, i64, i32, vp, i32, i32, vp, vp, vp],
    "moep_topk_logits": [vp, i32, i64, i32, i32, vp, vp],
    "moep_rank_order": [vp, i32, i64, i32, vp, vp],
    "moep_counters_reduce": [vp, i32, i32, vp, vp],
    "moep_input_norm": [vp, i32, i64, i32, i32, vp, vp, f64, vp, vp, vp],
    "moep_labels": [vp, i32, i64, i32, i32, vp, vp, vp, vp],
    "moep_loss": [C.POINTER(LossArgs), vp],
    "moep_loss_finalize": [vp, i32, i64, i32, i32, f64, i32, i32, vp, vp, vp, vp],
    "moep_act_backward": [vp, vp, vp, i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp],
    "moep_act_backward_bf16split": [vp, vp, vp, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp],
    "moep_optim_step": [C.POINTER(OptimArgs), vp],
    "moep_bn_forward": [vp, i64, i32, vp, vp, vp, vp, f64, f64, f64, C.c_uint64, C.c_uint64, vp, vp, vp, vp,
                        vp, vp, i32, vp],
    "moep_rows_dot": [vp, vp, vp, i64, i32, i32, vp, vp],
    "moep_bn_backward": [vp, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp],
    "moep_prefetch_plan": [vp, i64, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp],
    "moep_prefetch_commit": [vp, vp, vp, vp, vp, vp],
    "moep_gather_experts": [vp, i64, vp, vp, vp, vp, i32, vp],
    "moep_trace_ingest": [vp, i64, i32, i32, i32, i32, vp, vp, vp, i64, vp, vp],
    "moep_teacher_normals": [C.c_uint64, i64, i64, i32, i32, vp, vp, vp, vp],
    "moep_layer_norm_np": [vp, i64, i32, f64, vp, vp],
    "moep_dgemm_nt": [vp, i64, vp, i64, vp, i64, i64, i64, i64, i32, vp],
    "moep_dgemm_tn": [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp],
    "moep_dw1_workspace_floats": [i32, i32, i64, i32],
    "moep_dw1_bf16": [vp, vp, i64, i32, i32, i32, vp, vp, i64, vp],
    "moep_softmax_np": [vp, i64, i32, vp, vp],
    "moep_teacher_finish": [vp, i64, i32, i32, vp, vp, vp],
    "moep_num_sms": [],
    "moep_version": [],
}
_RESTYPES = {"moep_version": C.c_char_p, "moep_predict_split_floats": i64, "moep_dw1_workspace_floats": i64}
EXPORTED = tuple(_SIGS)

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
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, i32)
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


def dtype_code(t) -> int:
    import torch
    return {torch.float64: MOEP_F64, torch.float32: MOEP_F32, torch.bfloat16: MOEP_BF16}[t.dtype]
