"""ctypes binding of the C ABI in include/tk_render.h.

The product path is the CUDA library lib/libtkrender.so; there is no CPU fallback.  Loading
fails loudly if the library is missing (run ``python -m paper_2602_06991_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
# TK_RENDER_LIB: load an alternative build of the same library (A/B kernel experiments)
RENDER_LIB = os.environ.get("TK_RENDER_LIB") or os.path.join(LIB_DIR, "libtkrender.so")

TK_HOST, TK_DEVICE, TK_HOST_ASYNC = 0, 1, 2
TK_OK, TK_ERR_STALE_INDEX, TK_ERR_BAD_ARG, TK_ERR_CUDA, TK_ERR_NCCL, TK_ERR_OOM, TK_ERR_STATE = range(7)

dbl_p = C.POINTER(C.c_double)
flt_p = C.POINTER(C.c_float)
i32_p = C.POINTER(C.c_int32)
u8_p = C.POINTER(C.c_uint8)
i64_p = C.POINTER(C.c_int64)


class tk_camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_double),
                ("far_plane", C.c_double)]


class tk_pose(C.Structure):
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


class tk_settings(C.Structure):
    _fields_ = [("top_k", C.c_int32), ("tile_size", C.c_int32), ("transmittance_floor", C.c_double),
                ("background", C.c_double * 3), ("cov2d_dilation", C.c_double), ("alpha_clamp", C.c_double)]


class tk_scene_view(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("mean", C.c_void_p), ("log_scale", C.c_void_p),
                ("rotation", C.c_void_p), ("opacity_logit", C.c_void_p), ("color", C.c_void_p),
                ("feature", C.c_void_p), ("generation", C.c_uint64)]


class tk_topk_view(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("k", C.c_int32), ("index", C.c_void_p),
                ("weight", C.c_void_p), ("count", C.c_void_p), ("mem", C.c_int32)]


class tk_geom_out(C.Structure):
    _fields_ = [("mem", C.c_int32), ("color", C.c_void_p), ("depth", C.c_void_p), ("alpha", C.c_void_p),
                ("topk_index", C.c_void_p), ("topk_weight", C.c_void_p), ("topk_count", C.c_void_p),
                ("contributions", C.c_void_p), ("generation", C.c_uint64), ("map_size", C.c_int64)]


class tk_geom_grads(C.Structure):
    _fields_ = [("mem", C.c_int32), ("mean", C.c_void_p), ("log_scale", C.c_void_p), ("rotation", C.c_void_p),
                ("opacity_logit", C.c_void_p), ("color", C.c_void_p), ("pose_twist", C.c_double * 6)]


class tk_device_view(C.Structure):
    _fields_ = [("color", C.c_void_p), ("depth", C.c_void_p), ("alpha", C.c_void_p),
                ("topk_index", C.c_void_p), ("topk_weight", C.c_void_p), ("topk_count", C.c_void_p),
                ("contributions", C.c_void_p), ("feature_out", C.c_void_p), ("feature_grad", C.c_void_p),
                ("grad_feature_in", C.c_void_p), ("mean", C.c_void_p), ("feature", C.c_void_p),
                ("n", C.c_int64), ("d", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("k", C.c_int32)]


class tk_mapper_config(C.Structure):
    _fields_ = [("lambda_geo", C.c_double), ("lambda_feat", C.c_double), ("lambda1", C.c_double),
                ("lambda2", C.c_double), ("color_secondary", C.c_int32), ("feature_update_period", C.c_int32),
                ("l1_deadband", C.c_double), ("lr_mean", C.c_double), ("lr_log_scale", C.c_double),
                ("lr_rotation", C.c_double), ("lr_opacity", C.c_double), ("lr_color", C.c_double),
                ("lr_feature", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("min_log_scale", C.c_double), ("max_log_scale", C.c_double)]


class tk_frame_view(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("d", C.c_int32), ("color", C.c_void_p),
                ("depth", C.c_void_p), ("feature", C.c_void_p), ("mem", C.c_int32)]


class tk_scene_out(C.Structure):
    _fields_ = [("mem", C.c_int32), ("mean", C.c_void_p), ("log_scale", C.c_void_p), ("rotation", C.c_void_p),
                ("opacity_logit", C.c_void_p), ("color", C.c_void_p), ("feature", C.c_void_p),
                ("topk_count", C.c_void_p), ("max_contribution", C.c_void_p)]


class tk_source_view(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("position", C.c_void_p), ("color", C.c_void_p),
                ("feature", C.c_void_p), ("spacing", C.c_void_p), ("distance", C.c_void_p), ("mem", C.c_int32)]


# (name, restype, argtypes) of every symbol include/tk_render.h declares.
RENDER_SYMBOLS = [
    ("tk_default_settings", None, [C.POINTER(tk_settings)]),
    ("tk_last_error", C.c_char_p, []),
    ("tk_abi_version", C.c_int32, []),
    ("tk_create", C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    ("tk_destroy", C.c_int, [C.c_void_p]),
    ("tk_synchronize", C.c_int, [C.c_void_p]),
    ("tk_join", C.c_int, [C.c_void_p]),
    ("tk_get_stream", C.c_void_p, [C.c_void_p]),
    ("tk_host_alloc", C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    ("tk_host_free", C.c_int, [C.c_void_p]),
    ("tk_scene_upload", C.c_int, [C.c_void_p, C.POINTER(tk_scene_view), C.c_int32]),
    ("tk_scene_upload_features", C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int32]),
    ("tk_device_view_get", C.c_int, [C.c_void_p, C.POINTER(tk_device_view)]),
    ("tk_prepare_scene", C.c_int, [C.c_void_p, C.POINTER(tk_pose), C.POINTER(tk_camera), C.POINTER(tk_settings),
                                   i64_p, i64_p, i32_p, i32_p]),
    ("tk_prepared_export", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tk_render_geometric", C.c_int, [C.c_void_p, C.POINTER(tk_pose), C.POINTER(tk_camera),
                                      C.POINTER(tk_settings), C.POINTER(tk_geom_out)]),
    ("tk_render_feature", C.c_int, [C.c_void_p, C.POINTER(tk_topk_view), C.c_void_p, C.c_int32]),
    ("tk_render_feature_full_blend", C.c_int, [C.c_void_p, C.POINTER(tk_pose), C.POINTER(tk_camera),
                                               C.POINTER(tk_settings), C.c_void_p, C.c_int32]),
    ("tk_backward_feature", C.c_int, [C.c_void_p, C.POINTER(tk_topk_view), C.c_void_p, C.c_int32, C.c_void_p,
                                      C.c_int32]),
    ("tk_backward_geometric", C.c_int, [C.c_void_p, C.POINTER(tk_pose), C.POINTER(tk_camera),
                                        C.POINTER(tk_settings), C.c_void_p, C.c_void_p, C.c_int32,
                                        C.POINTER(tk_geom_grads)]),
    ("tk_comm_unique_id", C.c_int, [C.c_void_p]),
    ("tk_comm_init", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    ("tk_allgather_feature", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    ("tk_comm_p2p_setup", C.c_int, [C.c_void_p, C.c_int64]),
    ("tk_optimizer_flush", C.c_int, [C.c_void_p]),
    ("tk_keyframe_load_features", C.c_int, [C.c_void_p, C.c_int32, C.c_char_p]),
    ("tk_keyframe_save_features", C.c_int, [C.c_void_p, C.c_int32, C.c_char_p]),
    ("tk_comm_set_peers", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64]),
    ("tk_render_feature_gathered", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    ("tk_comm_gathered_buffer", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tk_geometry_band", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("tk_allreduce_sum_f64", C.c_int, [C.c_void_p, dbl_p, C.c_int32]),
    ("tk_kernel_launches", C.c_int64, [C.c_void_p]),
    ("tk_invalidate", C.c_int, [C.c_void_p]),
    ("tk_pair_count", C.c_int, [C.c_void_p, i64_p, C.c_int32]),
    ("tk_fp64_rate", C.c_int, [C.c_void_p, dbl_p]),
    ("tk_profile_enable", C.c_int, [C.c_void_p, C.c_int32]),
    ("tk_profile_read", C.c_int, [C.c_void_p, dbl_p, i64_p, C.c_int32]),
    ("tk_default_mapper_config", None, [C.POINTER(tk_mapper_config)]),
    ("tk_keyframe_set", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(tk_pose), C.POINTER(tk_frame_view)]),
    ("tk_optimizer_reset", C.c_int, [C.c_void_p, C.c_int32]),
    ("tk_optimize_step", C.c_int, [C.c_void_p, C.POINTER(tk_mapper_config), C.POINTER(tk_camera),
                                   C.POINTER(tk_settings), C.c_int32, C.c_int64, dbl_p, i32_p]),
    ("tk_loss_values", C.c_int, [C.c_void_p, dbl_p]),
    ("tk_scene_download", C.c_int, [C.c_void_p, C.POINTER(tk_scene_out)]),
    ("tk_scene_info", C.c_int, [C.c_void_p, i64_p, i32_p, C.POINTER(C.c_uint64)]),
    ("tk_insert_gaussians", C.c_int, [C.c_void_p, C.POINTER(tk_source_view), C.c_double, C.POINTER(tk_pose),
                                      i32_p]),
    ("tk_prune_map", C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_int32, C.c_void_p, i64_p]),
    ("tk_prune_draw", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_uint64, C.c_int32, C.c_void_p,
                                i64_p]),
    ("tk_checkpoint_save", C.c_int, [C.c_void_p, C.c_char_p]),
    ("tk_checkpoint_load", C.c_int, [C.c_void_p, C.c_char_p]),
    ("tk_segment_by_query", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_int32]),
]

PHASES = ["prepare", "geom_fwd", "gather", "fbwd_index", "fbwd", "geom_bwd", "chain", "full_blend", "allgather",
          "copy", "loss", "adam"]


_render = None


def _bind(lib, symbols):
    for name, res, args in symbols:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def render_lib():
    """The CUDA library.  Raises if it is not built: there is no fallback path."""
    global _render
    if _render is None:
        if not os.path.exists(RENDER_LIB):
            raise ImportError(f"{RENDER_LIB} missing: build it with `python -m paper_2602_06991_b200.build`")
        _render = _bind(C.CDLL(RENDER_LIB, mode=C.RTLD_GLOBAL), RENDER_SYMBOLS)
    return _render


class TkError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def check(status: int) -> None:
    if status != TK_OK:
        msg = render_lib().tk_last_error()
        raise TkError(status, msg.decode() if msg else f"tk status {status}")
