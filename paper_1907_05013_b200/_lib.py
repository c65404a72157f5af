"""ctypes loader for libpooch.so (the C ABI in include/pooch.h).

Argument marshalling only: every step of the training path runs in the CUDA
kernels and C++ runtime behind this library. There is no fallback: if the
shared library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POOCH_LIB") or os.path.join(_HERE, "libpooch.so")


class PoochError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"pooch status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1907_05013_b200.build` "
                          "(or __graft_entry__.build())")
    return C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)


lib = _load()

c_i32, c_i64, c_u64, c_f32, c_f64, c_sz, c_vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double, C.c_size_t, C.c_void_p
P = C.POINTER


class ConvDesc(C.Structure):
    _fields_ = [(n, c_i32) for n in ("N", "H", "W", "C", "K", "R", "S", "stride", "pad", "precision", "D", "C1",
                                     "groups", "stride_d")]


class DivInfo(C.Structure):
    _fields_ = [("chunks", c_i32), ("rows_per_chunk", c_i32), ("ms", c_f64), ("h2d_bytes", c_u64),
                ("d2h_bytes", c_u64)]


class LayerDesc(C.Structure):
    _fields_ = [("kind", c_i32), ("in0", c_i32), ("in1", c_i32), ("cin", c_i32), ("cout", c_i32),
                ("hout", c_i32), ("wout", c_i32), ("k", c_i32), ("stride", c_i32), ("pad", c_i32),
                ("name", C.c_char * 48), ("dout", c_i32), ("groups", c_i32), ("stride_d", c_i32)]


class IODesc(C.Structure):
    _fields_ = [("batch", c_i32), ("in_c", c_i32), ("in_h", c_i32), ("in_w", c_i32), ("classes", c_i32),
                ("in_d", c_i32)]


class ProfileT(C.Structure):
    _fields_ = [("n", c_i32), ("fwd_ns", P(c_i64)), ("bwd_ns", P(c_i64)), ("rec_ns", P(c_i64)),
                ("d2h_ns", P(c_i64)), ("h2d_ns", P(c_i64)), ("bytes", P(c_u64)), ("tail_ns", c_i64),
                ("resident_bytes", c_u64), ("d2h_gbs", c_f64), ("h2d_gbs", c_f64), ("duplex_gbs", c_f64),
                ("mode", c_i32), ("d2h_issue_ns", P(c_i64)), ("h2d_issue_ns", P(c_i64)), ("step_ns", c_i64)]


class Problem(C.Structure):
    _fields_ = [("n", c_i32), ("fwd_ns", P(c_i64)), ("bwd_ns", P(c_i64)), ("rec_ns", P(c_i64)),
                ("d2h_ns", P(c_i64)), ("h2d_ns", P(c_i64)), ("bytes", P(c_u64)),
                ("in_ptr", P(c_i32)), ("in_idx", P(c_i32)), ("need_ptr", P(c_i32)), ("need_idx", P(c_i32)),
                ("resident_bytes", c_u64), ("budget_bytes", c_u64), ("tail_ns", c_i64), ("is_conv", P(C.c_uint8)),
                ("host_budget_bytes", c_u64), ("duplex_d2h_permille", C.c_int32),
                ("duplex_h2d_permille", C.c_int32)]


class SimResult(C.Structure):
    _fields_ = [("oom", c_i32), ("makespan_ns", c_i64), ("peak_bytes", c_u64), ("n_events", c_i32),
                ("in_lo", P(C.c_uint8)), ("in_li", P(C.c_uint8)), ("stall_ns", P(c_i64)),
                ("events_cap", c_i32), ("ev_lane", P(c_i32)), ("ev_kind", P(c_i32)), ("ev_id", P(c_i32)),
                ("ev_start", P(c_i64)), ("ev_end", P(c_i64))]


class SearchCfg(C.Structure):
    _fields_ = [("li_cap", c_i32), ("threads", c_i32), ("sched", c_i32)]


class PlanReport(C.Structure):
    _fields_ = [("makespan_ns", c_i64), ("peak_bytes", c_u64), ("arena_bytes", c_u64), ("n_keep", c_i32),
                ("n_swap", c_i32), ("n_recompute", c_i32), ("host_bytes", c_u64), ("n_sims", c_i64),
                ("wall_ms", c_f64), ("lo_size", c_i32), ("li_size", c_i32), ("feasible", c_i32)]


# name -> (restype, argtypes); every symbol declared in include/pooch.h
SIGNATURES = {
    "pooch_last_error": (C.c_char_p, [c_vp]),
    "pooch_build_net": (c_i32, [c_i32, c_i32, c_i32, c_i32, P(LayerDesc), P(c_i32)]),
    "pooch_create": (c_i32, [P(LayerDesc), c_i32, P(IODesc), c_i32, P(c_vp)]),
    "pooch_destroy": (None, [c_vp]),
    "pooch_set_budget": (c_i32, [c_vp, c_vp, c_sz, c_vp, c_sz]),
    "pooch_resident_bytes": (c_i32, [c_vp, P(c_u64)]),
    "pooch_set_streams": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_set_comm": (c_i32, [c_vp, c_vp, c_i32, c_i32]),
    "pooch_peer_open": (c_i32, [c_vp, c_i32, c_i32, c_vp, P(C.c_uint64)]),
    "pooch_set_peers": (c_i32, [c_vp, c_vp]),
    "pooch_input_slot": (c_i32, [c_vp, P(c_vp), P(c_vp)]),
    "pooch_num_params": (c_i32, [c_vp, P(c_i32)]),
    "pooch_param_info": (c_i32, [c_vp, c_i32, C.c_char_p, P(c_i64)]),
    "pooch_get_param": (c_i32, [c_vp, c_i32, c_i32, P(c_f32), c_i64]),
    "pooch_set_param": (c_i32, [c_vp, c_i32, c_i32, P(c_f32), c_i64]),
    "pooch_profile": (c_i32, [c_vp, c_i32, P(ProfileT)]),
    "pooch_set_profile": (c_i32, [c_vp, P(c_i64), P(c_i64), P(c_i64), P(c_i64), P(c_i64), c_i64]),
    "pooch_set_link": (c_i32, [c_vp, c_f64, c_f64, c_f64]),
    "pooch_simulate": (c_i32, [P(Problem), P(C.c_uint8), c_i32, P(SimResult)]),
    "pooch_plan_problem": (c_i32, [P(Problem), c_i32, P(SearchCfg), P(C.c_uint8), P(C.c_uint8), P(PlanReport)]),
    "pooch_pack_problem": (c_i32, [P(Problem), P(C.c_uint8), c_i32, c_u64, P(c_u64), P(c_i32), P(c_i32), P(c_u64),
                                   P(c_u64)]),
    "pooch_plan": (c_i32, [c_vp, c_i32, P(SearchCfg), P(C.c_uint8), P(C.c_uint8), P(PlanReport)]),
    "pooch_train_step": (c_i32, [c_vp, c_f32, P(c_f32)]),
    "pooch_set_timing": (c_i32, [c_vp, c_i32]),
    "pooch_last_timing": (c_i32, [c_vp, P(c_i64), P(c_i64), P(c_i64), P(c_i64), P(c_i64), P(c_i64)]),
    "pooch_family_stats": (c_i32, [c_vp, c_i32, P(c_f64), P(c_i64), P(c_f64), P(c_f64)]),
    "pooch_loss_slot": (c_i32, [c_vp, P(c_vp)]),
    "pooch_set_precision": (c_i32, [c_vp, c_i32]),
    "pooch_read_buffer": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_sz]),
    "pooch_kernel_launches": (c_i32, [c_vp, P(c_i64)]),
    "pooch_op_conv_fwd": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_op_conv_dgrad": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_i32, c_vp]),
    "pooch_op_conv_wgrad": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pooch_op_conv_wgrad_ws_bytes": (c_sz, [P(ConvDesc)]),
    "pooch_op_conv_stat_tiles": (c_i64, [P(ConvDesc)]),
    "pooch_timing_segments": (c_i32, [c_vp, P(c_i32), c_vp, c_vp, c_vp, c_vp]),
    "pooch_allreduce_buckets": (c_i32, [c_vp, P(c_i32), c_vp, c_vp, c_vp]),
    "pooch_op_conv_fwd2": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_op_conv_dgrad2": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "pooch_op_conv_wgrad2": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pooch_refine_problem": (c_i32, [c_vp, c_vp, c_i32, c_u64, c_vp, P(c_i64), P(c_i32)]),
    "pooch_op_conv_fwd_bnrelu": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_op_conv_wgrad_bnrelu": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pooch_op_maxpool3d_fwd_k": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pooch_op_maxpool3d_bwd_k": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32,
                                         c_i32, c_vp]),
    "pooch_div_conv3d_fwd": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "pooch_div_bn_relu_fwd": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_sz, c_vp, c_vp]),
    "pooch_div_bn_relu_bwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_sz,
                                      c_vp, c_vp]),
    "pooch_div_conv3d_dgrad": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "pooch_div_conv3d_wgrad": (c_i32, [P(ConvDesc), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp]),
    "pooch_op_maxpool2d_fwd": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pooch_op_maxpool2d_bwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pooch_op_bn_ws_bytes": (c_sz, [c_i32]),
    "pooch_op_bn_finalize": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_op_bn_relu_fwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pooch_op_bn_relu_bwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp,
                                     c_vp]),
    "pooch_op_maxpool3d_fwd": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pooch_op_maxpool3d_bwd": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pooch_set_profile_mode": (c_i32, [c_vp, c_i32]),
    "pooch_set_rng": (c_i32, [c_vp, C.c_uint32, C.c_uint32]),
    "pooch_last_trace": (c_i32, [c_vp, P(c_i32), c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_plan_trace": (c_i32, [c_vp, P(c_i32), c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pooch_step_graph": (c_i32, [c_vp, P(c_i32)]),
    "pooch_op_lrn_fwd": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pooch_op_lrn_bwd": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pooch_comm_info": (c_i32, [c_vp, P(c_i32), P(c_i32), P(c_i32)]),
    "pooch_op_gemm_test": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    if hasattr(lib, _name):
        _f = getattr(lib, _name)
        _f.restype = _res
        _f.argtypes = _args


def check(status, ctx=None):
    if status != 0:
        msg = lib.pooch_last_error(ctx)
        raise PoochError(status, msg.decode() if msg else "")
