"""ctypes mirror of include/gfb200.h (plan records and kernel argument blocks).

`tests/test_abi.py` compiles a probe against the header and checks every
size and offset here, so the two cannot drift apart silently.
"""

from __future__ import annotations

import ctypes as C

GFB_OK = 0

K_EW_F32, K_EW_F64, K_EW_I64, K_EW_U8 = 1, 2, 3, 4
K_EWS_F32, K_EWS_F64 = 5, 6
K_EW1_F32, K_EW1_F64 = 7, 8
K_DOT_F32, K_DOT_F64, K_DOT_TC32, K_SPLIT_TF32, K_DOT_TC32W = 10, 11, 12, 13, 14
K_DOT_SM_F32, K_DOT_SM_F64 = 15, 16
K_DOT_TC32P = 19
K_DOT_F16P, K_SPLIT_F16 = 34, 35
K_CHMAX, K_CHSPLIT, K_FSPLIT, K_CONV_TCXH64, K_CONV_TCXH128 = 36, 37, 38, 39, 40
K_CONV_TCGWH64, K_CONV_TCGWH128 = 41, 42
K_MEMSET = 43
K_CONV_STEMH = 44
K_CONV_STEMH_C3R7 = 45
K_CONV_STEMWH_C3R7 = 46
K_CONV_TCG64, K_CONV_TCG128 = 17, 18
K_CONV_TCX64, K_CONV_TCX128 = 22, 23
K_CONV_TCGG64, K_CONV_TCGG128 = 24, 25
K_CONV_TCGW64, K_CONV_TCGW128 = 28, 29
K_CONV_STEM64 = 32
K_DOT_TH_F32, K_DOT_TH_F64 = 26, 27
K_CONV_F32, K_CONV_F64 = 20, 21
K_ALLREDUCE = 30
K_ROWJIT = 33
ROW_MAX_REFS = 30

SLOT_ARENA, SLOT_CONST, SLOT_IO = 0, 1, 2
MAX_LEAVES, MAX_DIGITS, MAX_INSTR = 16, 6, 128
PLAN_CUDA_GRAPH = 1


def ref(slot: int, offset: int) -> int:
    assert 0 <= offset < (1 << 56)
    return (slot << 56) | offset


class Digit(C.Structure):
    _fields_ = [
        ("div_mul", C.c_uint64), ("mod_mul", C.c_uint64),
        ("div_sh", C.c_uint32), ("mod_sh", C.c_uint32), ("mod", C.c_uint32),
        ("stride", C.c_int32), ("src", C.c_int32), ("pad", C.c_int32),
    ]


class Leaf(C.Structure):
    _fields_ = [
        ("ref", C.c_uint64), ("splat", C.c_uint64),
        ("mode", C.c_int32), ("ndig", C.c_int32), ("vec", C.c_int32), ("rlin", C.c_int32),
        ("dig", Digit * MAX_DIGITS),
        ("dv", C.c_int32 * 8),
        ("same", C.c_int32), ("pad", C.c_int32),
    ]


class EwArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p),
        ("n_o", C.c_uint32), ("n_r", C.c_uint32), ("ninstr", C.c_uint32), ("nleaves", C.c_uint32),
        ("mode", C.c_int32), ("red_kind", C.c_int32), ("vec_axis", C.c_int32), ("split", C.c_int32),
        ("npre", C.c_int32), ("depth", C.c_int32), ("wpr", C.c_int32),
        ("ty_ext", C.c_int32), ("ty_div", C.c_int32), ("pad", C.c_int32),
        ("prog", C.c_uint32 * MAX_INSTR),
        ("leaves", Leaf * MAX_LEAVES),
        ("red_out", Leaf),
    ]


class DotArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p),
        ("a", C.c_uint64), ("b", C.c_uint64), ("c", C.c_uint64),
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
        ("a_sm", C.c_int64), ("a_sk", C.c_int64), ("b_sk", C.c_int64), ("b_sn", C.c_int64),
        ("c_sm", C.c_int64), ("c_sn", C.c_int64),
    ]


class SplitArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("src", C.c_uint64), ("hi", C.c_uint64), ("lo", C.c_uint64),
        ("rows", C.c_int64), ("k", C.c_int64), ("kp", C.c_int64), ("s_r", C.c_int64), ("s_k", C.c_int64),
        ("mode", C.c_int32), ("pad", C.c_int32),
        ("geo", C.c_int64 * 16), ("st", C.c_int64 * 4),
    ]


class Split16Args(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("src", C.c_uint64), ("hi", C.c_uint64), ("lo", C.c_uint64), ("sc", C.c_uint64),
        ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
    ]


class ChsplitArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("src", C.c_uint64), ("partial", C.c_uint64), ("sc", C.c_uint64), ("hi", C.c_uint64),
        ("lo", C.c_uint64), ("P", C.c_int64), ("C", C.c_int64), ("nblocks", C.c_int32), ("mode", C.c_int32),
    ]


class FsplitArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("w", C.c_uint64), ("sc", C.c_uint64), ("hi", C.c_uint64), ("lo", C.c_uint64),
        ("inv", C.c_uint64), ("rows", C.c_int64), ("K", C.c_int64), ("s_r", C.c_int64),
        ("e0", C.c_int64), ("e1", C.c_int64), ("e2", C.c_int64), ("t0", C.c_int64), ("t1", C.c_int64), ("t2", C.c_int64),
    ]


class TcxhArgs(C.Structure):
    # 64-byte aligned in C: tmap sits at offset 256, size 768.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a_hi", C.c_uint64), ("a_lo", C.c_uint64), ("b_hi", C.c_uint64),
        ("b_lo", C.c_uint64), ("b_inv", C.c_uint64),
        ("N", C.c_int64), ("K", C.c_int64),
        ("o_n", C.c_int64), ("o_y", C.c_int64), ("o_x", C.c_int64), ("c_sn", C.c_int64),
        ("a_dims", C.c_int64 * 4), ("a_strides", C.c_int64 * 4),
        ("No", C.c_int32), ("Yo", C.c_int32), ("Xo", C.c_int32), ("BX", C.c_int32), ("BY", C.c_int32),
        ("BNI", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
        ("sx", C.c_int32), ("sy", C.c_int32), ("ox", C.c_int32), ("oy", C.c_int32), ("S", C.c_int32),
        ("CB", C.c_int32), ("ksign", C.c_int32), ("pad0", C.c_int32),
        ("pad", C.c_int64 * 3),
        ("tmap", (C.c_uint64 * 16) * 4),
    ]


class TcgwhArgs(C.Structure):
    # 64-byte aligned in C: tmap sits at offset 384, size 896.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a_hi", C.c_uint64), ("a_lo", C.c_uint64), ("b_hi", C.c_uint64),
        ("b_lo", C.c_uint64), ("a_sc", C.c_uint64), ("b_sc", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("C", C.c_int64), ("S", C.c_int64), ("pt", C.c_int64), ("pl", C.c_int64),
        ("c_s_hi", C.c_int64), ("c_s_lo", C.c_int64), ("c_sn", C.c_int64),
        ("k_splits", C.c_int64), ("boxes_per_split", C.c_int64), ("split_stride", C.c_int64),
        ("a_dims", C.c_int64 * 4), ("a_strides", C.c_int64 * 4), ("b_dims", C.c_int64 * 4), ("b_strides", C.c_int64 * 4),
        ("No", C.c_int32), ("Yo", C.c_int32), ("Xo", C.c_int32), ("BX", C.c_int32), ("BY", C.c_int32),
        ("BNI", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
        ("pad", C.c_int64 * 8),
        ("tmap", (C.c_uint64 * 16) * 4),
    ]


class TcArgs(C.Structure):
    # 64-byte aligned in C (GFB_ALIGN64): tmap sits at offset 320, size 832.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("c_sm", C.c_int64), ("c_sn", C.c_int64),
        ("a_hi", C.c_uint64), ("a_lo", C.c_uint64), ("b_hi", C.c_uint64), ("b_lo", C.c_uint64),
        ("kp_a", C.c_int64), ("kp_b", C.c_int64),
        ("c_rdiv", C.c_int64), ("c_s_hi", C.c_int64), ("c_s_lo", C.c_int64),
        ("k_splits", C.c_int64), ("k_per_split", C.c_int64), ("split_stride", C.c_int64),
        ("a_ld_mn", C.c_int64), ("b_ld_mn", C.c_int64), ("group_m", C.c_int64),
        ("epi_kind", C.c_int64), ("e_bias", C.c_uint64), ("e_aux1", C.c_uint64), ("e_aux2", C.c_uint64),
        ("e_out2", C.c_uint64), ("e_lo", C.c_uint64), ("epi_flags", C.c_int64),
        ("a_sc", C.c_uint64), ("b_sc", C.c_uint64),
        ("a_sc_r", C.c_int64), ("a_sc_k", C.c_int64), ("b_sc_r", C.c_int64), ("b_sc_k", C.c_int64),
        ("e_hi", C.c_uint64), ("e_sc", C.c_uint64), ("e_mask", C.c_uint64), ("e_csum", C.c_uint64),
        ("pad", C.c_int64 * 1),
        ("tmap", (C.c_uint64 * 16) * 4),
    ]


class TcgArgs(C.Structure):
    # 64-byte aligned in C: tmap sits at offset 192, size 448.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("c_sm", C.c_int64), ("c_sn", C.c_int64), ("c_rdiv", C.c_int64), ("c_s_hi", C.c_int64), ("c_s_lo", C.c_int64),
        ("a", C.c_uint64), ("b_hi", C.c_uint64), ("b_lo", C.c_uint64),
        ("xs0", C.c_int64), ("xs2", C.c_int64), ("xs3", C.c_int64),
        ("Y", C.c_int32), ("X", C.c_int32), ("sy", C.c_int32), ("sx", C.c_int32), ("oy", C.c_int32), ("ox", C.c_int32),
        ("H", C.c_int32), ("W", C.c_int32), ("S", C.c_int32), ("CB", C.c_int32), ("ksign", C.c_int32), ("C", C.c_int32),
        ("pad", C.c_int64 * 2),
        ("tmap", (C.c_uint64 * 16) * 2),
    ]


class StemhArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a", C.c_uint64), ("w", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("c_s_hi", C.c_int64), ("c_sm", C.c_int64), ("c_s_lo", C.c_int64), ("c_sn", C.c_int64),
        ("xs0", C.c_int64), ("xs1", C.c_int64), ("xs2", C.c_int64), ("xs3", C.c_int64),
        ("ws0", C.c_int64), ("ws1", C.c_int64), ("ws2", C.c_int64), ("ws3", C.c_int64),
        ("Y", C.c_int32), ("X", C.c_int32), ("oy", C.c_int32), ("ox", C.c_int32),
        ("H", C.c_int32), ("W", C.c_int32), ("S", C.c_int32), ("C", C.c_int32),
        ("c2", C.c_uint64), ("flags", C.c_int64),
    ]


class TcxArgs(C.Structure):
    # 64-byte aligned in C: tmap sits at offset 256, size 640.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a", C.c_uint64), ("b_hi", C.c_uint64), ("b_lo", C.c_uint64),
        ("N", C.c_int64), ("K", C.c_int64),
        ("o_n", C.c_int64), ("o_y", C.c_int64), ("o_x", C.c_int64), ("c_sn", C.c_int64),
        ("a_dims", C.c_int64 * 4), ("a_strides", C.c_int64 * 4),
        ("No", C.c_int32), ("Yo", C.c_int32), ("Xo", C.c_int32), ("BX", C.c_int32), ("BY", C.c_int32),
        ("BNI", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
        ("sx", C.c_int32), ("sy", C.c_int32), ("ox", C.c_int32), ("oy", C.c_int32), ("S", C.c_int32),
        ("CB", C.c_int32), ("ksign", C.c_int32), ("pad0", C.c_int32),
        ("pad", C.c_int64 * 5),
        ("tmap", (C.c_uint64 * 16) * 3),
    ]


class TcggArgs(C.Structure):
    # 64-byte aligned in C: tmap sits at offset 256, size 512.
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a", C.c_uint64), ("b_hi", C.c_uint64), ("b_lo", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("Kp", C.c_int64), ("kp_b", C.c_int64),
        ("c_sm", C.c_int64), ("c_sn", C.c_int64), ("c_rdiv", C.c_int64), ("c_s_hi", C.c_int64), ("c_s_lo", C.c_int64),
        ("ro0", C.c_int64), ("ro1", C.c_int64), ("ro2", C.c_int64),
        ("ko0", C.c_int64), ("ko1", C.c_int64), ("ko2", C.c_int64), ("kbase", C.c_int64),
        ("k_splits", C.c_int64), ("split_stride", C.c_int64),
        ("E1", C.c_int32), ("E2", C.c_int32), ("hm", C.c_int32), ("wm", C.c_int32), ("h0", C.c_int32),
        ("w0", C.c_int32), ("H", C.c_int32), ("W", C.c_int32),
        ("Ke1", C.c_int32), ("Ke2", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("dh0", C.c_int32),
        ("dw0", C.c_int32), ("kb_per_split", C.c_int32), ("pad0", C.c_int32),
        ("tmap", (C.c_uint64 * 16) * 2),
    ]


class TcgwArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("c", C.c_uint64), ("a", C.c_uint64), ("b", C.c_uint64),
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("c_sm", C.c_int64), ("c_sn", C.c_int64), ("c_rdiv", C.c_int64), ("c_s_hi", C.c_int64), ("c_s_lo", C.c_int64),
        ("ro0", C.c_int64), ("ro1", C.c_int64), ("ro2", C.c_int64),
        ("ko0", C.c_int64), ("ko1", C.c_int64), ("ko2", C.c_int64), ("kbase", C.c_int64),
        ("yo0", C.c_int64), ("yo1", C.c_int64), ("yo2", C.c_int64),
        ("k_splits", C.c_int64), ("split_stride", C.c_int64),
        ("E1", C.c_int32), ("E2", C.c_int32), ("h0", C.c_int32), ("w0", C.c_int32), ("H", C.c_int32), ("W", C.c_int32),
        ("Ke1", C.c_int32), ("Ke2", C.c_int32), ("kb_per_split", C.c_int32), ("pad", C.c_int32),
    ]


class ConvArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p),
        ("x", C.c_uint64), ("y", C.c_uint64), ("out", C.c_uint64),
        ("op", C.c_int32), ("pad0", C.c_int32),
        ("N", C.c_int64), ("C", C.c_int64), ("H", C.c_int64), ("W", C.c_int64),
        ("K", C.c_int64), ("R", C.c_int64), ("S", C.c_int64), ("Ho", C.c_int64), ("Wo", C.c_int64),
        ("sh", C.c_int64), ("sw", C.c_int64), ("pt", C.c_int64), ("pl", C.c_int64),
        ("xs", C.c_int64 * 4), ("ys", C.c_int64 * 4), ("os", C.c_int64 * 4),
    ]


class MemsetArgs(C.Structure):
    _fields_ = [("tab", C.c_void_p), ("buf", C.c_uint64), ("bytes", C.c_uint64)]


class AllReduceArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("buf", C.c_uint64), ("count", C.c_uint64),
        ("dtype", C.c_int32), ("op", C.c_int32),
    ]


class RowArgs(C.Structure):
    _fields_ = [
        ("tab", C.c_void_p), ("n_refs", C.c_uint32), ("pad", C.c_uint32), ("refs", C.c_uint64 * 30),
    ]


class Launch(C.Structure):
    _fields_ = [
        ("kind", C.c_uint32), ("grid", C.c_uint32 * 3), ("block", C.c_uint32 * 3),
        ("smem", C.c_uint32), ("arg_offset", C.c_uint32), ("arg_size", C.c_uint32),
    ]


class Plan(C.Structure):
    _fields_ = [
        ("arena_bytes", C.c_uint64), ("const_bytes", C.c_uint64), ("const_data", C.c_void_p),
        ("n_inputs", C.c_uint32), ("n_outputs", C.c_uint32), ("n_launches", C.c_uint32),
        ("flags", C.c_uint32),
        ("launches", C.POINTER(Launch)),
        ("args_bytes", C.c_uint64), ("args", C.c_void_p),
        ("comm", C.c_void_p),
    ]


STRUCTS = {
    "gfb_digit": Digit, "gfb_leaf": Leaf, "gfb_ew_args": EwArgs, "gfb_dot_args": DotArgs,
    "gfb_conv_args": ConvArgs, "gfb_split_args": SplitArgs, "gfb_split16_args": Split16Args, "gfb_chsplit_args": ChsplitArgs, "gfb_fsplit_args": FsplitArgs, "gfb_tcxh_args": TcxhArgs, "gfb_tcgwh_args": TcgwhArgs, "gfb_tc_args": TcArgs, "gfb_tcg_args": TcgArgs, "gfb_stemh_args": StemhArgs, "gfb_tcx_args": TcxArgs, "gfb_tcgg_args": TcggArgs, "gfb_tcgw_args": TcgwArgs, "gfb_allreduce_args": AllReduceArgs, "gfb_memset_args": MemsetArgs, "gfb_row_args": RowArgs, "gfb_launch": Launch, "gfb_plan": Plan,
}
