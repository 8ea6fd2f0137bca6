"""ctypes binding of the product library ``lib/libhlf_b200.so`` (C-ABI in
include/hlf_b200.h).  There is no fallback: if the shared library is missing
the import fails loudly."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HLF_B200_LIB_OVERRIDE") or os.path.join(HERE, "lib", "libhlf_b200.so")

HLF_OK = 0
HLF_CONFIG_ERROR = 1
HLF_INSTABILITY = 2
HLF_INVALID_ARGUMENT = 3
HLF_CUDA_ERROR = 4
HLF_NCCL_ERROR = 5

# every exported symbol declared in include/hlf_b200.h
EXPORTS = [
    "hlf_abi_version", "hlf_build_interp_operator", "hlf_create", "hlf_destroy", "hlf_last_error",
    "hlf_num_nodes", "hlf_num_coeffs", "hlf_set_field", "hlf_get_field", "hlf_set_coeff", "hlf_set_coeff_separable",
    "hlf_set_forcing", "hlf_clear_forcing", "hlf_set_graph_steps", "hlf_l2_error_separable", "hlf_energy_1d",
    "hlf_set_times", "hlf_get_times", "hlf_set_dt", "hlf_advance_p", "hlf_advance_v", "hlf_step",
    "hlf_advance_n", "hlf_plan_steps", "hlf_advance_to", "hlf_advance_p_indexed", "hlf_advance_v_indexed", "hlf_advance_layers", "hlf_commit_half",
    "hlf_poll_finite", "hlf_clear_finite", "hlf_synchronize", "hlf_field_device",
    "hlf_fill_separable", "hlf_error_separable", "hlf_zero_field", "hlf_halo_send_ptr", "hlf_halo_recv_ptr",
    "hlf_launch_count", "hlf_kernel_variant", "hlf_set_kernel_variant", "hlf_enable_path_counters",
    "hlf_read_path_counters", "hlf_time_launches", "hlf_slabs_create", "hlf_slabs_destroy",
    "hlf_slabs_last_error", "hlf_slabs_count", "hlf_slabs_transport", "hlf_slabs_solver", "hlf_slabs_set_times",
    "hlf_slabs_advance_n", "hlf_slabs_synchronize", "hlf_get_stream",
]


class HlfDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("m", C.c_int),
        ("K", C.c_int * 3),
        ("x_min", C.c_double * 3),
        ("h", C.c_double),
        ("boundary", C.c_int * 3),
        ("ap", C.c_double),
        ("av", C.c_double),
        ("variable_ap", C.c_int),
        ("M", C.POINTER(C.c_double)),
        ("device", C.c_int),
        ("stream", C.c_void_p),
        ("z_slab", C.c_int),
        ("scheme", C.c_int),
    ]


_dp = C.POINTER(C.c_double)
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension (python -c 'import __graft_entry__ as g; g.build()')"
        )
    L = C.CDLL(LIB_PATH)
    S = C.c_void_p
    st = C.c_int
    sig = {
        "hlf_abi_version": ([], C.c_int),
        "hlf_build_interp_operator": ([C.c_int, _dp, _dp], st),
        "hlf_create": ([C.POINTER(HlfDesc), C.POINTER(C.c_void_p)], st),
        "hlf_destroy": ([S], None),
        "hlf_last_error": ([S], C.c_char_p),
        "hlf_num_nodes": ([S, C.c_int], C.c_int64),
        "hlf_num_coeffs": ([S], C.c_int),
        "hlf_set_field": ([S, C.c_int, C.c_void_p], st),
        "hlf_get_field": ([S, C.c_int, C.c_void_p], st),
        "hlf_set_coeff": ([S, C.c_int, C.c_void_p], st),
        "hlf_set_coeff_separable": ([S, C.c_double, C.c_double, _dp, _dp], st),
        "hlf_set_forcing": ([S, C.c_int, C.c_void_p], st),
        "hlf_set_graph_steps": ([S, C.c_int], st),
        "hlf_clear_forcing": ([S], st),
        "hlf_set_times": ([S, C.c_double, C.c_double, C.c_double], st),
        "hlf_get_times": ([S, _dp, _dp, _dp], st),
        "hlf_set_dt": ([S, C.c_double], st),
        "hlf_advance_p": ([S], st),
        "hlf_advance_v": ([S], st),
        "hlf_step": ([S, C.c_int], st),
        "hlf_advance_n": ([S, C.c_int, C.c_int], st),
        "hlf_plan_steps": ([C.c_double, C.c_double, C.POINTER(C.c_int), _dp], st),
        "hlf_advance_to": ([S, C.c_double, C.c_int, C.POINTER(C.c_int)], st),
        "hlf_advance_p_indexed": ([S, C.c_int], st),
        "hlf_advance_v_indexed": ([S, C.c_int], st),
        "hlf_advance_layers": ([S, C.c_int, C.c_int, C.c_int, C.c_int], st),
        "hlf_commit_half": ([S, C.c_int], st),
        "hlf_poll_finite": ([S, C.POINTER(C.c_int)], st),
        "hlf_clear_finite": ([S], st),
        "hlf_synchronize": ([S], st),
        "hlf_field_device": ([S, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                              C.POINTER(C.c_int)], st),
        "hlf_fill_separable": ([S, C.c_int, C.c_double, _dp, _dp], st),
        "hlf_zero_field": ([S, C.c_int], st),
        "hlf_error_separable": ([S, C.c_int, C.c_double, _dp, _dp, _dp, _dp], st),
        "hlf_l2_error_separable": ([S, C.c_int, C.c_double, _dp, _dp, _dp], st),
        "hlf_energy_1d": ([S, C.c_int, C.c_double, _dp], st),
        "hlf_halo_send_ptr": ([S, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)], st),
        "hlf_halo_recv_ptr": ([S, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)], st),
        "hlf_launch_count": ([S], C.c_int64),
        "hlf_kernel_variant": ([S], C.c_int),
        "hlf_set_kernel_variant": ([S, C.c_int], st),
        "hlf_enable_path_counters": ([S, C.c_int], st),
        "hlf_read_path_counters": ([S, C.POINTER(C.c_int64)], st),
        "hlf_time_launches": ([S, C.c_int, C.c_int, _dp, C.POINTER(C.c_int)], st),
        "hlf_slabs_create": ([C.POINTER(HlfDesc), C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)], st),
        "hlf_slabs_destroy": ([S], None),
        "hlf_slabs_last_error": ([S], C.c_char_p),
        "hlf_slabs_count": ([S], C.c_int),
        "hlf_slabs_transport": ([S], C.c_int),
        "hlf_slabs_solver": ([S, C.c_int], C.c_void_p),
        "hlf_slabs_set_times": ([S, C.c_double, C.c_double, C.c_double], st),
        "hlf_slabs_advance_n": ([S, C.c_int, C.c_int], st),
        "hlf_slabs_synchronize": ([S], st),
        "hlf_get_stream": ([S], C.c_void_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L
