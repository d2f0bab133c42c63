"""ctypes binding of libktb.so (include/ktb.h). No fallback: importing the
package on a machine without the built library raises immediately."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", os.environ.get("KTB_LIB_NAME", "libktb.so"))

I64 = C.c_int64
VP = C.c_void_p

_lib = None


class KtbLoadError(ImportError):
    pass


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise KtbLoadError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2405_01599_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "ktb_last_error": ([], C.c_char_p),
        "ktb_version": ([], C.c_int),
        "ktb_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "ktb_matrix_create": ([I64, VP, VP, VP, C.c_int, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_matrix_create_i32": ([I64, VP, VP, VP, C.c_int, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_matrix_destroy": ([VP], C.c_int),
        "ktb_matrix_info": ([VP, C.POINTER(I64), C.POINTER(I64), C.POINTER(C.c_int),
                             C.POINTER(I64), C.POINTER(I64)], C.c_int),
        "ktb_matrix_download": ([VP, VP, VP, VP], C.c_int),
        "ktb_matrix_slice": ([VP, I64, I64, C.POINTER(VP)], C.c_int),
        "ktb_mm_probe": ([C.c_char_p, C.POINTER(I64), C.POINTER(I64), C.POINTER(C.c_int)],
                         C.c_int),
        "ktb_mm_read": ([C.c_char_p, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_csr_host_info": ([VP, C.POINTER(I64), C.POINTER(I64), C.POINTER(C.c_int)], C.c_int),
        "ktb_csr_host_copy": ([VP, VP, VP, VP], C.c_int),
        "ktb_csr_host_upload": ([VP, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_csr_host_destroy": ([VP], C.c_int),
        "ktb_mm_write": ([C.c_char_p, I64, VP, VP, VP, C.c_int], C.c_int),
        "ktb_ilu0_create": ([VP, VP, C.POINTER(VP)], C.c_int),
        "ktb_ilu0_info": ([VP] + [C.POINTER(I64)] * 4, C.c_int),
        "ktb_ilu0_download": ([VP, VP, VP], C.c_int),
        "ktb_ilu0_apply": ([VP, VP, VP, C.c_int, VP], C.c_int),
        "ktb_ilu0_destroy": ([VP], C.c_int),
        "ktb_vec_mdot_scratch": ([C.c_int], I64),
        "ktb_vec_mdot": ([I64, C.c_int, VP, I64, VP, VP, VP, VP], C.c_int),
        "ktb_vec_maxpy": ([I64, C.c_int, VP, I64, VP, C.c_double, VP, VP], C.c_int),
        "ktb_vec_axpby": ([I64, C.c_double, VP, C.c_double, VP, VP], C.c_int),
        "ktb_vec_scale": ([I64, C.c_double, C.c_int, VP, VP], C.c_int),
        "ktb_dist_create": ([I64, C.c_int, VP, C.c_int, VP, VP, VP, C.POINTER(VP)], C.c_int),
        "ktb_dist_destroy": ([VP], C.c_int),
        "ktb_dist_info": ([VP] + [C.POINTER(I64)] * 5, C.c_int),
        "ktb_dist_ghosts": ([VP, VP, VP], C.c_int),
        "ktb_dist_set_sends": ([VP, VP, VP], C.c_int),
        "ktb_dist_local_csr": ([VP, VP, VP, VP], C.c_int),
        "ktb_dist_ghost_csr": ([VP, VP, VP, VP, VP], C.c_int),
        "ktb_dist_upload": ([VP, C.c_int], C.c_int),
        "ktb_dist_local_matrix": ([VP, C.POINTER(VP)], C.c_int),
        "ktb_dist_pack": ([VP, VP, VP, VP], C.c_int),
        "ktb_dist_ghost_spmv": ([VP, VP, VP, VP], C.c_int),
        "ktb_comm_id": ([VP], C.c_int),
        "ktb_comm_create": ([VP, C.c_int, C.c_int, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_comm_wrap": ([VP, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_loopback_world_create": ([C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_loopback_world_destroy": ([VP], C.c_int),
        "ktb_comm_create_loopback": ([VP, C.c_int, C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_comm_info": ([VP] + [C.POINTER(C.c_int)] * 5, C.c_int),
        "ktb_comm_destroy": ([VP], C.c_int),
        "ktb_comm_allreduce": ([VP, VP, I64, C.c_int, VP], C.c_int),
        "ktb_comm_allgather": ([VP, VP, VP, C.c_size_t, VP], C.c_int),
        "ktb_comm_sendrecv": ([VP, VP, C.c_size_t, C.c_int, VP, C.c_size_t, C.c_int, VP],
                              C.c_int),
        "ktb_halo_create": ([VP, I64, I64, VP, C.c_int, I64, C.POINTER(VP)], C.c_int),
        "ktb_halo_create_stencil7": ([I64, I64, I64, C.c_double, C.c_double, VP, C.c_int, I64,
                                      C.POINTER(VP)], C.c_int),
        "ktb_halo_create_csr": ([I64, I64, I64, VP, VP, VP, VP, C.c_int, I64, C.POINTER(VP)],
                                C.c_int),
        "ktb_halo_info": ([VP] + [C.POINTER(I64)] * 6 + [C.POINTER(C.c_int)], C.c_int),
        "ktb_halo_parts": ([VP] + [C.POINTER(I64)] * 4, C.c_int),
        "ktb_halo_plan_params": ([VP] + [C.POINTER(I64)] * 2, C.c_int),
        "ktb_halo_spmv": ([VP, VP, VP, VP], C.c_int),
        "ktb_halo_exchange": ([VP, VP, VP], C.c_int),
        "ktb_halo_spmv_host": ([VP, VP, VP, C.c_int], C.c_int),
        "ktb_halo_destroy": ([VP], C.c_int),
        "ktb_halo_set_timing": ([VP, C.c_int], C.c_int),
        "ktb_halo_timing": ([VP, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
        "ktb_dist_connect": ([VP, VP, C.c_int, I64], C.c_int),
        "ktb_dist_set_plan": ([VP, VP], C.c_int),
        "ktb_dist_spmv": ([VP, VP, VP, VP], C.c_int),
        "ktb_dist_exchange": ([VP, VP, VP], C.c_int),
        "ktb_dist_launches": ([VP, C.POINTER(C.c_int)], C.c_int),
        "ktb_dist_sends": ([VP, VP, VP], C.c_int),
        "ktb_gen_stencil7": ([I64, I64, I64, C.c_double, C.c_double, C.c_double, C.c_double,
                              C.c_int, C.POINTER(VP)], C.c_int),
        "ktb_gen_stencil27_upper": ([I64, I64, I64, C.c_double, C.c_double, C.c_int,
                                     C.POINTER(VP)], C.c_int),
        "ktb_gen_stencil7_slab": ([I64, I64, I64, I64, I64, C.c_double, C.c_double, C.c_int,
                                   C.POINTER(VP)], C.c_int),
        "ktb_seeded_vector": ([I64, C.c_uint64, I64, VP, VP], C.c_int),
        "ktb_gen_powerlaw": ([I64, C.c_uint64, I64, C.c_double, I64, C.c_int, C.POINTER(VP)],
                             C.c_int),
        "ktb_gen_powerlaw_host": ([I64, C.c_uint64, I64, C.c_double, I64, VP, VP, VP], C.c_int),
        "ktb_row_partition": ([VP, C.c_int, C.c_int, VP], C.c_int),
        "ktb_row_partition_rowptr": ([VP, I64, C.c_int, C.c_int, C.c_int, VP], C.c_int),
        "ktb_reduction_regions": ([VP, C.c_int, VP, VP, VP], C.c_int),
        "ktb_bss_plan_size": ([VP, I64, C.POINTER(I64), C.POINTER(I64)], C.c_int),
        "ktb_bss_plan_copy": ([VP, I64, VP, VP, VP, VP, VP, VP], C.c_int),
        "ktb_expand_symmetric": ([VP, C.POINTER(VP)], C.c_int),
        "ktb_plan_create": ([VP, C.c_int, I64, C.c_int, VP, C.POINTER(VP)], C.c_int),
        "ktb_plan_destroy": ([VP], C.c_int),
        "ktb_plan_info": ([VP, C.POINTER(C.c_int), C.POINTER(I64), C.POINTER(I64),
                           C.POINTER(C.c_int), C.POINTER(I64)], C.c_int),
        "ktb_plan_set_stream": ([VP, VP], C.c_int),
        "ktb_plan_s3_info": ([VP] + [C.POINTER(I64)] * 4 + [C.POINTER(C.c_int),
                                                            C.POINTER(I64)], C.c_int),
        "ktb_spmv": ([VP, VP, VP, C.c_int], C.c_int),
        "ktb_spmv_host_pipelined": ([VP, I64, VP, I64, VP, I64], C.c_int),
        "ktb_spmv_rows": ([VP, I64, I64, VP, VP], C.c_int),
        "ktb_select": ([VP, VP, VP, C.POINTER(VP), VP, C.c_int, C.POINTER(C.c_int),
                        C.POINTER(C.c_int)], C.c_int),
        "ktb_host_alloc": ([C.c_size_t, C.POINTER(VP)], C.c_int),
        "ktb_host_free": ([VP], C.c_int),
        "ktb_device_alloc": ([C.c_int, C.c_size_t, C.POINTER(VP)], C.c_int),
        "ktb_device_free": ([VP], C.c_int),
        "ktb_memcpy": ([VP, VP, C.c_size_t, C.c_int, VP], C.c_int),
        "ktb_stream_sync": ([VP], C.c_int),
        "ktb_time_spmv": ([VP, VP, VP, C.c_int, C.c_size_t, C.POINTER(C.c_double),
                           C.POINTER(C.c_double)], C.c_int),
        "ktb_gmres": ([VP, VP, VP, I64, C.c_double, I64, VP, VP], C.c_int),
        "ktb_gmres_ilu0": ([VP, VP, VP, VP, I64, C.c_double, I64, VP, VP], C.c_int),
    }
    for name, spec in sig.items():
        if spec is None:
            continue
        f = getattr(L, name)
        f.argtypes, f.restype = spec
    _lib = L
    return L


# exported symbols declared in include/ktb.h (checked by tests without a GPU)
def declared_symbols() -> list[str]:
    import re

    hdr = os.path.join(os.path.dirname(HERE), "include", "ktb.h")
    txt = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*|void)\s+(ktb_\w+)\(", txt,
                                 re.M)))
