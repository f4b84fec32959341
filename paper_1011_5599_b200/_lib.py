"""ctypes binding of libhanf.so (include/hanf.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_1011_5599_b200/csrc``.  There is no fallback: if the library
is missing, importing the engine raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_int32, c_uint32,
                    c_uint64, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
# HANF_LIB=checked loads the bounds-checked build (csrc/Makefile `checked`)
LIB_PATH = os.path.join(_HERE, "libhanf_checked.so" if os.environ.get("HANF_LIB") == "checked"
                        else "libhanf.so")


class GraphView(Structure):
    _fields_ = [("n", c_uint64), ("num_arcs", c_uint64),
                ("offsets", POINTER(c_uint64)), ("arcs", POINTER(c_uint32))]


class Config(Structure):
    _fields_ = [("bucket_bits", c_uint32), ("register_bits", c_uint32),
                ("seed", c_uint64), ("threads", c_uint32), ("task_size", c_uint64),
                ("systolic_threshold", c_double), ("termination", c_int32),
                ("eps_inc", c_double), ("max_iterations", c_uint64),
                ("spill_to_disk", c_int32), ("track_modified", c_int32),
                ("use_systolic", c_int32), ("device", c_int32),
                ("exact_sum", c_int32), ("shard_begin", c_uint64),
                ("shard_end", c_uint64), ("shard_count", c_uint32), ("expected_runs", c_uint32)]


class IterationReportC(Structure):
    _fields_ = [("sum", c_double), ("modified", c_uint64)]


class SketchParamsC(Structure):
    _fields_ = [("bucket_bits", c_uint32), ("registers", c_uint32),
                ("register_bits", c_uint32), ("words_per_counter", c_uint32),
                ("alpha", c_double), ("seed", c_uint64)]


class BuffersC(Structure):
    _fields_ = [("next_counters", c_void_p), ("next_modified", c_void_p),
                ("block_sums", c_void_p), ("words_per_counter", c_uint64),
                ("blocks", c_uint64), ("shard_begin", c_uint64),
                ("shard_end", c_uint64), ("row_pitch", c_uint64),
                ("relabelled", c_uint32), ("reserved", c_uint32)]


class ShardPeerC(Structure):
    """hanf_shard_peer: one rank's exchange arena (peer-push exchange)."""
    _fields_ = [("ipc_handle", ctypes.c_uint8 * 64), ("arena_bytes", c_uint64),
                ("n", c_uint64), ("row_pitch", c_uint64), ("shard_begin", c_uint64),
                ("shard_end", c_uint64), ("device", c_int32), ("relabelled", c_int32)]


MAX_PEERS = 7

# status codes (hanf.h)
OK, INVALID_ARGUMENT, GUARD, OUT_OF_RANGE, CUDA_ERROR, OUT_OF_MEMORY, CAPACITY, \
    IO_ERROR, PARSE_ERROR = range(9)

_P = c_void_p
_SIGNATURES = {
    "hanf_config_init": [POINTER(Config)],
    "hanf_sketch_params_make": [c_uint32, c_uint64, c_uint32, POINTER(SketchParamsC)],
    "hanf_create": [POINTER(GraphView), POINTER(Config), POINTER(_P)],
    "hanf_create_multi": [POINTER(GraphView), POINTER(Config), POINTER(c_int32), c_uint32,
                          POINTER(_P)],
    "hanf_reset": [_P],
    "hanf_reseed": [_P, c_uint64],
    "hanf_create_batch": [POINTER(GraphView), POINTER(Config), POINTER(c_uint64), c_uint32,
                          POINTER(_P)],
    "hanf_run_batch": [_P, POINTER(c_double), POINTER(c_uint64), c_uint64, POINTER(c_uint64)],
    "hanf_save_counters": [_P, c_char_p],
    "hanf_exact_nf": [POINTER(GraphView), c_int32, c_uint64, c_uint64, POINTER(c_uint64),
                      c_uint64, POINTER(c_uint64)],
    "hanf_restore_counters": [_P, c_char_p, c_uint64],
    "hanf_sum_estimates": [_P, POINTER(c_double)],
    "hanf_step": [_P, POINTER(IterationReportC)],
    "hanf_step_launch": [_P],
    "hanf_step_complete": [_P, POINTER(IterationReportC)],
    "hanf_run_to_stabilisation": [_P, POINTER(c_double), POINTER(c_uint64), c_uint64,
                                  POINTER(c_uint64), POINTER(c_double)],
    "hanf_last_result": [_P, POINTER(c_double), POINTER(c_uint64), c_uint64,
                         POINTER(c_uint64)],
    "hanf_estimate_nf": [POINTER(GraphView), POINTER(Config), POINTER(c_double),
                         POINTER(c_uint64), c_uint64, POINTER(c_uint64), POINTER(c_double)],
    "hanf_read_counters": [_P, c_uint64, c_uint64, POINTER(c_uint64)],
    "hanf_params": [_P, POINTER(SketchParamsC)],
    "hanf_iteration": [_P, POINTER(c_uint64)],
    "hanf_systolic_active": [_P, POINTER(c_int32)],
    "hanf_num_nodes": [_P, POINTER(c_uint64)],
    "hanf_stream": [_P, POINTER(_P)],
    "hanf_launch_count": [_P, POINTER(c_uint64)],
    "hanf_block_stats": [_P, POINTER(c_uint64), POINTER(c_uint64)],
    "hanf_device_buffers": [_P, POINTER(BuffersC)],
    "hanf_set_timing": [_P, c_int32],
    "hanf_timing": [_P, POINTER(c_double), POINTER(c_double), POINTER(c_double),
                    POINTER(c_uint64)],
    "hanf_shard_compute": [_P],
    "hanf_shard_pack": [_P, _P, _P, c_uint64, POINTER(c_uint64)],
    "hanf_shard_unpack": [_P, _P, _P, c_uint64],
    "hanf_shard_commit": [_P, POINTER(IterationReportC)],
    "hanf_shard_export": [_P, POINTER(ShardPeerC)],
    "hanf_shard_attach": [_P, POINTER(ShardPeerC), c_uint32, c_uint32],
    "hanf_shard_attach_local": [_P, POINTER(_P), c_uint32, c_uint32],
    "hanf_shard_detach": [_P],
    "hanf_shard_wait": [_P],
    "hanf_shard_reduce": [_P],
    "hanf_shard_push_stats": [_P, POINTER(c_uint64), POINTER(c_uint64)],
    "hanf_distance_distribution": [POINTER(c_double), c_uint64, POINTER(c_double),
                                   POINTER(c_double), POINTER(c_double)],
    "hanf_effective_diameter": [POINTER(c_double), c_uint64, c_double, c_int32,
                                POINTER(c_double)],
    "hanf_graph_from_edges": [c_uint64, POINTER(c_uint32), POINTER(c_uint32), c_uint64,
                              POINTER(_P)],
    "hanf_gen_uniform_random": [c_uint64, c_double, c_uint64, POINTER(_P)],
    "hanf_gen_clique_path": [c_uint64, c_uint64, POINTER(_P)],
    "hanf_gen_erdos_renyi": [c_uint64, c_double, c_uint64, POINTER(_P)],
    "hanf_gen_rmat": [c_uint32, c_uint32, c_double, c_double, c_double, c_uint64,
                      c_uint64, POINTER(_P)],
    "hanf_gen_copying": [c_uint64, c_double, c_double, c_uint64, c_double, c_uint64,
                         c_uint64, POINTER(_P)],
    "hanf_gen_barabasi_albert": [c_uint64, c_uint32, c_uint64, c_uint64, POINTER(_P)],
    "hanf_graph_transpose": [_P, POINTER(_P)],
    "hanf_graph_save_csr": [_P, c_char_p],
    "hanf_graph_load_csr": [c_char_p, POINTER(_P)],
    "hanf_graph_view_of": [_P, POINTER(GraphView)],
    "hanf_pin_host": [_P, c_uint64],
    "hanf_graph_from_edges_gpu": [c_int32, c_uint64, POINTER(c_uint32), POINTER(c_uint32),
                                  c_uint64, POINTER(_P)],
    "hanf_gen_rmat_gpu": [c_int32, c_uint32, c_uint32, c_double, c_double, c_double, c_uint64,
                          c_uint64, POINTER(_P)],
    "hanf_unpin_host": [_P],
}
_VOID = {"hanf_destroy": [_P], "hanf_graph_free": [_P]}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libhanf.so once; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import "
                f"__graft_entry__ as g; g.build()'` or `make -C paper_1011_5599_b200/csrc`")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c_int32
        for name, args in _VOID.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = None
        L.hanf_last_error.argtypes = []
        L.hanf_last_error.restype = c_char_p
        _lib = L
    return _lib


class GuardError(RuntimeError):
    """hyperanf::GuardError (errors.hpp:18-20): a resource guard refused."""


class ParseError(RuntimeError):
    """hyperanf::ParseError (errors.hpp:8-10)."""


class IoError(RuntimeError):
    """hyperanf::IoError (errors.hpp:13-15)."""


class CudaError(RuntimeError):
    """Device failure (std::runtime_error on the C++ side)."""


class CapacityError(RuntimeError):
    """Caller-provided output buffer too small."""


def check(status: int) -> None:
    """Maps a hanf_status to the reference's exception taxonomy."""
    if status == OK:
        return
    msg = lib().hanf_last_error().decode("utf-8", "replace")
    if status == INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if status == GUARD:
        raise GuardError(msg)
    if status == OUT_OF_RANGE:
        raise IndexError(msg)          # std::out_of_range
    if status == OUT_OF_MEMORY:
        raise MemoryError(msg)
    if status == CAPACITY:
        raise CapacityError(msg)
    if status == IO_ERROR:
        raise IoError(msg)
    if status == PARSE_ERROR:
        raise ParseError(msg)
    raise CudaError(msg)
