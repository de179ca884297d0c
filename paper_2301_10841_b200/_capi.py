"""ctypes binding of include/fjg.h (libfjg.so).

The product path has no fallback: if libfjg.so is missing or fails to load,
importing this module raises (build it with paper_2301_10841_b200/build.py or
__graft_entry__.build()).
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FJG_LIB") or os.path.join(_HERE, "libfjg.so")

FJG_OK, FJG_E_IO, FJG_E_PARSE, FJG_E_VALIDATION, FJG_E_RESOURCE, FJG_E_ENGINE = range(6)
MAX_NODES = 32
MAX_ATOMS = 16


# error.hpp:9-33 categories, mirrored as Python exceptions
class Error(RuntimeError):
    code = FJG_E_ENGINE


class IoError(Error):
    code = FJG_E_IO


class ParseError(Error):
    code = FJG_E_PARSE


class ValidationError(Error):
    code = FJG_E_VALIDATION


class ResourceError(Error):
    code = FJG_E_RESOURCE


class EngineError(Error):
    code = FJG_E_ENGINE


_BY_CODE = {c.code: c for c in (IoError, ParseError, ValidationError, ResourceError, EngineError)}


class ExecOptions(C.Structure):
    _fields_ = [("batch_size", C.c_uint64), ("dynamic_cover", C.c_int32), ("output_mode", C.c_int32),
                ("min_var", C.c_int32), ("collect_timing", C.c_int32), ("backend", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("count_lo", C.c_uint64), ("count_hi", C.c_uint64), ("checksum", C.c_uint64),
                ("min_value", C.c_int64), ("has_min", C.c_int32), ("num_nodes", C.c_int32),
                ("output_rows", C.c_uint64), ("probes", C.c_uint64), ("probe_misses", C.c_uint64),
                ("node_body_entries", C.c_uint64 * MAX_NODES), ("node_probes", C.c_uint64 * MAX_NODES),
                ("node_inputs", C.c_uint64 * MAX_NODES), ("maps_built", C.c_uint64),
                ("keys_inserted", C.c_uint64), ("forces", C.c_uint64), ("rows_forced", C.c_uint64),
                ("build_ms", C.c_double), ("join_ms", C.c_double), ("last_node_ms", C.c_double),
                ("last_node_launches", C.c_uint64), ("last_node_candidates", C.c_uint64),
                ("first_node_ms", C.c_double),
                ("memo_ms", C.c_double), ("memo_rows_resolved", C.c_uint64), ("memo_rows_gathered", C.c_uint64),
                ("memo_rows_init", C.c_uint64),
                ("atom_maps_built", C.c_uint64 * MAX_ATOMS), ("atom_levels_forced", C.c_uint32 * MAX_ATOMS),
                ("kernel_launches", C.c_uint32),
                ("host_syncs", C.c_uint32)]


MAX_VIEWS = 16
COMM_ID_BYTES = 128


class MultiInfo(C.Structure):
    _fields_ = [("local_count_lo", C.c_uint64), ("local_count_hi", C.c_uint64), ("local_checksum", C.c_uint64),
                ("bytes_sent", C.c_uint64), ("bytes_received", C.c_uint64),
                ("view_rows", C.c_uint64 * MAX_VIEWS), ("nviews", C.c_int32), ("pad_", C.c_int32),
                ("exchange_ms", C.c_double), ("reduce_ms", C.c_double)]


class Predicate(C.Structure):
    _fields_ = [("column", C.c_int32), ("cmp", C.c_int32), ("is_column", C.c_int32), ("rhs_column", C.c_int32),
                ("constant", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_2301_10841_b200/build.py (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    P, I, U64, SZ = C.c_void_p, C.c_int, C.c_uint64, C.c_size_t
    sig = {
        "fjg_last_error": (C.c_char_p, []),
        "fjg_abi_version": (I, []),
        "fjg_compile_plan": (I, [C.c_char_p, I, I, C.c_char_p, SZ, C.POINTER(SZ)]),
        "fjg_plan_op": (I, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, SZ, C.POINTER(SZ)]),
        "fjg_engine_create": (I, [I, C.POINTER(P)]),
        "fjg_engine_destroy": (None, [P]),
        "fjg_engine_sync": (I, [P]),
        "fjg_engine_stream": (P, [P]),
        "fjg_relation_create": (I, [P, C.POINTER(P), I, U64, C.POINTER(P)]),
        "fjg_relation_create_i64": (I, [P, C.POINTER(P), I, U64, C.POINTER(P)]),
        "fjg_relation_from_device": (I, [P, C.POINTER(P), I, U64, I, C.POINTER(P)]),
        "fjg_relation_filter": (I, [P, C.POINTER(Predicate), I, C.POINTER(P)]),
        "fjg_relation_rows": (U64, [P]),
        "fjg_relation_cols": (I, [P]),
        "fjg_relation_device_col": (P, [P, I]),
        "fjg_relation_download": (I, [P, I, P]),
        "fjg_relation_destroy": (None, [P]),
        "fjg_relation_partition": (I, [P, I, I, C.POINTER(P), C.POINTER(U64)]),
        "fjg_relation_partition_into": (I, [P, I, I, C.POINTER(P), C.POINTER(U64)]),
        "fjg_query_create": (I, [P, C.c_char_p, C.c_char_p, C.POINTER(P), I, C.POINTER(P)]),
        "fjg_execute": (I, [P, C.POINTER(ExecOptions), C.POINTER(Result)]),
        "fjg_query_output": (I, [P, P, U64, C.POINTER(U64)]),
        "fjg_query_num_head_vars": (I, [P]),
        "fjg_query_output_relation": (I, [P, C.POINTER(P)]),
        "fjg_query_destroy": (None, [P]),
        "fjg_device_tuple_hash": (I, [P, P, I, U64, P]),
        "fjg_device_primitive_check": (I, [P, I, U64, I, I, U64, P]),
        "fjg_host_tuple_hash": (U64, [P, I]),
        "fjg_parse_csv": (I, [C.c_char_p, I, P, U64, C.POINTER(U64)]),
        "fjg_comm_unique_id": (I, [P]),
        "fjg_comm_create": (I, [P, P, I, I, C.POINTER(P)]),
        "fjg_comm_size": (I, [P]),
        "fjg_comm_rank": (I, [P]),
        "fjg_comm_destroy": (None, [P]),
        "fjg_sharded_create": (I, [P, C.c_char_p, C.c_char_p, C.POINTER(P), I, C.POINTER(I), C.POINTER(I), I,
                                   C.POINTER(P)]),
        "fjg_execute_multi": (I, [P, C.POINTER(ExecOptions), C.POINTER(Result), C.POINTER(MultiInfo)]),
        "fjg_sharded_destroy": (None, [P]),
        "fjg_exchange_layout": (I, [P, I, I, I, P, P, P]),
        "fjg_colt_create": (I, [P, P, P, P, I, C.POINTER(P)]),
        "fjg_colt_levels": (I, [P]),
        "fjg_colt_force": (I, [P, I, P, P, U64]),
        "fjg_colt_get": (I, [P, I, P, P, P, U64, P, P, P]),
        "fjg_colt_iter": (I, [P, I, C.c_uint32, C.c_uint32, P, P, P, U64, C.POINTER(U64)]),
        "fjg_colt_rows": (I, [P, I, C.c_uint32, C.c_uint32, I, P]),
        "fjg_colt_estimated_key_count": (I, [P, I, C.c_uint32, C.c_uint32, C.POINTER(U64)]),
        "fjg_colt_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()

# every symbol include/fjg.h declares (checked by tests/test_capi.py)
EXPORTED = ["fjg_last_error", "fjg_abi_version", "fjg_compile_plan", "fjg_plan_op", "fjg_engine_create",
            "fjg_engine_destroy", "fjg_engine_sync", "fjg_engine_stream", "fjg_relation_create", "fjg_relation_create_i64",
            "fjg_relation_from_device",
            "fjg_relation_filter", "fjg_relation_rows", "fjg_relation_cols", "fjg_relation_device_col",
            "fjg_relation_download", "fjg_relation_destroy", "fjg_relation_partition",
            "fjg_relation_partition_into", "fjg_query_create",
            "fjg_execute", "fjg_query_output", "fjg_query_num_head_vars", "fjg_query_output_relation", "fjg_query_destroy",
            "fjg_device_tuple_hash", "fjg_device_primitive_check", "fjg_host_tuple_hash", "fjg_parse_csv", "fjg_comm_unique_id", "fjg_comm_create",
            "fjg_comm_size", "fjg_comm_rank", "fjg_comm_destroy", "fjg_sharded_create", "fjg_execute_multi",
            "fjg_sharded_destroy", "fjg_exchange_layout", "fjg_colt_create", "fjg_colt_levels", "fjg_colt_force",
            "fjg_colt_get", "fjg_colt_iter", "fjg_colt_rows", "fjg_colt_estimated_key_count", "fjg_colt_destroy"]


def check(rc):
    if rc != FJG_OK:
        msg = lib.fjg_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, Error)(msg)


def call_str(fn, *args):
    """Call an fjg_* function with the (out, cap, needed) string convention."""
    need = C.c_size_t(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = fn(*args, buf, cap, C.byref(need))
        if rc == FJG_E_RESOURCE and need.value > cap:
            cap = need.value
            continue
        check(rc)
        return buf.value.decode()
