"""ctypes binding of include/fsdp.h -- argument marshalling only.

Every step of the hot path runs inside libfsdp_b200.so (C++ host core +
sm_100a kernels + NCCL).  Importing this module loads the library and fails
loudly if it is missing: there is no fallback.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSDP_B200_LIB selects a tuning variant built by build.py (tools/kernel_sweep.py).
LIB_PATH = os.environ.get("FSDP_B200_LIB") or os.path.join(_HERE, "libfsdp_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "libfsdp_b200.so is not built (%s); run `python -m paper_2411_00284_b200.build` "
        "or __graft_entry__.build(). There is no CPU fallback." % LIB_PATH)

lib = C.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants
FSDP_OK, FSDP_ERR_INVALID_ARG, FSDP_ERR_CUDA, FSDP_ERR_NCCL, FSDP_ERR_OOM, FSDP_ERR_UNSUPPORTED = range(6)
BF16, FP32 = 0, 1
PLAN_PER_PARAM, PLAN_MANUAL, PLAN_SIZE_CAP, PLAN_GREEDY = range(4)
PHASE_FWD, PHASE_BWD = 0, 1
ISSUE, WAIT, NO_COLLECTIVE = 1, 2, 4
NVLS_HANDLE_BYTES = 80
NVLS_FABRIC, NVLS_POSIX_FD = 1, 2
(OP_PACK_AG, OP_AG, OP_WAIT_AG, OP_UNPACK, OP_COMPUTE_F, OP_COMPUTE_B, OP_PACK_RS, OP_RS,
 OP_WAIT_RS, OP_COPYOUT_RS) = range(10)
N_OPS = 10
SCHED_REORDER, SCHED_FWD_AG_BEFORE_WAIT, SCHED_BWD_AG_BEFORE_WAIT = 1, 2, 4
SCHED_NO_COMM, SCHED_DRY_RUN, SCHED_TIMING, SCHED_P2P = 8, 16, 32, 64
SCHED_KEEP_LAST_GATHERED = 128
SCHED_COPY_STREAM = 256
BUCKET_SEGMENT_SHARDS, BUCKET_SEGMENT_GRAD_SHARDS, BUCKET_FP32_MASTER, BUCKET_GROUPED_AG = 1, 2, 4, 8
BUCKET_BF16_GRAD_SHARDS = 16
REG_LOCAL, REG_SYMMETRIC = 0, 1

EXPORTED = [
    "fsdp_last_error", "fsdp_abi_version", "fsdp_nccl_get_unique_id", "fsdp_ctx_create",
    "fsdp_ctx_destroy", "fsdp_ctx_split", "fsdp_ctx_info", "fsdp_ctx_create_config", "fsdp_nccl_estimate_ns", "fsdp_shard", "fsdp_plan_buckets", "fsdp_layout", "fsdp_bucket_create",
    "fsdp_bucket_destroy", "fsdp_bucket_query", "fsdp_bucket_set_grad_accumulation",
    "fsdp_allgather_bucket", "fsdp_reduce_scatter_bucket", "fsdp_bucket_launch_kernel",
    "fsdp_run_schedule", "fsdp_proxy_launch", "fsdp_proxy_calibrate",
    "fsdp_p2p_allgather_bucket", "fsdp_p2p_reduce_scatter_bucket", "fsdp_p2p_signal", "fsdp_p2p_wait",
    "fsdp_ipc_alloc", "fsdp_ipc_open", "fsdp_ipc_close", "fsdp_ipc_free",
    "fsdp_mem_alloc", "fsdp_mem_free", "fsdp_register_buffer", "fsdp_window_peer_pointers",
    "fsdp_window_multimem_pointer",
    "fsdp_nvls_create", "fsdp_nvls_import", "fsdp_nvls_bind", "fsdp_nvls_destroy",
    "fsdp_nvls_reduce_scatter_bucket",
    "fsdp_step_graph_create", "fsdp_step_graph_launch", "fsdp_step_graph_info", "fsdp_step_graph_destroy",
    "fsdp_comm_time_ns", "fsdp_simulate_schedule", "fsdp_simulate_memory", "fsdp_plan_search",
]


# -------------------------------------------------------------------- structs
class ParamDesc(C.Structure):
    _fields_ = [("dim0", C.c_int64), ("row_numel", C.c_int64), ("module_id", C.c_int32),
                ("reserved", C.c_int32)]


class ShardInfo(C.Structure):
    _fields_ = [("shard_rows", C.c_int64), ("row_begin", C.c_int64), ("valid_rows", C.c_int64),
                ("shard_numel", C.c_int64)]


class Link(C.Structure):
    _fields_ = [("alpha_ns", C.c_int64), ("beta_fs_per_byte", C.c_int64)]


class PlanIn(C.Structure):
    _fields_ = [("params", C.POINTER(ParamDesc)), ("t_compute_ns", C.POINTER(C.c_int64)),
                ("mem_bytes", C.POINTER(C.c_int64)), ("ag", Link), ("rs", Link),
                ("mem_max_bytes", C.c_int64), ("n_params", C.c_int32), ("world", C.c_int32),
                ("align_bytes", C.c_int32), ("mode", C.c_int32), ("phase", C.c_int32),
                ("param_dtype", C.c_int32), ("reduce_bytes", C.c_int32), ("reserved", C.c_int32)]


class PlanTrace(C.Structure):
    _fields_ = [("t_lhs_ns", C.c_int64), ("t_rhs_ns", C.c_int64), ("m_lhs", C.c_int64),
                ("m_rhs", C.c_int64), ("param", C.c_int32), ("accept", C.c_int32)]


class BucketDesc(C.Structure):
    _fields_ = [("params", C.POINTER(ParamDesc)), ("shards", C.POINTER(C.c_void_p)),
                ("fulls", C.POINTER(C.c_void_p)), ("full_grads", C.POINTER(C.c_void_p)),
                ("grad_shards", C.POINTER(C.c_void_p)), ("k", C.c_int32), ("align_bytes", C.c_int32),
                ("param_dtype", C.c_int32), ("grad_dtype", C.c_int32), ("flags", C.c_uint32),
                ("reserved", C.c_int32)]


class BucketInfo(C.Structure):
    _fields_ = [("ag_seg_bytes", C.c_int64), ("rs_seg_bytes", C.c_int64), ("kernel_bytes", C.c_int64 * 4),
                ("kernel_chunks", C.c_int32 * 4), ("ag_zero_copy", C.c_int32), ("rs_zero_copy", C.c_int32),
                ("p2p_bytes", C.c_int64 * 2), ("ag_direct", C.c_int32), ("ag_grouped", C.c_int32)]


class P2PSchedule(C.Structure):
    _fields_ = [("ag_peers", C.POINTER(C.c_void_p)), ("rs_peers", C.POINTER(C.c_void_p)),
                ("ready_slots", C.POINTER(C.c_void_p)), ("done_slots", C.POINTER(C.c_void_p)),
                ("ready_flags", C.c_void_p), ("done_flags", C.c_void_p), ("epoch_base", C.c_uint64),
                ("timeout_ns", C.c_int64), ("error_flag", C.c_void_p), ("epoch_counter", C.c_void_p),
                ("max_ctas", C.c_int32), ("grad_slots", C.c_int32)]


class HostIO(C.Structure):
    _fields_ = [("fwd_host_shards", C.POINTER(C.c_void_p)), ("bwd_host_grads", C.POINTER(C.c_void_p)),
                ("h2d", C.c_void_p), ("d2h", C.c_void_p), ("async_d2h", C.c_int32), ("reserved", C.c_int32)]


class GemmCompute(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("x", C.c_void_p), ("dy", C.c_void_p), ("y", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64)]


class CommEmulation(C.Structure):
    _fields_ = [("ag", Link), ("rs", Link), ("ctas", C.c_int32), ("reserved", C.c_int32)]


COMPUTE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p)


class ComputeHook(C.Structure):
    _fields_ = [("fn", COMPUTE_FN), ("user", C.c_void_p)]


class Schedule(C.Structure):
    _fields_ = [("fwd", C.POINTER(C.c_void_p)), ("bwd", C.POINTER(C.c_void_p)),
                ("proxy_iters_fwd", C.POINTER(C.c_int64)), ("proxy_iters_bwd", C.POINTER(C.c_int64)),
                ("ag_staging", C.c_void_p * 2), ("rs_staging", C.c_void_p * 2),
                ("compute", C.c_void_p), ("comm", C.c_void_p), ("n_fwd", C.c_int32),
                ("n_bwd", C.c_int32), ("flags", C.c_uint32), ("proxy_ctas_per_sm", C.c_int32),
                ("proxy_smem_bytes", C.c_int32), ("reserved", C.c_int32), ("p2p", C.POINTER(P2PSchedule)),
                ("io", C.POINTER(HostIO)), ("gemm", C.POINTER(GemmCompute)),
                ("hook", C.POINTER(ComputeHook)), ("emulate", C.POINTER(CommEmulation))]


class MemSizes(C.Structure):
    _fields_ = [("ag_fwd", C.POINTER(C.c_int64)), ("full_fwd", C.POINTER(C.c_int64)),
                ("ag_bwd", C.POINTER(C.c_int64)), ("full_bwd", C.POINTER(C.c_int64)),
                ("grad_bwd", C.POINTER(C.c_int64)), ("rs_bwd", C.POINTER(C.c_int64)),
                ("n_fwd", C.c_int32), ("n_bwd", C.c_int32)]


class NcclConfig(C.Structure):
    _fields_ = [("min_ctas", C.c_int32), ("max_ctas", C.c_int32), ("nvls_ctas", C.c_int32),
                ("cta_policy", C.c_int32)]


class SearchCost(C.Structure):
    _fields_ = [("unpack_bytes_per_us", C.c_int64), ("pack_rs_bytes_per_us", C.c_int64),
                ("copy_launch_ns", C.c_int64), ("compute_overhead_ns", C.c_int64), ("sched_flags", C.c_uint32),
                ("max_moves", C.c_int32)]


class LogEntry(C.Structure):
    _fields_ = [("ns", C.c_int64), ("phase", C.c_int32), ("op", C.c_int32), ("bucket", C.c_int32),
                ("stream", C.c_int32), ("start_ns", C.c_int64)]


class StepReport(C.Structure):
    _fields_ = [("log", C.POINTER(LogEntry)), ("log_capacity", C.c_int32), ("log_len", C.c_int32),
                ("step_ns", C.c_int64), ("op_ns", C.c_int64 * N_OPS), ("op_count", C.c_int32 * N_OPS),
                ("kernel_launches", C.c_int32), ("collectives", C.c_int32)]


# ------------------------------------------------------------------ prototypes
_P = C.c_void_p
_sigs = {
    "fsdp_last_error": (C.c_char_p, []),
    "fsdp_abi_version": (C.c_int32, []),
    "fsdp_nccl_get_unique_id": (C.c_int, [_P]),
    "fsdp_ctx_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "fsdp_ctx_destroy": (C.c_int, [_P]),
    "fsdp_ctx_create_config": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, C.c_int32, _P,
                                         C.POINTER(NcclConfig)]),
    "fsdp_nccl_estimate_ns": (C.c_int, [_P, C.c_int32, C.c_int64, C.POINTER(C.c_int64)]),
    "fsdp_ctx_split": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "fsdp_ctx_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fsdp_shard": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(ParamDesc), C.c_int, _P, _P,
                             C.POINTER(ShardInfo), _P]),
    "fsdp_plan_buckets": (C.c_int, [C.POINTER(PlanIn), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(PlanTrace)]),
    "fsdp_layout": (C.c_int, [C.POINTER(ParamDesc), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                              C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "fsdp_bucket_create": (C.c_int, [_P, C.POINTER(BucketDesc), C.POINTER(_P), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]),
    "fsdp_bucket_destroy": (C.c_int, [_P]),
    "fsdp_bucket_query": (C.c_int, [_P, C.POINTER(BucketInfo)]),
    "fsdp_bucket_set_grad_accumulation": (C.c_int, [_P, C.c_int32]),
    "fsdp_allgather_bucket": (C.c_int, [_P, _P, _P, _P, _P, C.c_uint32]),
    "fsdp_reduce_scatter_bucket": (C.c_int, [_P, _P, _P, _P, _P, C.c_uint32]),
    "fsdp_bucket_launch_kernel": (C.c_int, [_P, _P, C.c_int32, _P, _P, C.POINTER(C.c_int32)]),
    "fsdp_run_schedule": (C.c_int, [_P, C.POINTER(Schedule), C.POINTER(StepReport)]),
    "fsdp_proxy_launch": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, _P]),
    "fsdp_proxy_calibrate": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P,
                                       C.POINTER(C.c_int64)]),
    "fsdp_p2p_allgather_bucket": (C.c_int, [_P, _P, C.POINTER(_P), _P]),
    "fsdp_p2p_reduce_scatter_bucket": (C.c_int, [_P, _P, C.POINTER(_P), _P]),
    "fsdp_p2p_signal": (C.c_int, [_P, C.POINTER(_P), C.c_uint64, _P]),
    "fsdp_p2p_wait": (C.c_int, [_P, _P, C.c_uint64, C.c_int64, _P, _P]),
    "fsdp_ipc_alloc": (C.c_int, [C.c_int64, C.POINTER(_P), _P]),
    "fsdp_ipc_open": (C.c_int, [_P, C.POINTER(_P)]),
    "fsdp_ipc_close": (C.c_int, [_P]),
    "fsdp_ipc_free": (C.c_int, [_P]),
    "fsdp_mem_alloc": (C.c_int, [_P, C.c_int64, C.POINTER(_P)]),
    "fsdp_mem_free": (C.c_int, [_P, _P]),
    "fsdp_register_buffer": (C.c_int, [_P, _P, C.c_int64, C.c_int32]),
    "fsdp_window_peer_pointers": (C.c_int, [_P, _P, C.POINTER(C.c_void_p)]),
    "fsdp_window_multimem_pointer": (C.c_int, [_P, _P, C.POINTER(C.c_void_p)]),
    "fsdp_nvls_create": (C.c_int, [_P, C.c_int64, _P, C.POINTER(_P)]),
    "fsdp_nvls_import": (C.c_int, [_P, _P, C.c_int64, C.POINTER(_P)]),
    "fsdp_nvls_bind": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(C.c_int64)]),
    "fsdp_nvls_destroy": (C.c_int, [_P]),
    "fsdp_nvls_reduce_scatter_bucket": (C.c_int, [_P, _P, _P, _P]),
    "fsdp_step_graph_create": (C.c_int, [_P, C.POINTER(Schedule), C.POINTER(_P)]),
    "fsdp_step_graph_launch": (C.c_int, [_P, _P]),
    "fsdp_step_graph_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fsdp_step_graph_destroy": (C.c_int, [_P]),
    "fsdp_comm_time_ns": (C.c_int, [C.c_int64, C.POINTER(Link), C.POINTER(C.c_int64)]),
    "fsdp_simulate_schedule": (C.c_int, [C.POINTER(LogEntry), C.c_int32, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64)]),
    "fsdp_plan_search": (C.c_int, [C.POINTER(PlanIn), C.POINTER(SearchCost), C.POINTER(C.c_int32), C.c_int32,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "fsdp_simulate_memory": (C.c_int, [C.POINTER(LogEntry), C.c_int32, C.POINTER(MemSizes),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class FsdpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("fsdp status %d: %s" % (status, msg))
        self.status = status


def check(status):
    if status != FSDP_OK:
        raise FsdpError(status, lib.fsdp_last_error().decode(errors="replace"))


def descs(params):
    """params: iterable of (dim0, row_numel, module_id) -> ctypes array."""
    params = list(params)
    arr = (ParamDesc * len(params))()
    for i, p in enumerate(params):
        arr[i].dim0, arr[i].row_numel, arr[i].module_id, arr[i].reserved = int(p[0]), int(p[1]), int(p[2]), 0
    return arr


def ptr_array(ptrs):
    if ptrs is None:
        return None
    ptrs = list(ptrs)
    return (C.c_void_p * len(ptrs))(*[C.c_void_p(int(p)) for p in ptrs])


def i64_array(vals):
    if vals is None:
        return None
    vals = list(vals)
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])
