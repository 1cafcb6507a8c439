"""B200-native SimpleFSDP (arXiv 2411.00284) data-parallel hot path.

The product is the C-ABI library ``libfsdp_b200.so`` (include/fsdp.h):
fsdp_shard, fsdp_plan_buckets, fsdp_allgather_bucket, fsdp_reduce_scatter_bucket,
fsdp_run_schedule.  ``paper_2411_00284_b200.fsdp`` exposes the same names to
Python (marshalling only).  Any use of the API loads the built library and
raises ImportError if it is missing: there is no CPU fallback.  (Attributes are
resolved lazily so that ``python -m paper_2411_00284_b200.build`` can run
before the library exists.)
"""
_API = ("Bucket", "Ctx", "abi_version", "allgather_bucket", "layout", "nccl_get_unique_id",
        "plan_buckets", "proxy_calibrate", "proxy_launch", "reduce_scatter_bucket", "run_schedule",
        "shard", "p2p_allgather_bucket", "p2p_reduce_scatter_bucket", "p2p_signal", "p2p_wait",
        "ipc_alloc", "ipc_open", "ipc_close", "ipc_free", "comm_time_ns", "simulate_schedule",
        "mem_alloc", "mem_free", "register_buffer", "Nvls", "nvls_reduce_scatter_bucket",
        "StepGraph", "simulate_memory", "plan_search", "bucket_launch_kernel",
        "window_peer_pointers", "window_multimem_pointer")


def __getattr__(name):
    if name in _API:
        from . import fsdp
        return getattr(fsdp, name)
    if name.isupper() or name == "FsdpError":
        from . import _lib
        return getattr(_lib, name)
    raise AttributeError(name)
