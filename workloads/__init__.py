"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This package holds NO arithmetic of the method (no sharding, layout, bucketing,
collective, planning or scheduling logic).  It only describes workloads:
parameter shapes in forward-use order (Table 2 of the paper), seeded
random tensors, and the synthetic per-parameter compute times that stand in
for the profiler's measured T_ci.  Both ``oracle/`` and the
product binding may import it; it imports neither.
"""
from .shapes import ParamSpec, toy_mlp, llama, LLAMA_CONFIGS  # noqa: F401
