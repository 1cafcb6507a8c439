"""CPU oracle for the SimpleFSDP (arXiv 2411.00284) data-parallel hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2411_00284_b200``, ``csrc``) never
imports, links or executes it, and this package imports nothing from the
product: the two share no code.  Inputs for both sides come from the separate
``workloads`` package, which holds none of the method's arithmetic.

Plain, slow, obviously-correct NumPy, following the paper's wording.
Citations ``P:<line>`` are lines of ``PAPER.md`` (the paper's LaTeX source),
``S:<line>`` lines of ``SPEC.md``; ``SURVEY §8(c) O<k>`` names the oracle part
in the blueprint and ``G<k>`` a reading from the ambiguity register that
DESIGN.md restates.

Modules
-------
bf16        O1  bf16 codec (widen / round-to-nearest-even narrow)
shard       O2  per-parameter dim-0 sharding
layout      O3  flat bucket layout
collectives O4/O5 bucketed all-gather and reduce-scatter(avg) over N simulated ranks;
            mixed-precision (fp32 master) all-gather, gradient accumulation
cost        O6  alpha + beta*n communication model
planner     O8  Algorithm 1 greedy auto-wrap + manual / per-param / size-cap plans
schedule    O9  reordered / vanilla op sequences (Table 6)
sim         O10 two-stream discrete-event simulator
brute       O8(iv) exhaustive contiguous-partition search
mesh        O11 2-D DP x TP composition: TP blocks, FSDP on the DP sub-mesh

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against values or properties the paper or the
mathematics fix.  Measured quantities (alpha/beta fits, calibrated proxy
times, measured exposure) are inputs, not oracle functions: parity unpinned
by construction and never used as a pass/fail parity value.
"""
