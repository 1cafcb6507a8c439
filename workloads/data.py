"""Seeded synthetic tensors (no method arithmetic).

Host generators use NumPy's counter-based Philox bit generator, so every
array is a pure function of (seed, shape).  bf16 values are produced as bit
patterns by truncating a float32 draw to its high 16 bits (a generator choice,
not the method's fp32 -> bf16 rounding).

Recipe: parameters ~ N(0, 0.02) (Llama init), norm
weights = 1.0; gradients of rank r ~ N(0, 1e-3) from seed + r; an
exactly-representable set k * 2^-8 (|k| <= 256) and an edge set
(+-0, subnormals, +-inf, NaN) for unit tests.
"""
import numpy as np

BF16_ONE = np.uint16(0x3F80)


def rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def f32_normal(shape, std, seed):
    return (rng(seed).standard_normal(shape, dtype=np.float32) * np.float32(std)).astype(np.float32)


def bf16_normal(shape, std, seed):
    """bf16 bit patterns (uint16) of N(0, std) draws, by truncation."""
    f = f32_normal(shape, std, seed)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def f32_exact(shape, seed):
    """k * 2^-8 with integer |k| <= 256: exactly representable in bf16, and
    every partial sum of such values (times 2^-j) is exact in fp32."""
    k = rng(seed).integers(-256, 257, size=shape).astype(np.float32)
    return (k * np.float32(2.0 ** -8)).astype(np.float32)


def bf16_exact(shape, seed):
    """The same values as ``f32_exact`` as bf16 bit patterns (the low 16 bits
    of each fp32 pattern are zero, so truncation loses nothing)."""
    f = f32_exact(shape, seed)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


EDGE_F32_BITS = np.array([
    0x00000000, 0x80000000,               # +0, -0
    0x00000001, 0x807FFFFF, 0x00400000,   # fp32 subnormals
    0x7F800000, 0xFF800000,               # +inf, -inf
    0x7FC00000, 0xFFC00001,               # NaNs
    0x7F7FFFFF, 0x00800000, 0x3F800000,   # max, min normal, 1.0
], dtype=np.uint32)

EDGE_BF16_BITS = np.array([
    0x0000, 0x8000,          # +0, -0
    0x0001, 0x807F, 0x0040,  # bf16 subnormals
    0x7F80, 0xFF80,          # +-inf
    0x7FC0, 0xFFC1,          # NaNs
    0x7F7F, 0x0080, 0x3F80,  # max, min normal, 1.0
], dtype=np.uint16)


def param_tensor(spec, dtype, seed):
    """Full [d, R] parameter for a ParamSpec: norms (R == 1, name *norm*) are
    1.0, everything else N(0, 0.02)."""
    shape = (spec.dim0, spec.row_numel)
    is_norm = spec.row_numel == 1 and "norm" in spec.name
    if dtype == "bf16":
        if is_norm:
            return np.full(shape, BF16_ONE, dtype=np.uint16)
        return bf16_normal(shape, 0.02, seed)
    if dtype == "f32":
        if is_norm:
            return np.ones(shape, dtype=np.float32)
        return f32_normal(shape, 0.02, seed)
    raise ValueError(dtype)


def grad_tensor(spec, dtype, seed, rank, kind="normal"):
    """Rank ``rank``'s full gradient of a parameter (seed + rank)."""
    shape = (spec.dim0, spec.row_numel)
    s = seed * 1009 + rank
    if kind == "exact":
        return bf16_exact(shape, s) if dtype == "bf16" else f32_exact(shape, s)
    if dtype == "bf16":
        return bf16_normal(shape, 1e-3, s)
    if dtype == "f32":
        return f32_normal(shape, 1e-3, s)
    raise ValueError(dtype)
