"""O6 -- communication cost model (test infrastructure; see oracle/__init__.py).

P:222: "we formulate the estimated communication time as T_m = alpha + beta n
where n denotes the transmitted word size".  P:175: the base latency is paid
once per issued collective.

Readings: integer nanoseconds (G9, following S:237), beta in femtoseconds per
byte, ceiling rounding; n is the collective's full bucket bytes in its dtype,
layout padding included (G8).
"""


def comm_time(nbytes, alpha_ns, beta_fs_per_byte):
    """T(n) = alpha + ceil(n * beta / 10^6) ns (exact integer arithmetic)."""
    if nbytes < 0 or alpha_ns < 0 or beta_fs_per_byte < 0:
        raise ValueError("negative cost input")
    return alpha_ns + -(-(nbytes * beta_fs_per_byte) // 10**6)
