"""O9 -- op sequences of one training step (test infrastructure; see oracle/__init__.py).

Reordering, P:184-193 (Fig. 2 prose):
  (1) forward: "AG34 is reordered in front of Wa12.  It allows AG34 to overlap
      with compute C1";
  (2) backward: "AG34 is placed after Wa12 ... The Wr12 is placed before RS34,
      such that RS12 can overlap with the later compute C3 and C4".
Placement ablation, Table 6: AG before / after the last AG-wait,
per phase; default = forward before, backward after (the table's best row,
G17).  "After" = after the wait *and its copy-out* (G33).
Vanilla: each collective issued immediately before its wait.
Prefetch depth 1 (G16); first AG of each phase and the last RS are exposed
(G18); every parameter is re-gathered in backward (G29).

An entry is (phase, op, bucket, stream): phase 0 forward / 1 backward, bucket =
index within the phase's execution order, stream 0 compute / 1 comm.  The
sequence is the host enqueue order.
"""
PACK_AG, AG, WAIT_AG, UNPACK, COMPUTE_F, COMPUTE_B, PACK_RS, RS, WAIT_RS, COPYOUT_RS = range(10)
OP_NAMES = ["PACK_AG", "AG", "WAIT_AG", "UNPACK", "COMPUTE_F", "COMPUTE_B",
            "PACK_RS", "RS", "WAIT_RS", "COPYOUT_RS"]
COMM_OPS = (AG, RS)
BEFORE, AFTER = "before", "after"


def _e(phase, op, b):
    return (phase, op, b, 1 if op in COMM_OPS else 0)


def forward_sequence(k, reorder=True, placement=BEFORE):
    s = []
    if not reorder:
        for b in range(k):
            s += [_e(0, PACK_AG, b), _e(0, AG, b), _e(0, WAIT_AG, b), _e(0, UNPACK, b),
                  _e(0, COMPUTE_F, b)]
        return s
    if k:
        s += [_e(0, PACK_AG, 0), _e(0, AG, 0)]
    for b in range(k):
        pre = [_e(0, PACK_AG, b + 1), _e(0, AG, b + 1)] if b + 1 < k else []
        wait = [_e(0, WAIT_AG, b), _e(0, UNPACK, b)]
        s += (pre + wait) if placement == BEFORE else (wait + pre)
        s.append(_e(0, COMPUTE_F, b))
    return s


def backward_sequence(k, reorder=True, placement=AFTER, keep_first=False):
    """keep_first (reading G42, an FSDP2-style option the paper does not
    describe -- P:137 re-gathers every parameter): the first backward bucket
    reuses the parameters the last forward bucket gathered, so its re-gather
    (PACK_AG, AG, WAIT_AG, UNPACK of bucket 0) is left out of the sequence;
    everything else is unchanged."""
    s = _backward_sequence(k, reorder, placement)
    if keep_first:
        s = [e for e in s if not (e[2] == 0 and e[1] in (PACK_AG, AG, WAIT_AG, UNPACK))]
    return s


def _backward_sequence(k, reorder, placement):
    s = []
    if not reorder:
        for b in range(k):
            s += [_e(1, PACK_AG, b), _e(1, AG, b), _e(1, WAIT_AG, b), _e(1, UNPACK, b),
                  _e(1, COMPUTE_B, b), _e(1, PACK_RS, b), _e(1, RS, b), _e(1, WAIT_RS, b),
                  _e(1, COPYOUT_RS, b)]
        return s
    if k:
        s += [_e(1, PACK_AG, 0), _e(1, AG, 0)]
    for b in range(k):
        pre = [_e(1, PACK_AG, b + 1), _e(1, AG, b + 1)] if b + 1 < k else []
        wait = [_e(1, WAIT_AG, b), _e(1, UNPACK, b)]
        s += (pre + wait) if placement == BEFORE else (wait + pre)
        s += [_e(1, COMPUTE_B, b), _e(1, PACK_RS, b)]
        if b >= 1:
            s += [_e(1, WAIT_RS, b - 1), _e(1, COPYOUT_RS, b - 1)]
        s.append(_e(1, RS, b))
    if k:
        s += [_e(1, WAIT_RS, k - 1), _e(1, COPYOUT_RS, k - 1)]
    return s


def step_sequence(k_fwd, k_bwd, reorder=True, fwd_placement=BEFORE, bwd_placement=AFTER, keep_first=False):
    return (forward_sequence(k_fwd, reorder, fwd_placement)
            + backward_sequence(k_bwd, reorder, bwd_placement, keep_first and k_fwd > 0))


def dependencies_respected(seq):
    """Linear-extension check of the data dependencies of O9:
    AG after its PACK_AG, WAIT_AG after its AG, UNPACK after its WAIT_AG,
    COMPUTE after its UNPACK, PACK_RS after its COMPUTE_B, RS after its
    PACK_RS, WAIT_RS after its RS, COPYOUT_RS after its WAIT_RS; every op
    appears exactly once.  A backward bucket 0 without its re-gather (G42)
    computes on the last forward bucket's parameters: after its COMPUTE_F."""
    pos = {}
    for i, (ph, op, b, _) in enumerate(seq):
        key = (ph, op, b)
        if key in pos:
            return False
        pos[key] = i
    need = {AG: PACK_AG, WAIT_AG: AG, UNPACK: WAIT_AG, COMPUTE_F: UNPACK, COMPUTE_B: UNPACK,
            PACK_RS: COMPUTE_B, RS: PACK_RS, WAIT_RS: RS, COPYOUT_RS: WAIT_RS}
    last_f = max([b for (ph, op, b) in pos if ph == 0 and op == COMPUTE_F], default=None)
    for (ph, op, b), i in pos.items():
        if op in need:
            dep = (ph, need[op], b)
            if (ph, op, b) == (1, COMPUTE_B, 0) and dep not in pos and last_f is not None:
                dep = (0, COMPUTE_F, last_f)      # kept from the forward (G42)
            j = pos.get(dep)
            if j is None or j > i:
                return False
    return True
