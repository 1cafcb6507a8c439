"""O10 -- two-stream discrete-event simulator (test infrastructure; see
oracle/__init__.py).

P:184: collectives "are asynchronous, allowing [them] to occur concurrently with
the computation on different CUDA streams".  Semantics as S:405-413 / S:441-443,
in integer nanoseconds:
  * the compute stream runs its ops (packs, copy-outs, computes) in order;
  * the comm stream is FIFO; a collective starts when it is at the head of the
    comm stream and its pack has finished;
  * a WAIT blocks the compute stream until its collective has finished;
  * exposed = total blocked time = total - sum(compute-stream durations).
"""
from .schedule import AG, RS, WAIT_AG, WAIT_RS, PACK_AG, PACK_RS


def simulate(seq, dur, t_coll):
    """seq: O9 entries (phase, op, bucket, stream) in enqueue order.
    dur(phase, op, bucket) -> ns for compute-stream ops (WAITs excluded).
    t_coll(phase, op, bucket) -> ns for AG / RS.
    Returns dict(total, exposed, compute_busy, comm_busy, events)."""
    t_cmp = 0
    t_comm = 0
    pack_end = {}
    coll_end = {}
    busy = 0
    comm_busy = 0
    exposed = 0
    events = []
    for ph, op, b, stream in seq:
        if op in (AG, RS):
            pk = PACK_AG if op == AG else PACK_RS
            start = max(t_comm, pack_end[(ph, pk, b)])
            d = t_coll(ph, op, b)
            t_comm = start + d
            coll_end[(ph, op, b)] = t_comm
            comm_busy += d
            events.append((ph, op, b, 1, start, t_comm))
        elif op in (WAIT_AG, WAIT_RS):
            c = coll_end[(ph, AG if op == WAIT_AG else RS, b)]
            if c > t_cmp:
                exposed += c - t_cmp
                events.append((ph, op, b, 0, t_cmp, c))
                t_cmp = c
        else:
            d = dur(ph, op, b)
            start = t_cmp
            t_cmp += d
            busy += d
            if op in (PACK_AG, PACK_RS):
                pack_end[(ph, op, b)] = t_cmp
            events.append((ph, op, b, 0, start, t_cmp))
    total = max(t_cmp, t_comm)
    return dict(total=total, exposed=exposed, compute_busy=busy, comm_busy=comm_busy,
                events=events)


# --------------------------------------------------------------- memory curve
# Memory is the paper's other metric (Table 5 and Table 6 report peak
# GiB).  Reading G40: the FSDP buffers of a step live like tensors of an
# allocate-on-produce / free-after-last-use allocator, walked in the
# sequence's (stream) order:
#   PACK_AG (ph, b)  allocates the flat gathered buffer  A(ph, b) (P:177 copy-in);
#   UNPACK  (ph, b)  allocates the full parameters        F(ph, b) (P:177 copy-out),
#                    then frees A(ph, b);
#   COMPUTE_F b      frees F(0, b) afterwards: released after forward use;
#   COMPUTE_B b      allocates the full gradients         G(b), then frees F(1, b);
#   PACK_RS b        allocates the flat RS input          R(b) (P:179 copy-in),
#                    then frees G(b);
#   COPYOUT_RS b     frees R(b) (the gradient shard it fills is resident);
#   AG, RS, WAIT_*   allocate nothing (in-place collectives).
# A backward bucket 0 without UNPACK reuses the last forward bucket's gathered
# parameters (G42): that bucket's COMPUTE_F then frees nothing, and COMPUTE_B 0
# frees them.
# The peak is taken after every allocation, before that op's frees.  Resident
# shards / gradient shards and activations are outside the curve.
from .schedule import UNPACK, COMPUTE_F, COMPUTE_B, COPYOUT_RS  # noqa: E402


def memory_curve(seq, A, Fp, G, R):
    """seq: O9 entries (phase, op, bucket, stream).  A(ph, b), Fp(ph, b): flat
    gathered and full-parameter bytes of bucket b of phase ph; G(b), R(b): full
    gradient and flat RS-input bytes of backward bucket b.
    Returns dict(peak, live (after each entry), final)."""
    live = 0
    peak = 0
    after = []
    ops = {(e[0], e[1], e[2]) for e in seq}
    keep = (1, COMPUTE_B, 0) in ops and (1, UNPACK, 0) not in ops
    last_f = max([e[2] for e in seq if e[0] == 0 and e[1] == COMPUTE_F], default=None)
    for ph, op, b, _stream in seq:
        if op == PACK_AG:
            live += A(ph, b)
            peak = max(peak, live)
        elif op == UNPACK:
            live += Fp(ph, b)
            peak = max(peak, live)
            live -= A(ph, b)
        elif op == COMPUTE_F:
            if not (keep and b == last_f):
                live -= Fp(ph, b)
        elif op == COMPUTE_B:
            live += G(b)
            peak = max(peak, live)
            live -= Fp(ph, b)
        elif op == PACK_RS:
            live += R(b)
            peak = max(peak, live)
            live -= G(b)
        elif op == COPYOUT_RS:
            live -= R(b)
        after.append(live)
    return dict(peak=peak, live=after, final=live)
