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
