"""O3 -- flat bucket layout (test infrastructure; see oracle/__init__.py).

P:177 (AG bucketing): "allocate a bigger buffer that flattens and concatenates
the tensor from each individual all-gather".
P:179 (RS bucketing): "splits the obtained gradient into chunks based on world
size and concatenates the gradients from the individual reduce-scatter".

Per rank the bucket holds one *segment*: the member shards (c_j x R_j elements
of e bytes each) concatenated in forward order, each member starting at a byte
offset aligned to A (reading G4: A = 16 default, A = 1 gives tight packing),
the segment itself padded to A.  The collective buffer is N segments
back-to-back, segment q being rank q's.

    off_1 = 0,  off_{k+1} = align_A(off_k + c_k R_k e),  seg = align_A(off_K + c_K R_K e)
"""


def align_up(x, a):
    return -(-x // a) * a


def bucket_layout(members, world, elem_bytes, align=16):
    """members: list of (d_j, R_j).  Returns (offsets_bytes, seg_bytes)."""
    if align < 1:
        raise ValueError("align must be >= 1")
    offs = []
    cur = 0
    for d, r in members:
        c = -(-d // world)
        offs.append(cur)
        cur = align_up(cur + c * r * elem_bytes, align)
    return offs, cur
