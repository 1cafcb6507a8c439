import sys
sys.path.insert(0, '.')
import torch
import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
ptr = F.mem_alloc(ctx, 1 << 21)
F.register_buffer(ctx, ptr, 1 << 21, L.REG_SYMMETRIC)
try:
    mc = F.window_multimem_pointer(ctx, ptr)
    print("MULTIMEM OK", hex(mc))
except L.FsdpError as e:
    print("MULTIMEM FAIL", e.status, e)
F.mem_free(ctx, ptr)
ctx.close()
