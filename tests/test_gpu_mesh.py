"""-m gpu parity of the 2-D DP x TP composition: FSDP over the DP
sub-mesh of TP-local tensors, bit-exact against oracle.mesh; and
fsdp_ctx_split (ncclCommSplit) at world 1 with a real communicator."""
import numpy as np
import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from oracle import mesh as OM
from workloads import llama
from workloads.data import grad_tensor, param_tensor
from workloads.shapes import tp_axis

from .test_gpu_parity import sim_allgather, sim_reduce_scatter

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dp,tp", [(4, 2), (2, 4), (3, 2)])
def test_dp_tp_block_bucket(dp, tp):
    """One Llama-3-8B block: every TP index's DP all-gather rebuilds its TP
    blocks and its DP reduce-scatter averages TP-local gradients, bit-exact."""
    specs = llama("8b", n_layers=1, with_embeddings=False)
    axes = [tp_axis(p) for p in specs]
    params = [param_tensor(p, "bf16", 500 + i) for i, p in enumerate(specs)]
    for t in range(tp):
        blocks = [OM.tp_slice(p, tp, t, a) for p, a in zip(params, axes)]
        # the kernels see the TP-local tensors as their "full" parameters
        assert sim_allgather(blocks, dp, L.BF16, check_all_ranks=False)
        _, fulls = OM.dp_all_gather(params, axes, dp, tp, t)
        assert all(np.array_equal(a, b) for a, b in zip(fulls, blocks))
    # reduce-scatter on a reduced-width copy of the block (row_numel / 64) to keep it quick
    small = [p._replace(row_numel=max(1, p.row_numel // 64) * (tp if tp_axis(p) == 1 else 1)) for p in specs]
    grads = [[grad_tensor(p, "bf16", 9, r) for p in small] for r in range(dp)]
    saxes = [tp_axis(p) for p in small]
    for t in range(tp):
        local = [[OM.tp_slice(g, tp, t, a) for g, a in zip(gs, saxes)] for gs in grads]
        assert sim_reduce_scatter(local, dp, L.BF16)


def test_ctx_split_world1():
    """fsdp_ctx_split at world 1: the sub-mesh ctx owns its communicator and
    runs the bucket collectives (NCCL world-1 AG / RS) bit-exactly."""
    parent = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    sub = parent.split(0, 0)
    assert sub.world == 1 and sub.rank == 0
    assert parent.split(-1, 0) is None           # NCCL_SPLIT_NOCOLOR
    d, R = 64, 32
    p = np.random.Generator(np.random.Philox(1)).integers(0, 65536, size=(d, R)).astype(np.uint16)
    sh = torch.from_numpy(p.copy()).cuda()
    full = torch.zeros_like(sh)
    nsh = torch.ones(5, dtype=torch.int16, device="cuda")    # a 1-D member (kept alive)
    nfull = torch.zeros(5, dtype=torch.int16, device="cuda")
    b = F.Bucket(sub, [(d, R, 0), (5, 1, 0)], shards=[sh.data_ptr(), nsh.data_ptr()],
                 fulls=[full.data_ptr(), nfull.data_ptr()])
    st = torch.zeros(b.ag_seg, dtype=torch.uint8, device="cuda")
    F.allgather_bucket(sub, b, st.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(full.cpu().numpy(), p) and torch.equal(nfull, nsh)
    b.close()
    sub.close()
    parent.close()
    with pytest.raises(RuntimeError):
        F.Ctx(2, 0).split(0, 0)                 # layout-only parent: no communicator
