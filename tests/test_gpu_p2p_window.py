"""-m gpu: the peer-memory path over NCCL symmetric windows (the NCCL 2.28
device API) instead of CUDA IPC handles, at world 1 with
a real communicator: the window's peer table is this rank's own buffer, the
FSDP_SCHED_P2P step (K8 / K9 and the epoch flags through the window
pointers) leaves the same bytes as with IPC-mapped buffers, and the window's
NVLS multicast address either works as K10's staging or is reported
unsupported; bench.py's N > 1 code path runs with --p2p-transport window."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

import paper_2411_00284_b200 as F
from paper_2411_00284_b200 import _lib as L
from paper_2411_00284_b200 import harness as H
from workloads import llama

pytestmark = pytest.mark.gpu

FLAGS = L.SCHED_REORDER | L.SCHED_FWD_AG_BEFORE_WAIT | L.SCHED_P2P


def _assert_alias(ptr, t, write=False):
    """`ptr` maps the same memory as tensor `t` (NCCL's flat window VA of this
    rank aliases the registered buffer)."""
    from paper_2411_00284_b200.dlpack_view import uint8_view
    v = uint8_view(ptr, t.numel(), torch.cuda.current_device())
    if write:
        t[:4096].copy_(torch.arange(4096, device=t.device).to(torch.uint8))
    torch.cuda.synchronize()
    assert torch.count_nonzero(t[:4096]) > 0 and torch.equal(v[:4096], t[:4096])


def _step(windows):
    specs = llama("8b", n_layers=2)
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    fplan, bplan = H.plans_for(specs, 1, L.PLAN_MANUAL)
    st = H.RankState(specs, 1, 0, fplan, bplan, ctx, seed=31, ipc=not windows, windows=windows)
    if windows:
        st.setup_p2p_windows()
        _assert_alias(F.window_peer_pointers(ctx, st.shard_buf.data_ptr())[0], st.shard_buf)
    else:
        st.setup_p2p_ipc(lambda o: [o])
    for t in st.full_slots:
        t.zero_()
    cs, ms = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    for _ in range(2):
        st.step(FLAGS, cs.cuda_stream, ms.cuda_stream)
    torch.cuda.synchronize()
    st.check_p2p()
    out = ([t.clone() for t in st.full_slots], st.gshard_buf.clone())
    st.close_ipc()
    st.close_nccl_mem()
    del st
    ctx.close()
    return out


def test_window_transport_matches_ipc():
    a, b = _step(False), _step(True)
    for x, y in zip(a[0], b[0]):
        assert torch.equal(x, y)
    assert torch.equal(a[1], b[1])


def test_window_multimem_pointer_or_unsupported():
    ctx = F.Ctx(1, 0, 0, nccl_uid=F.nccl_get_unique_id())
    ptr = F.mem_alloc(ctx, 1 << 20)
    F.register_buffer(ctx, ptr, 1 << 20, L.REG_SYMMETRIC)
    with pytest.raises(L.FsdpError):
        F.window_peer_pointers(ctx, ptr + 4096)          # not a window base
    from paper_2411_00284_b200.dlpack_view import uint8_view
    _assert_alias(F.window_peer_pointers(ctx, ptr)[0], uint8_view(ptr, 1 << 20, torch.cuda.current_device()),
                  write=True)
    try:
        mc = F.window_multimem_pointer(ctx, ptr)
        assert mc and mc % 16 == 0
    except L.FsdpError as e:
        assert e.status == L.FSDP_ERR_UNSUPPORTED, e
    F.mem_free(ctx, ptr)
    ctx.close()


def test_bench_window_transport_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", "1", "--dist", "--collective", "p2p", "--p2p-transport", "window", "--layers", "2",
           "--steps", "2", "--warmup", "3", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["parity"]["ok"] and line["p2p_wait_timeouts"] == 0
