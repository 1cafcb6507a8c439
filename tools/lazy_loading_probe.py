"""Probe: a spinning fsdp_p2p_wait on stream A must not block an fsdp_p2p_signal on stream B.

Failed (3 s timeout) before the library preloaded its kernels: under CUDA lazy
loading the first launch of the signal kernel waited for the spinning kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("CUDA_DEVICE_MAX_CONNECTIONS =", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"))
import torch
import paper_2411_00284_b200 as F
ctx = F.Ctx(1, 0)
flag = torch.zeros(1, dtype=torch.int64, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
nstreams = int(sys.argv[1]) if len(sys.argv) > 1 else 2
streams = [torch.cuda.Stream() for _ in range(nstreams)]
torch.cuda.synchronize()
t = time.time()
F.p2p_wait(ctx, flag.data_ptr(), 1, 3 * 10**9, err.data_ptr(), streams[0].cuda_stream)
F.p2p_signal(ctx, [flag.data_ptr()], 1, streams[-1].cuda_stream)
torch.cuda.synchronize()
print("streams", nstreams, "err", int(err.item()), "secs %.3f" % (time.time() - t))
