"""Helpers for the -m gpu tests: device buffers from host arrays and back.
Plumbing only (torch allocates, copies); all method work goes through the C ABI."""
import numpy as np
import torch

ALIGN = 256


def dev_bytes(nbytes, fill=None):
    t = torch.empty(max(int(nbytes), 1) + ALIGN, dtype=torch.uint8, device="cuda")
    if fill is not None:
        t.fill_(fill)
    off = (-t.data_ptr()) % ALIGN
    return t, t.data_ptr() + off, off


class DevArray:
    """A host NumPy array mirrored in an aligned device buffer."""

    def __init__(self, host=None, nbytes=None, fill=None, dtype=None, shape=None):
        if host is not None:
            host = np.ascontiguousarray(host)
            nbytes, dtype, shape = host.nbytes, host.dtype, host.shape
        self.nbytes, self.dtype, self.shape = int(nbytes), np.dtype(dtype) if dtype is not None else np.uint8, shape
        self.t, self.ptr, self.off = dev_bytes(self.nbytes, fill)
        if host is not None and self.nbytes:
            src = torch.from_numpy(host.reshape(-1).view(np.uint8).copy())
            self.t[self.off:self.off + self.nbytes].copy_(src)

    def get(self):
        torch.cuda.synchronize()
        b = self.t[self.off:self.off + self.nbytes].cpu().numpy()
        a = b.view(self.dtype)
        return a.reshape(self.shape) if self.shape is not None else a


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype.itemsize == 2 else a.view(np.uint32)


def bf16_ulp_distance(a, b):
    """Element-wise distance in bf16 units in the last place between two bf16
    bit-pattern arrays (uint16): the patterns mapped to a monotone integer
    order (+0 and -0 both 0, negatives below), then |ord(a) - ord(b)|.  The
    north star's tolerance for gradients cast to bf16 after the fp32 RS."""
    def order(u):
        u = np.asarray(u, dtype=np.uint16).astype(np.int64)
        return np.where(u < 0x8000, u, 0x8000 - u)
    return np.abs(order(a) - order(b))
