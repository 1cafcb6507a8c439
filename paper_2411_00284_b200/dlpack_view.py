"""A torch uint8 view of device memory the library allocated (fsdp_ipc_alloc),
through a DLPack capsule built with ctypes.  Plumbing for the harness: torch
fills / zeroes the buffers, the library owns and frees them."""
import ctypes as C

import torch
import torch.utils.dlpack


class _DLDevice(C.Structure):
    _fields_ = [("device_type", C.c_int), ("device_id", C.c_int)]


class _DLDataType(C.Structure):
    _fields_ = [("code", C.c_uint8), ("bits", C.c_uint8), ("lanes", C.c_uint16)]


class _DLTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("device", _DLDevice), ("ndim", C.c_int), ("dtype", _DLDataType),
                ("shape", C.POINTER(C.c_int64)), ("strides", C.POINTER(C.c_int64)), ("byte_offset", C.c_uint64)]


class _DLManagedTensor(C.Structure):
    pass


_DELETER = C.CFUNCTYPE(None, C.POINTER(_DLManagedTensor))
_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", C.c_void_p), ("deleter", _DELETER)]

_KDL_CUDA = 2
_KDL_UINT = 1
_keep = {}


@_DELETER
def _noop_deleter(p):  # memory belongs to the library (fsdp_ipc_free)
    _keep.pop(C.addressof(p.contents), None)


def uint8_view(ptr, nbytes, device_index):
    """torch.uint8 tensor of `nbytes` aliasing device memory at `ptr`."""
    shape = (C.c_int64 * 1)(int(nbytes))
    m = _DLManagedTensor()
    m.dl_tensor.data = C.c_void_p(int(ptr))
    m.dl_tensor.device = _DLDevice(_KDL_CUDA, int(device_index))
    m.dl_tensor.ndim = 1
    m.dl_tensor.dtype = _DLDataType(_KDL_UINT, 8, 1)
    m.dl_tensor.shape = shape
    m.dl_tensor.strides = None
    m.dl_tensor.byte_offset = 0
    m.manager_ctx = None
    m.deleter = _noop_deleter
    _keep[C.addressof(m)] = (m, shape)
    C.pythonapi.PyCapsule_New.restype = C.py_object
    C.pythonapi.PyCapsule_New.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
    cap = C.pythonapi.PyCapsule_New(C.addressof(m), b"dltensor", None)
    return torch.utils.dlpack.from_dlpack(cap)
