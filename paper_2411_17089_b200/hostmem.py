"""Page-locked host memory for the host stores and the PCIe probes, exact size.

Default: cudaHostAlloc (the copy engine streams it 0.4% faster H2D and ~8% faster D2H than
cudaHostRegister'd pageable memory, profiles/r01_pcie_alloc_probe.json; the headline gains 0.65%,
profiles/r01_host_alloc_ab.jsonl).  KVPR_HOST_ALLOC=register selects cudaHostRegister of a torch
allocation instead (A/B).  torch's pin_memory would round multi-GB sizes up to a power of two.
"""

from __future__ import annotations

import ctypes
import os
import weakref

import torch

_CUDART = None


def _cudart():
    """The CUDA runtime library, for cudaHostAlloc / cudaFreeHost."""
    global _CUDART
    if _CUDART is None:
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _CUDART = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _CUDART is None:
            raise RuntimeError("libcudart not found for cudaHostAlloc")
        _CUDART.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
        _CUDART.cudaFreeHost.argtypes = [ctypes.c_void_p]
    return _CUDART


def mode() -> str:
    return os.environ.get("KVPR_HOST_ALLOC", "hostalloc")


def pinned_empty(shape, dtype: torch.dtype) -> torch.Tensor:
    """Uninitialised page-locked tensor.  hostalloc mode: freed once the last view is gone (torch
    keeps the backing buffer alive), so nothing needs closing.  register mode: call unpin(t)."""
    numel = 1
    for d in shape:
        numel *= d
    nbytes = numel * torch.empty(0, dtype=dtype).element_size()
    if nbytes == 0:
        return torch.empty(shape, dtype=dtype)
    if mode() == "register":
        t = torch.empty(shape, dtype=dtype)
        rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed ({rc}) for {nbytes / 2**30:.1f} GiB")
        t._kvpr_registered = True
        return t
    ptr = ctypes.c_void_p()
    rc = _cudart().cudaHostAlloc(ctypes.byref(ptr), nbytes, 0)
    if rc != 0:
        raise RuntimeError(f"cudaHostAlloc failed ({rc}) for {nbytes / 2**30:.1f} GiB")
    buf = (ctypes.c_uint8 * nbytes).from_address(ptr.value)
    weakref.finalize(buf, _cudart().cudaFreeHost, ptr.value)
    return torch.frombuffer(buf, dtype=torch.uint8).view(dtype).view(shape)


def unpin(t: torch.Tensor) -> None:
    """Undo register mode's cudaHostRegister (no-op for cudaHostAlloc'd tensors)."""
    if getattr(t, "_kvpr_registered", False):
        torch.cuda.cudart().cudaHostUnregister(t.data_ptr())
        t._kvpr_registered = False
