"""Thin Python binding of libkrp.so (include/krp.h) — argument marshalling only.

Every computation runs in the library's sm_100a kernels.  torch is used for
device memory, streams and (for the sharded calls) process groups.  There is no
CPU or eager fallback: if libkrp.so is missing or a call fails, an exception is
raised.

Names mirror the C ABI.  Tensors follow the ABI layouts:
  X       fp32, flat (or any shape) first-index-fastest buffer of prod(dims) elements
  omega_k fp32 (I_k, R) row-major;  Y_n (I_n, R);  Q_n (I_n, r_n);  core flat prod(r_n).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
from typing import List, Optional, Sequence, Tuple

import torch

__all__ = [
    "krp_profile_enable", "krp_profile_read", "krp_profile_reset",
    "lib", "KrpError", "OP_SKETCH_ALL", "OP_SKETCH_MODE", "OP_RHOSVD", "OP_STHOSVD", "OP_SKETCH_ALL_HOST",
    "OP_RHOSVD_ERR", "krp_workspace_bytes",
    "krp_sketch_all_modes", "krp_sketch_all_modes_host", "krp_sketch_mode", "krp_rhosvd", "krp_sthosvd",
    "krp_launch_count", "krp_reset_launch_count", "Comm", "krp_sketch_all_modes_dist", "krp_rhosvd_dist",
    "krp_sthosvd_dist", "krp_rhosvd_fresh", "krp_rhosvd_gaussian", "krp_sthosvd_gaussian", "OP_RHOSVD_FRESH",
    "OP_RHOSVD_GAUSSIAN", "OP_STHOSVD_GAUSSIAN", "krp_hadamard_tucker", "krp_ttm", "OP_TTM",
    "krp_workspace_bytes_dist", "EXPORTED_SYMBOLS", "LIB_PATH", "krp_slab_range", "krp_pack_layout",
]

LIB_PATH = os.environ.get("KRP_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libkrp.so")
(OP_SKETCH_ALL, OP_SKETCH_MODE, OP_RHOSVD, OP_STHOSVD, OP_SKETCH_ALL_HOST, OP_RHOSVD_ERR, OP_RHOSVD_FRESH,
 OP_RHOSVD_GAUSSIAN, OP_STHOSVD_GAUSSIAN, OP_TTM) = range(10)

# every function declared in include/krp.h
EXPORTED_SYMBOLS = [
    "krp_status_string", "krp_last_error_message", "krp_version", "krp_workspace_bytes",
    "krp_sketch_all_modes", "krp_sketch_all_modes_host", "krp_sketch_mode", "krp_rhosvd", "krp_sthosvd",
    "krp_comm_id_bytes", "krp_comm_get_unique_id", "krp_comm_init", "krp_comm_destroy",
    "krp_sketch_all_modes_dist", "krp_rhosvd_dist", "krp_sthosvd_dist", "krp_workspace_bytes_dist", "krp_launch_count",
    "krp_reset_launch_count", "krp_profile_enable", "krp_profile_read", "krp_profile_reset",
    "krp_slab_range", "krp_pack_layout", "krp_rhosvd_fresh", "krp_rhosvd_gaussian", "krp_sthosvd_gaussian",
    "krp_hadamard_workspace_bytes", "krp_hadamard_tucker", "krp_ttm",
]

_lib = None
_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_IP = ctypes.POINTER(ctypes.c_int)


class KrpError(RuntimeError):
    def __init__(self, status: int, where: str):
        l_ = lib()
        msg = l_.krp_status_string(status).decode()
        detail = l_.krp_last_error_message().decode()
        super().__init__(f"{where}: {msg} ({status}): {detail}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libkrp.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2507_23207_b200.build` "
                              "(or __graft_entry__.build()) first")
        l_ = ctypes.CDLL(LIB_PATH)
        l_.krp_status_string.restype = ctypes.c_char_p
        l_.krp_status_string.argtypes = [ctypes.c_int]
        l_.krp_last_error_message.restype = ctypes.c_char_p
        l_.krp_version.restype = ctypes.c_int
        l_.krp_workspace_bytes.restype = ctypes.c_size_t
        l_.krp_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, _I64P, ctypes.c_int, _IP]
        l_.krp_workspace_bytes_dist.restype = ctypes.c_size_t
        l_.krp_workspace_bytes_dist.argtypes = [ctypes.c_int, ctypes.c_int, _I64P, ctypes.c_int64, ctypes.c_int, _IP]
        ptrs = ctypes.POINTER(ctypes.c_void_p)
        l_.krp_sketch_all_modes.argtypes = [_P, ctypes.c_int, _I64P, ptrs, ctypes.c_int, ptrs, _P, ctypes.c_size_t, _P]
        l_.krp_sketch_all_modes_host.argtypes = l_.krp_sketch_all_modes.argtypes
        l_.krp_sketch_mode.argtypes = [_P, ctypes.c_int, _I64P, ctypes.c_int, ptrs, ctypes.c_int, _P, _P,
                                       ctypes.c_size_t, _P]
        l_.krp_ttm.argtypes = [_P, ctypes.c_int, _I64P, ctypes.c_int, _P, ctypes.c_int, _P, _P, ctypes.c_size_t, _P]
        l_.krp_rhosvd.argtypes = [_P, ctypes.c_int, _I64P, _IP, ctypes.c_int, ptrs, ptrs, _P,
                                  ctypes.POINTER(ctypes.c_double), _P, ctypes.c_size_t, _P]
        l_.krp_sthosvd.argtypes = l_.krp_rhosvd.argtypes
        l_.krp_rhosvd_fresh.argtypes = l_.krp_rhosvd.argtypes
        l_.krp_hadamard_workspace_bytes.restype = ctypes.c_size_t
        l_.krp_hadamard_workspace_bytes.argtypes = [_I64P, _I64P, _I64P, _IP, _IP]
        l_.krp_hadamard_tucker.argtypes = [_P, _I64P, ptrs, _P, _I64P, ptrs, _I64P, _IP, _IP, ptrs, ptrs, _P, _P,
                                           ctypes.c_size_t, _P]
        l_.krp_rhosvd_gaussian.argtypes = l_.krp_rhosvd.argtypes
        l_.krp_sthosvd_gaussian.argtypes = l_.krp_rhosvd.argtypes
        l_.krp_comm_id_bytes.restype = ctypes.c_size_t
        l_.krp_comm_get_unique_id.argtypes = [_P]
        l_.krp_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, _P]
        l_.krp_comm_destroy.argtypes = [_P]
        l_.krp_sketch_all_modes_dist.argtypes = [_P, ctypes.c_int, _I64P, ctypes.c_int64, ctypes.c_int64, ptrs,
                                                 ctypes.c_int, ptrs, _P, ctypes.c_size_t, _P, _P]
        l_.krp_rhosvd_dist.argtypes = [_P, ctypes.c_int, _I64P, ctypes.c_int64, ctypes.c_int64, _IP, ctypes.c_int,
                                       ptrs, ptrs, _P, ctypes.POINTER(ctypes.c_double), _P, ctypes.c_size_t, _P, _P]
        l_.krp_sthosvd_dist.argtypes = l_.krp_rhosvd_dist.argtypes
        l_.krp_slab_range.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _I64P, _I64P]
        l_.krp_pack_layout.argtypes = [ctypes.c_int, _I64P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _I64P, _I64P]
        l_.krp_launch_count.restype = ctypes.c_uint64
        l_.krp_profile_enable.argtypes = [ctypes.c_int]
        l_.krp_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        _lib = l_
    return _lib


# ------------------------------------------------------------------ marshalling helpers
def _dims(dims: Sequence[int]):
    return (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])


def _ints(v: Sequence[int]):
    return (ctypes.c_int * len(v))(*[int(x) for x in v])


def _ptr_array(tensors):
    return (ctypes.c_void_p * len(tensors))(*[None if t is None else t.data_ptr() for t in tensors])


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(status: int, where: str):
    if status != 0:
        raise KrpError(status, where)


def _dev_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA float32 tensor")
    return t


def _ws(nbytes: int, device, ws: Optional[torch.Tensor]):
    if ws is not None:
        if ws.numel() * ws.element_size() < nbytes:
            raise ValueError("workspace tensor too small")
        return ws
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def krp_workspace_bytes(op: int, dims: Sequence[int], R: int, ranks: Optional[Sequence[int]] = None) -> int:
    return int(lib().krp_workspace_bytes(op, len(dims), _dims(dims), int(R), _ints(ranks) if ranks else None))


def krp_workspace_bytes_dist(op: int, dims_local: Sequence[int], I_d_global: int, R: int,
                             ranks: Optional[Sequence[int]] = None) -> int:
    return int(lib().krp_workspace_bytes_dist(op, len(dims_local), _dims(dims_local), int(I_d_global), int(R),
                                              _ints(ranks) if ranks else None))


def krp_launch_count() -> int:
    return int(lib().krp_launch_count())


def krp_reset_launch_count() -> None:
    lib().krp_reset_launch_count()


def krp_profile_enable(on: bool = True) -> None:
    _check(lib().krp_profile_enable(1 if on else 0), "krp_profile_enable")


def krp_profile_reset() -> None:
    lib().krp_profile_reset()


def krp_profile_read():
    """(kernel_ms total, launches, algorithmic bytes, algorithmic flops) of the dominant sketch kernel."""
    ms, n, b, f = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double(), ctypes.c_double()
    _check(lib().krp_profile_read(ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b), ctypes.byref(f)),
           "krp_profile_read")
    return ms.value, int(n.value), b.value, f.value


# ------------------------------------------------------------------ entry points
def krp_sketch_all_modes(X: torch.Tensor, dims: Sequence[int], omegas: Sequence[torch.Tensor],
                         Y: Optional[List[torch.Tensor]] = None, ws: Optional[torch.Tensor] = None,
                         stream=None) -> List[torch.Tensor]:
    """Y_n = X_(n)(Ω_d ⊙..⊙Ω_{n+1}⊙Ω_{n-1}⊙..⊙Ω_1) for every n (memoized)."""
    _dev_f32(X, "X")
    R = int(omegas[0].shape[1])
    for k, o in enumerate(omegas):
        _dev_f32(o, f"omega[{k}]")
    if Y is None:
        Y = [torch.empty((int(n), R), dtype=torch.float32, device=X.device) for n in dims]
    w = _ws(krp_workspace_bytes(OP_SKETCH_ALL, dims, R), X.device, ws)
    _check(lib().krp_sketch_all_modes(X.data_ptr(), len(dims), _dims(dims), _ptr_array(omegas), R, _ptr_array(Y),
                                      w.data_ptr(), w.numel(), _stream(stream)), "krp_sketch_all_modes")
    return Y


def krp_sketch_all_modes_host(X: torch.Tensor, dims: Sequence[int], omegas: Sequence[torch.Tensor],
                              Y: Optional[List[torch.Tensor]] = None, ws: Optional[torch.Tensor] = None,
                              stream=None, device=None) -> List[torch.Tensor]:
    """Host-buffer variant: X, omegas, Y are CPU tensors (pin them for full speed)."""
    R = int(omegas[0].shape[1])
    if Y is None:
        Y = [torch.empty((int(n), R), dtype=torch.float32, pin_memory=X.is_pinned()) for n in dims]
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    w = _ws(krp_workspace_bytes(OP_SKETCH_ALL_HOST, dims, R), dev, ws)
    _check(lib().krp_sketch_all_modes_host(X.data_ptr(), len(dims), _dims(dims), _ptr_array(omegas), R,
                                           _ptr_array(Y), w.data_ptr(), w.numel(), _stream(stream)),
           "krp_sketch_all_modes_host")
    return Y


def krp_sketch_mode(X: torch.Tensor, dims: Sequence[int], n: int, omegas: Sequence[Optional[torch.Tensor]],
                    Y: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Y = X_(n)(⊙_{k≠n} Ω_k); omegas[n] may be None."""
    _dev_f32(X, "X")
    R = int(next(o for k, o in enumerate(omegas) if k != n).shape[1])
    if Y is None:
        Y = torch.empty((int(dims[n]), R), dtype=torch.float32, device=X.device)
    w = _ws(krp_workspace_bytes(OP_SKETCH_MODE, dims, R), X.device, ws)
    _check(lib().krp_sketch_mode(X.data_ptr(), len(dims), _dims(dims), int(n), _ptr_array(omegas), R, Y.data_ptr(),
                                 w.data_ptr(), w.numel(), _stream(stream)), "krp_sketch_mode")
    return Y


def krp_ttm(X: torch.Tensor, dims: Sequence[int], n: int, A: torch.Tensor, Y: Optional[torch.Tensor] = None,
            ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Y = X x_n A; A: J x I_n fp32 row-major on the device; Y flat, dims with I_n -> J."""
    _dev_f32(X, "X")
    _dev_f32(A, "A")
    J = int(A.shape[0])
    if Y is None:
        Y = torch.empty(X.numel() // int(dims[n]) * J, dtype=torch.float32, device=X.device)
    w = _ws(krp_workspace_bytes(OP_TTM, dims, J), X.device, ws)
    _check(lib().krp_ttm(X.data_ptr(), len(dims), _dims(dims), int(n), A.data_ptr(), J, Y.data_ptr(), w.data_ptr(),
                         w.numel(), _stream(stream)), "krp_ttm")
    return Y


def krp_rhosvd(X: torch.Tensor, dims: Sequence[int], ranks: Sequence[int], omegas: Sequence[torch.Tensor],
               with_error: bool = False, ws: Optional[torch.Tensor] = None, stream=None
               ) -> Tuple[List[torch.Tensor], torch.Tensor, Optional[float]]:
    """RHOSVD-KRP-MEMO (Alg. 7 + memoization) with core truncation; returns (Q list, core, rel_err)."""
    _dev_f32(X, "X")
    R = int(omegas[0].shape[1])
    Q = [torch.empty((int(n), int(r)), dtype=torch.float32, device=X.device) for n, r in zip(dims, ranks)]
    core = torch.empty(int(torch.tensor(list(ranks)).prod()), dtype=torch.float32, device=X.device)
    err = ctypes.c_double(0.0)
    op = OP_RHOSVD_ERR if with_error else OP_RHOSVD
    w = _ws(krp_workspace_bytes(op, dims, R, ranks), X.device, ws)
    _check(lib().krp_rhosvd(X.data_ptr(), len(dims), _dims(dims), _ints(ranks), R, _ptr_array(omegas), _ptr_array(Q),
                            core.data_ptr(), ctypes.byref(err) if with_error else None, w.data_ptr(), w.numel(),
                            _stream(stream)), "krp_rhosvd")
    return Q, core, (err.value if with_error else None)


def krp_sthosvd(X: torch.Tensor, dims: Sequence[int], ranks: Sequence[int],
                omegas: Sequence[Sequence[Optional[torch.Tensor]]], with_error: bool = False,
                ws: Optional[torch.Tensor] = None, stream=None):
    """RSTHOSVD-KRP (Alg. 8) with per-step truncation; omegas[i][j] = step i, mode j (None for j == i)."""
    _dev_f32(X, "X")
    d = len(dims)
    R = int(omegas[0][1].shape[1])
    flat = [omegas[i][j] for i in range(d) for j in range(d)]
    Q = [torch.empty((int(n), int(r)), dtype=torch.float32, device=X.device) for n, r in zip(dims, ranks)]
    core = torch.empty(int(torch.tensor(list(ranks)).prod()), dtype=torch.float32, device=X.device)
    err = ctypes.c_double(0.0)
    w = _ws(krp_workspace_bytes(OP_STHOSVD, dims, R, ranks), X.device, ws)
    _check(lib().krp_sthosvd(X.data_ptr(), d, _dims(dims), _ints(ranks), R, _ptr_array(flat), _ptr_array(Q),
                             core.data_ptr(), ctypes.byref(err) if with_error else None, w.data_ptr(), w.numel(),
                             _stream(stream)), "krp_sthosvd")
    return Q, core, (err.value if with_error else None)


# ------------------------------------------------------------------ multi-GPU
def krp_slab_range(I_d: int, nranks: int, rank: int) -> Tuple[int, int]:
    """(begin, length) of rank's contiguous last-mode slab (host-side geometry of the sharded path)."""
    b, n = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().krp_slab_range(int(I_d), int(nranks), int(rank), ctypes.byref(b), ctypes.byref(n)),
           "krp_slab_range")
    return b.value, n.value


def krp_pack_layout(dims_local: Sequence[int], I_d_global: int, slab_begin: int, R: int) -> Tuple[List[int], int]:
    """(offsets[0..d], slab_offset) of the packed all-reduce buffer [Y_1 | ... | Y_d] (floats)."""
    d = len(dims_local)
    offs = (ctypes.c_int64 * (d + 1))()
    so = ctypes.c_int64()
    _check(lib().krp_pack_layout(d, _dims(dims_local), int(I_d_global), int(slab_begin), int(R), offs,
                                 ctypes.byref(so)), "krp_pack_layout")
    return list(offs), so.value


class Comm:
    """NCCL communicator owned by libkrp, bootstrapped through a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        nbytes = int(lib().krp_comm_id_bytes())
        uid = torch.zeros(nbytes, dtype=torch.uint8)
        if self.rank == 0 and self.world > 1:
            buf = (ctypes.c_uint8 * nbytes)()
            _check(lib().krp_comm_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "krp_comm_get_unique_id")
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        if self.world > 1:
            backend = dist.get_backend(group)
            t = uid.cuda() if backend == "nccl" else uid
            dist.broadcast(t, src=0, group=group)
            uid = t.cpu()
        cbuf = (ctypes.c_uint8 * nbytes)(*uid.tolist())
        self.handle = ctypes.c_void_p()
        _check(lib().krp_comm_init(ctypes.byref(self.handle), self.world, self.rank, ctypes.cast(cbuf, ctypes.c_void_p)),
               "krp_comm_init")

    def close(self):
        if self.handle:
            lib().krp_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def krp_sketch_all_modes_dist(X_slab: torch.Tensor, dims_local: Sequence[int], I_d_global: int, slab_begin: int,
                              omegas: Sequence[torch.Tensor], comm: Comm, Y=None, ws=None, stream=None):
    _dev_f32(X_slab, "X_slab")
    R = int(omegas[0].shape[1])
    gdims = list(dims_local[:-1]) + [int(I_d_global)]
    if Y is None:
        Y = [torch.empty((int(n), R), dtype=torch.float32, device=X_slab.device) for n in gdims]
    w = _ws(krp_workspace_bytes_dist(OP_SKETCH_ALL, dims_local, I_d_global, R), X_slab.device, ws)
    _check(lib().krp_sketch_all_modes_dist(X_slab.data_ptr(), len(dims_local), _dims(dims_local), int(I_d_global),
                                           int(slab_begin), _ptr_array(omegas), R, _ptr_array(Y), w.data_ptr(),
                                           w.numel(), comm.handle, _stream(stream)), "krp_sketch_all_modes_dist")
    return Y


def krp_rhosvd_dist(X_slab: torch.Tensor, dims_local: Sequence[int], I_d_global: int, slab_begin: int,
                    ranks: Sequence[int], omegas: Sequence[torch.Tensor], comm: Comm, with_error: bool = False,
                    ws=None, stream=None):
    _dev_f32(X_slab, "X_slab")
    R = int(omegas[0].shape[1])
    gdims = list(dims_local[:-1]) + [int(I_d_global)]
    Q = [torch.empty((int(n), int(r)), dtype=torch.float32, device=X_slab.device) for n, r in zip(gdims, ranks)]
    core = torch.empty(int(torch.tensor(list(ranks)).prod()), dtype=torch.float32, device=X_slab.device)
    err = ctypes.c_double(0.0)
    op = OP_RHOSVD_ERR if with_error else OP_RHOSVD
    w = _ws(krp_workspace_bytes_dist(op, dims_local, I_d_global, R, ranks), X_slab.device, ws)
    _check(lib().krp_rhosvd_dist(X_slab.data_ptr(), len(dims_local), _dims(dims_local), int(I_d_global),
                                 int(slab_begin), _ints(ranks), R, _ptr_array(omegas), _ptr_array(Q), core.data_ptr(),
                                 ctypes.byref(err) if with_error else None, w.data_ptr(), w.numel(), comm.handle,
                                 _stream(stream)), "krp_rhosvd_dist")
    return Q, core, (err.value if with_error else None)


def krp_sthosvd_dist(X_slab: torch.Tensor, dims_local: Sequence[int], I_d_global: int, slab_begin: int,
                     ranks: Sequence[int], omegas: Sequence[Sequence[Optional[torch.Tensor]]], comm: Comm,
                     with_error: bool = False, ws=None, stream=None):
    """Slab-sharded RSTHOSVD-KRP (Alg. 8); omegas[i][j] as in krp_sthosvd with the GLOBAL I_d rows for j = d-1."""
    _dev_f32(X_slab, "X_slab")
    d = len(dims_local)
    R = int(omegas[0][1].shape[1])
    flat = [omegas[i][j] for i in range(d) for j in range(d)]
    gdims = list(dims_local[:-1]) + [int(I_d_global)]
    Q = [torch.empty((int(n), int(r)), dtype=torch.float32, device=X_slab.device) for n, r in zip(gdims, ranks)]
    core = torch.empty(int(torch.tensor(list(ranks)).prod()), dtype=torch.float32, device=X_slab.device)
    err = ctypes.c_double(0.0)
    w = _ws(krp_workspace_bytes_dist(OP_STHOSVD, dims_local, I_d_global, R, ranks), X_slab.device, ws)
    _check(lib().krp_sthosvd_dist(X_slab.data_ptr(), d, _dims(dims_local), int(I_d_global), int(slab_begin),
                                  _ints(ranks), R, _ptr_array(flat), _ptr_array(Q), core.data_ptr(),
                                  ctypes.byref(err) if with_error else None, w.data_ptr(), w.numel(), comm.handle,
                                  _stream(stream)), "krp_sthosvd_dist")
    return Q, core, (err.value if with_error else None)


def _decomp(fname, op, X, dims, ranks, ptrs, R, with_error, ws, stream):
    Q = [torch.empty((int(n), int(r)), dtype=torch.float32, device=X.device) for n, r in zip(dims, ranks)]
    core = torch.empty(int(torch.tensor(list(ranks)).prod()), dtype=torch.float32, device=X.device)
    err = ctypes.c_double(0.0)
    w = _ws(krp_workspace_bytes(op, dims, R, ranks), X.device, ws)
    _check(getattr(lib(), fname)(X.data_ptr(), len(dims), _dims(dims), _ints(ranks), R, _ptr_array(ptrs),
                                 _ptr_array(Q), core.data_ptr(), ctypes.byref(err) if with_error else None,
                                 w.data_ptr(), w.numel(), _stream(stream)), fname)
    return Q, core, (err.value if with_error else None)


def krp_rhosvd_fresh(X: torch.Tensor, dims: Sequence[int], ranks: Sequence[int],
                     omega_steps: Sequence[Sequence[Optional[torch.Tensor]]], with_error: bool = False, ws=None,
                     stream=None):
    """RHOSVD-KRP, Alg. 7 literally: omega_steps[n][j] is mode n's fresh I_j x R factor (None for j == n)."""
    _dev_f32(X, "X")
    d = len(dims)
    R = int(omega_steps[0][1].shape[1])
    flat = [omega_steps[i][j] for i in range(d) for j in range(d)]
    return _decomp("krp_rhosvd_fresh", OP_RHOSVD_FRESH, X, dims, ranks, flat, R, with_error, ws, stream)


def krp_rhosvd_gaussian(X: torch.Tensor, dims: Sequence[int], ranks: Sequence[int],
                        omega_dense: Sequence[torch.Tensor], with_error: bool = False, ws=None, stream=None):
    """RHOSVD with dense Gaussian test matrices (Table 1 baseline): omega_dense[n] is (N/I_n) x R."""
    _dev_f32(X, "X")
    R = int(omega_dense[0].shape[1])
    return _decomp("krp_rhosvd_gaussian", OP_RHOSVD_GAUSSIAN, X, dims, ranks, list(omega_dense), R, with_error, ws,
                   stream)


def krp_sthosvd_gaussian(X: torch.Tensor, dims: Sequence[int], ranks: Sequence[int],
                         omega_dense: Sequence[torch.Tensor], with_error: bool = False, ws=None, stream=None):
    """RSTHOSVD with dense Gaussian test matrices (Table 1 baseline): omega_dense[i] is (N_i/I_i) x R."""
    _dev_f32(X, "X")
    R = int(omega_dense[0].shape[1])
    return _decomp("krp_sthosvd_gaussian", OP_STHOSVD_GAUSSIAN, X, dims, ranks, list(omega_dense), R, with_error, ws,
                   stream)


def krp_hadamard_tucker(F: torch.Tensor, A: Sequence[torch.Tensor], G: torch.Tensor, U: Sequence[torch.Tensor],
                        ranks: Sequence[int], omegas: Sequence[Sequence[Optional[torch.Tensor]]], ws=None, stream=None):
    """Alg. 9: Tucker recompression of (F x_k A_k) * (G x_k U_k) without forming the product.  F, G are flat
    first-index-fastest cores with shapes given by the factors; omegas[i][j] is n_j x l_i (None for j == i).
    Returns (Q list, core)."""
    n = [int(a.shape[0]) for a in A]
    q = [int(a.shape[1]) for a in A]
    s = [int(u.shape[1]) for u in U]
    ls = [int(omegas[i][(i + 1) % 3].shape[1]) for i in range(3)]
    for t in [F, G, *A, *U]:
        _dev_f32(t, "argument")
    Q = [torch.empty((n[i], int(ranks[i])), dtype=torch.float32, device=F.device) for i in range(3)]
    core = torch.empty(int(np.prod(ranks)), dtype=torch.float32, device=F.device)
    nb = int(lib().krp_hadamard_workspace_bytes(_dims(n), _dims(q), _dims(s), _ints(ranks), _ints(ls)))
    w = _ws(nb, F.device, ws)
    flat = [omegas[i][j] for i in range(3) for j in range(3)]
    _check(lib().krp_hadamard_tucker(F.data_ptr(), _dims(q), _ptr_array(A), G.data_ptr(), _dims(s), _ptr_array(U),
                                     _dims(n), _ints(ranks), _ints(ls), _ptr_array(flat), _ptr_array(Q),
                                     core.data_ptr(), w.data_ptr(), w.numel(), _stream(stream)), "krp_hadamard_tucker")
    return Q, core
