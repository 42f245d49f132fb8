"""Pair shards of the packed power cache over an NCCL communicator owned by the C library
(include/fgfrft_b200.h `fgfrft_comm_*`, `fgfrft_pshard_*`; csrc/capi_pshard.cu).

Rank g owns the tile pairs {(I,J),(J,I)}, I <= J, whose smaller tile index I lies in its band
[I_g, I_(g+1)) (`pair_plan`: ~npairs / G pairs each). Its synthesised tiles cover two rectangles of
Q (and dQ/da): A = rows R_g x columns [32 I_g, N) and B = rows [32 I_(g+1), N) x columns R_g
(R_g = rows [32 I_g, 32 I_(g+1))), so its partial products are Y_g[R_g] = A X[32 I_g:] and
Y_g[32 I_(g+1):] = B X[R_g]; sum_g Y_g = Y. A step = one reduce-scatter of [Y; dY] by signal-
column chunks + one all-reduce of 2A doubles (loss and dL/da of every order).

`decomposed_partial` restates that decomposition in numpy on an explicit Q: the CPU tests run it
per rank over gloo (tests/test_pshard.py) to check the plan and the collectives; the product path
is the CUDA library.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _check, _cm, _ptr, lib

TILE = 32
COMM_ID_BYTES = 128


def pair_plan(n: int, world: int) -> list:
    """Tile-row band boundaries [I_0 = 0, ..., I_G = ceil(n / 32)] (fgfrft_pshard_plan)."""
    out = (ctypes.c_int * (world + 1))()
    _check(lib().fgfrft_pshard_plan(int(n), int(world), ctypes.addressof(out)))
    return list(out)


def pairs_before(i: int, nt: int) -> int:
    """Number of tile pairs (I <= J) with smaller index < i (the I-major enumeration)."""
    return i * nt - i * (i - 1) // 2


def rank_rows(n: int, world: int, rank: int):
    b = pair_plan(n, world)
    return min(n, b[rank] * TILE), min(n, b[rank + 1] * TILE)


def decomposed_partial(q: np.ndarray, x: np.ndarray, n: int, world: int, rank: int) -> np.ndarray:
    """Rank `rank`'s partial product of Y = Q X under the pair decomposition (numpy, any dtype):
    zero except rows [r0, N) -- rectangle A (rows [r0, r1) x cols [r0, N)) and rectangle B
    (rows [r1, N) x cols [r0, r1))."""
    r0, r1 = rank_rows(n, world, rank)
    y = np.zeros((n, x.shape[1]), dtype=np.result_type(q, x))
    if r1 <= r0:
        return y
    y[r0:r1] = q[r0:r1, r0:] @ x[r0:]
    y[r1:] = q[r1:, r0:r1] @ x[r0:r1]
    return y


class Comm:
    """An NCCL communicator held by the library (ncclCommInitRank). Bootstrap: rank 0 calls
    `unique_id()` and the launcher hands the bytes to every rank."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int = 0):
        if len(uid) != COMM_ID_BYTES:
            raise ValueError("Comm: the unique id is 128 bytes")
        self._h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, COMM_ID_BYTES)
        _check(lib().fgfrft_comm_create(buf, int(world), int(rank), int(device), ctypes.byref(self._h)))
        self.world, self.rank, self.device = int(world), int(rank), int(device)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(COMM_ID_BYTES)
        _check(lib().fgfrft_comm_unique_id(buf))
        return buf.raw

    @property
    def handle(self):
        return self._h

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_comm_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PairShard:
    """One rank's pair shard. `PairShard(f, l, budget, comm=comm)` (collectives through the
    library's NCCL communicator) or `PairShard(f, l, budget, world=G, rank=g)` (no communicator:
    partial products only). `f` may be None on ranks != 0 with a communicator (broadcast)."""

    def __init__(self, f: Optional[np.ndarray], l: int, memory_budget: int = 64 << 30, comm: Optional[Comm] = None,
                 world: int = 1, rank: int = 0, device: int = 0, n: Optional[int] = None):
        self._h = ctypes.c_void_p()
        fc = _cm(f) if f is not None else None
        nn = fc.shape[0] if fc is not None else int(n)
        fp = _ptr(fc) if fc is not None else None
        if comm is not None:
            _check(lib().fgfrft_pshard_create(fp, nn, int(l), int(memory_budget), comm.handle, ctypes.byref(self._h)))
            world, rank, device = comm.world, comm.rank, comm.device
        else:
            _check(lib().fgfrft_pshard_create_local(fp, nn, int(l), int(memory_budget), int(world), int(rank),
                                                    int(device), ctypes.byref(self._h)))
        self.n, self.l, self.world, self.rank, self.device, self.comm = nn, int(l), world, rank, device, comm

    @property
    def handle(self):
        return self._h

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().fgfrft_pshard_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        w, r = ctypes.c_int(), ctypes.c_int()
        p0, p1, r0, r1, nb = (ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(),
                              ctypes.c_uint64())
        _check(lib().fgfrft_pshard_info(self._h, *(ctypes.addressof(v) for v in (w, r, p0, p1, r0, r1, nb))))
        return {"world": w.value, "rank": r.value, "pair_begin": p0.value, "pair_end": p1.value,
                "row_begin": r0.value, "row_end": r1.value, "device_bytes": nb.value}

    def set_stream(self, stream_handle: int) -> None:
        _check(lib().fgfrft_pshard_set_stream(self._h, ctypes.c_void_p(stream_handle)))

    def _torch_stream(self):
        """Device calls are stream-ordered with torch's current stream (like the tensors they fill)."""
        import torch
        self.set_stream(torch.cuda.current_stream().cuda_stream)

    def partial(self, alphas: Sequence[float], x_dev, with_dq: bool = True):
        """This rank's partial products (device tensor [rows, b, n] complex128; column-major blocks)."""
        import torch
        self._torch_stream()
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        b = int(x_dev.shape[0])
        rows = len(al) * (2 if with_dq else 1)
        out = torch.empty((rows, b, self.n), dtype=torch.complex128, device=x_dev.device)
        _check(lib().fgfrft_pshard_partial_dev(self._h, al.ctypes.data, len(al), int(with_dq), x_dev.data_ptr(), b,
                                               out.data_ptr()))
        return out

    def partial_scatter(self, alphas: Sequence[float], x_dev, dests, with_dq: bool = True) -> None:
        """The fused reduce-scatter's data path: this rank's partial tiles stored by the GEMM epilogue
        into dests[h] (device pointers: this rank's receive slot in owner h's buffer, rows blocks of
        n x ceil(b / len(dests)) complex)."""
        self._torch_stream()
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        arr = (ctypes.c_void_p * len(dests))(*[ctypes.c_void_p(int(d)) for d in dests])
        _check(lib().fgfrft_pshard_partial_scatter_dev(self._h, al.ctypes.data, len(al), int(with_dq),
                                                       x_dev.data_ptr(), int(x_dev.shape[0]), arr, len(dests)))

    def mse_step_dev(self, alphas: Sequence[float], x_dev, xc_dev):
        """(loss, dL/da) device tensors, every rank (reduce-scatter + all-reduce inside)."""
        import torch
        self._torch_stream()
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        lo = torch.empty(len(al), dtype=torch.float64, device=x_dev.device)
        dl = torch.empty(len(al), dtype=torch.float64, device=x_dev.device)
        _check(lib().fgfrft_pshard_mse_step_dev(self._h, al.ctypes.data, len(al), x_dev.data_ptr(), xc_dev.data_ptr(),
                                                int(x_dev.shape[0]), lo.data_ptr(), dl.data_ptr()))
        return lo, dl

    def mse_step(self, alphas: Sequence[float], x: np.ndarray, x_clean: np.ndarray):
        """Host buffers (n x b complex): (loss[A], dL/da[A]) on every rank."""
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        xc, xcl = _cm(x), _cm(x_clean)
        lo, dl = np.empty(len(al)), np.empty(len(al))
        _check(lib().fgfrft_pshard_mse_step(self._h, _ptr(al), len(al), _ptr(xc), _ptr(xcl), xc.shape[1], _ptr(lo),
                                            _ptr(dl)))
        return lo, dl

    def apply_dev(self, alphas: Sequence[float], x_dev, inverse: bool = False):
        """Full Y = F^a X on every rank (all-reduce of the partials): [A, b, n] complex128."""
        import torch
        self._torch_stream()
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        b = int(x_dev.shape[0])
        y = torch.empty((len(al), b, self.n), dtype=torch.complex128, device=x_dev.device)
        _check(lib().fgfrft_pshard_apply_dev(self._h, al.ctypes.data, len(al), int(inverse), x_dev.data_ptr(), b,
                                             y.data_ptr()))
        return y
