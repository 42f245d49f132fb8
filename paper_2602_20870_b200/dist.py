"""Multi-GPU orchestration of the row-sharded hot path (one process per GPU).

SURVEY 8(e) / north star: when the cache exceeds one GPU's HBM (config 4: L=128, N=8192), the
powers are sharded by ROW SLABS. Rank g owns output rows R_g and stores P_k[R_g,:] and
P_k[:,R_g] (the rows of F^k and F^{-k}); F is replicated for the build. Everything else is
local (libfgfrft_b200.so `fgfrft_shard_*`), and the only collectives are

  * all_reduce(sum) of the per-order loss partials and dL/dalpha partials (device shards:
    `fgfrft_shard_mse_dlda_partial_dev`; a RankCompute without it sends the 2L+1 per-power
    partials s_k instead), and
  * an all_gather of the rows of Y = F^alpha X (only when the caller wants Y) -- either NCCL
    (`apply`) or fused into the GEMM epilogue (`apply_fused`: every rank's kernel stores its rows
    into every rank's Y buffer over NVLink through CUDA IPC mappings).

Collectives go through torch.distributed (NCCL over NVLink on GPUs; gloo on CPU in the tests).
The per-rank compute is the `RankCompute` interface: `CudaShard` is the product implementation;
tests substitute a CPU double to exercise the collective logic on gloo.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np

TILE = 32


def plan_rows(n: int, world: int) -> List[Tuple[int, int]]:
    """Split n rows into `world` contiguous ranges of whole 32-row tiles, as even as possible
    (the last range ends at n). Ranks beyond the tile count get empty ranges (r0 == r1)."""
    if n < 1 or world < 1:
        raise ValueError("plan_rows: need n >= 1 and world >= 1")
    nt = -(-n // TILE)
    out = []
    for g in range(world):
        t0 = (nt * g) // world
        t1 = (nt * (g + 1)) // world
        out.append((min(n, t0 * TILE), min(n, t1 * TILE)))
    return out


def _signals(x) -> int:
    """Number of signals b: host arrays are n x b; device tensors are stored transposed, b x n
    (the column-major n x b block)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return int(x.shape[0])
    except ImportError:
        pass
    return int(np.asarray(x).shape[1])


class RankCompute:
    """Per-rank work on rows [r0, r1). All arrays are numpy/torch on the rank's device."""

    r0: int
    r1: int
    n: int
    l: int

    def mse_partial(self, alphas: np.ndarray, x, xc_rows):
        """-> (loss_partial [A], s_partial [A, 2L+1], y_rows [A, rows, b])"""
        raise NotImplementedError

    def apply_rows(self, alphas: np.ndarray, x):
        raise NotImplementedError


class CudaShard(RankCompute):
    """Product path: a row shard in libfgfrft_b200.so on `device`, torch tensors as buffers."""

    def __init__(self, f: np.ndarray, l: int, r0: int, r1: int, device: int = 0, memory_budget: int = 1 << 40):
        import torch

        from . import _check, _cm, lib
        self.torch = torch
        self.n, self.l, self.r0, self.r1, self.device = f.shape[0], l, r0, r1, device
        self._h = ctypes.c_void_p()
        fc = _cm(f)
        _check(lib().fgfrft_shard_create(fc.ctypes.data, self.n, l, r0, r1, memory_budget, device,
                                         ctypes.byref(self._h)))
        self._lib = lib()
        self._check = _check
        # order the shard's kernels with torch's work on this device (outputs are torch tensors)
        self.set_stream(torch.cuda.current_stream(device).cuda_stream)

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._lib.fgfrft_shard_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    def set_stream(self, stream_handle: int) -> None:
        self._check(self._lib.fgfrft_shard_set_stream(self._h, ctypes.c_void_p(stream_handle)))

    def _dev(self):
        return self.torch.device("cuda", self.device)

    def mse_partial(self, alphas, x, xc_rows, want_y: bool = False):
        t = self.torch
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        A, b = len(al), _signals(x)
        xd = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(np.asarray(x).T)).to(self._dev())
        xcd = xc_rows if isinstance(xc_rows, t.Tensor) else \
            t.from_numpy(np.ascontiguousarray(np.asarray(xc_rows).T)).to(self._dev())
        loss = t.empty(A, dtype=t.float64, device=self._dev())
        s = t.empty((A, 2 * self.l + 1), dtype=t.float64, device=self._dev())
        y = t.empty((A, b, self.rows), dtype=t.complex128, device=self._dev()) if want_y else None
        self._check(self._lib.fgfrft_shard_mse_partial_dev(
            self._h, al.ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b, y.data_ptr() if want_y else None,
            loss.data_ptr(), s.data_ptr()))
        return loss, s, y

    def mse_dlda_partial(self, alphas, x, xc_rows):
        """-> (loss_partial [A], dlda_partial [A]) on the device: dL/dalpha per order without the
        per-power partials (dQ/dalpha rows from the same pass over the panels for <= 2 orders)."""
        t = self.torch
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        A, b = len(al), _signals(x)
        xd = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(np.asarray(x).T)).to(self._dev())
        xcd = xc_rows if isinstance(xc_rows, t.Tensor) else \
            t.from_numpy(np.ascontiguousarray(np.asarray(xc_rows).T)).to(self._dev())
        out = t.empty(2 * A, dtype=t.float64, device=self._dev())
        self._check(self._lib.fgfrft_shard_mse_dlda_partial_dev(
            self._h, al.ctypes.data, A, xd.data_ptr(), xcd.data_ptr(), b, None, out.data_ptr(),
            out[A:].data_ptr()))
        return out

    def apply_gather(self, alphas, x, y_full, peers: Sequence[int] = ()):
        """Rows [r0, r1) of Y into y_full ([A, b, n] device tensor = A column-major n x b blocks)
        and, by the same GEMM epilogue, into every peer buffer (device pointers mapped over
        NVLink, fgfrft_ipc_open): the fused all-gather of the row-sharded apply."""
        t = self.torch
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        b = _signals(x)
        xd = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(np.asarray(x).T)).to(self._dev())
        arr = (ctypes.c_void_p * max(1, len(peers)))(*[ctypes.c_void_p(int(p)) for p in peers])
        self._check(self._lib.fgfrft_shard_apply_gather_dev(self._h, al.ctypes.data, len(al), xd.data_ptr(), b,
                                                            y_full.data_ptr(), arr if peers else None, len(peers)))
        return y_full

    def apply_rows(self, alphas, x):
        t = self.torch
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        A, b = len(al), _signals(x)
        xd = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(np.asarray(x).T)).to(self._dev())
        y = t.empty((A, b, self.rows), dtype=t.complex128, device=self._dev())
        self._check(self._lib.fgfrft_shard_apply_dev(self._h, al.ctypes.data, A, xd.data_ptr(), b, y.data_ptr()))
        return y  # y[a] is the column-major rows x b block (stored transposed)

    def synthesize_rows(self, alphas, which: int = 0):
        t = self.torch
        al = np.ascontiguousarray(alphas, dtype=np.float64)
        out = t.empty((len(al), self.n, self.rows), dtype=t.complex128, device=self._dev())
        self._check(self._lib.fgfrft_shard_synthesize_dev(self._h, al.ctypes.data, len(al), which, out.data_ptr()))
        return out


class ShardedFGFRFT:
    """One rank of the row-sharded transform. `compute` does the local work; collectives run on
    `group` (torch.distributed). Coefficient derivatives c'_k come from the library's host code."""

    def __init__(self, compute: RankCompute, n: int, l: int, group=None):
        self.compute, self.n, self.l, self.group = compute, n, l, group

    def _dist(self):
        import torch.distributed as dist
        return dist

    def mse_step(self, alphas: Sequence[float], x, x_clean_rows) -> Tuple[np.ndarray, np.ndarray]:
        """Per order: loss = ||Q X - Xc||^2 / (n b), dloss/dalpha. Returns host arrays (all ranks)."""
        from . import sinc_coeffs
        torch = __import__("torch")
        dist = self._dist()
        A = len(alphas)
        b = _signals(x)
        if hasattr(self.compute, "mse_dlda_partial"):  # device: [loss partials | dL/dalpha partials]
            packed = self.compute.mse_dlda_partial(np.asarray(alphas, dtype=np.float64), x, x_clean_rows)
            if dist.is_initialized() and dist.get_world_size(self.group) > 1:
                dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=self.group)  # the only data collective
            packed = packed.cpu().numpy()
            return packed[:A] / (self.n * b), packed[A:].copy()
        loss_p, s_p, _ = self.compute.mse_partial(np.asarray(alphas, dtype=np.float64), x, x_clean_rows)
        loss_t = loss_p if isinstance(loss_p, torch.Tensor) else torch.from_numpy(np.asarray(loss_p))
        s_t = s_p if isinstance(s_p, torch.Tensor) else torch.from_numpy(np.asarray(s_p))
        packed = torch.cat([loss_t.reshape(-1), s_t.reshape(-1)])
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=self.group)  # the only data collective
        packed = packed.cpu().numpy()
        loss = packed[:A] / (self.n * b)
        s = packed[A:].reshape(A, 2 * self.l + 1)
        dl = np.array([float(np.dot(sinc_coeffs(float(a), self.l)[1], s[i])) for i, a in enumerate(alphas)])
        return loss, dl

    def _peer_buffers(self, y_full):
        """IPC-map every other rank's y_full once per buffer; returns their device pointers."""
        from . import _check, lib
        dist = self._dist()
        key = (y_full.data_ptr(), tuple(y_full.shape))
        cache = getattr(self, "_peer_cache", None)
        if cache and cache[0] == key:
            return cache[1]
        for base in getattr(self, "_peer_bases", []):
            lib().fgfrft_ipc_close(ctypes.c_void_p(base))
        h = (ctypes.c_char * 64)()
        off = ctypes.c_uint64()
        _check(lib().fgfrft_ipc_get(ctypes.c_void_p(y_full.data_ptr()), h, ctypes.addressof(off)))
        world, me = dist.get_world_size(self.group), dist.get_rank(self.group)
        mine = (bytes(h), off.value)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=self.group)
        ptrs, bases = [], []
        for r, (hb, o) in enumerate(allh):
            if r == me:
                continue
            base = ctypes.c_void_p()
            _check(lib().fgfrft_ipc_open(ctypes.create_string_buffer(hb, 64), y_full.device.index,
                                         ctypes.byref(base)))
            bases.append(base.value)
            ptrs.append(base.value + o)
        self._peer_cache, self._peer_bases = (key, ptrs), bases
        return ptrs

    def apply_fused(self, alphas: Sequence[float], x):
        """Full Y = F^alpha X on every rank with the all-gather fused into the GEMM epilogue: each
        rank's kernel stores its rows into every rank's Y buffer over NVLink (CUDA IPC mappings),
        then a host barrier. Returns a NEW [A, b, n] device tensor (column-major n x b blocks) owned
        by the caller; the IPC-mapped gather buffer itself is internal.

        Ordering: a barrier before the GEMM (no rank writes into a peer's gather buffer while that
        peer may still be copying out the previous call's result) and one after it (every rank's
        rows have landed in every buffer)."""
        torch = __import__("torch")
        dist = self._dist()
        A, b = len(alphas), _signals(x)
        shape = (A, b, self.n)
        y = getattr(self, "_yfull", None)
        if y is None or tuple(y.shape) != shape:
            y = torch.empty(shape, dtype=torch.complex128, device=self.compute._dev())
            self._yfull = y
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        peers = self._peer_buffers(y) if world > 1 else []
        if world > 1:
            torch.cuda.synchronize(y.device)
            dist.barrier(group=self.group)  # peers are done reading the previous call's rows
        self.compute.apply_gather(np.asarray(alphas, dtype=np.float64), x, y, peers)
        torch.cuda.synchronize(y.device)
        if world > 1:
            dist.barrier(group=self.group)  # every rank's rows have landed in every buffer
        out = y.clone()
        torch.cuda.synchronize(y.device)  # the copy-out completes before any peer's next write
        return out

    def apply(self, alphas: Sequence[float], x, plan: Optional[List[Tuple[int, int]]] = None):
        """Full Y = F^alpha X on every rank: local rows, then all_gather of the row blocks."""
        torch = __import__("torch")
        dist = self._dist()
        y_rows = self.compute.apply_rows(np.asarray(alphas, dtype=np.float64), x)
        y_t = y_rows if isinstance(y_rows, torch.Tensor) else torch.from_numpy(np.asarray(y_rows))
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        plan = plan or plan_rows(self.n, world)
        if world == 1:
            blocks = [y_t]
        else:
            maxr = max(r1 - r0 for r0, r1 in plan)
            pad = torch.zeros((y_t.shape[0], y_t.shape[1], maxr), dtype=y_t.dtype, device=y_t.device)
            pad[:, :, :y_t.shape[2]] = y_t
            blocks = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(blocks, pad, group=self.group)
            blocks = [blk[:, :, :r1 - r0] for blk, (r0, r1) in zip(blocks, plan)]
        full = torch.cat(blocks, dim=2)  # [A, b, n]: row-major storage of column-major n x b blocks
        return full.cpu().numpy().transpose(0, 2, 1)
