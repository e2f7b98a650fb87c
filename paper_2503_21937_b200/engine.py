"""Python binding of the C ABI (include/lobster.h): argument marshalling only.

Every step of the fixpoint runs in the CUDA kernels of liblobster.so; this
module converts numpy arrays / torch tensors to pointers and back.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

from . import _lib


class LobsterError(RuntimeError):
    def __init__(self, status: int, msg: str):
        name = _lib.STATUS_NAMES[status] if 0 <= status < len(_lib.STATUS_NAMES) else str(status)
        super().__init__(f"LOBSTER_E_{name}: {msg}")
        self.status = status


def _ptr(x):
    """(pointer, keepalive) for a numpy array or torch tensor (host or device)."""
    if x is None:
        return None, None
    if isinstance(x, np.ndarray):
        return x.ctypes.data, x
    if hasattr(x, "data_ptr"):
        return x.data_ptr(), x
    raise TypeError(f"unsupported buffer type {type(x)}")


def _as_i32(x):
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.int32)
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(torch.int32).contiguous()
    return np.ascontiguousarray(np.asarray(x), dtype=np.int32)


def _as_f32(x):
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.float32)
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(torch.float32).contiguous()
    return np.ascontiguousarray(np.asarray(x), dtype=np.float32)


class _CudaArray:
    """Zero-copy view of engine-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}
        self._owner = owner


def _np_view(ptr, n, dtype, copy=True):
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    ct = {np.int32: ctypes.c_int32, np.int64: ctypes.c_int64, np.float32: ctypes.c_float}[dtype]
    arr = (ct * n).from_address(ptr)
    v = np.frombuffer(arr, dtype=dtype, count=n)
    if copy:
        return v.copy()
    v.flags.writeable = False
    return v


@dataclass
class RelationOutput:
    n: int
    arity: int
    sample_ids: object
    cols: object              # (arity, n) host array or list of device tensors
    probs: object
    sample_offsets: object
    grad_offsets: object = None
    grad_fact_ids: object = None
    grad_values: object = None


class Group:
    """The ranks of one key-partitioned evaluation (include/lobster.h
    lobster_group_*).  `Group.local(W)`: W engines of this process (one host
    thread each); `Group.nccl(id, rank, W, device)`: one process per GPU, `id`
    from `Group.nccl_id()` on rank 0 (128 bytes, distributed by the caller)."""

    def __init__(self, handle):
        self._L = _lib.load()
        self._h = handle

    @classmethod
    def local(cls, world_size: int) -> "Group":
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.lobster_group_local(int(world_size), ctypes.byref(h))
        if rc != 0:
            raise LobsterError(rc, "lobster_group_local failed")
        return cls(h)

    @staticmethod
    def nccl_id() -> bytes:
        L = _lib.load()
        buf = ctypes.create_string_buffer(128)
        rc = L.lobster_nccl_id(buf)
        if rc != 0:
            raise LobsterError(rc, "lobster_nccl_id failed (libnccl.so.2 missing?)")
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, rank: int, world_size: int, device: int) -> "Group":
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.lobster_group_nccl(ctypes.create_string_buffer(bytes(uid), 128), int(rank), int(world_size),
                                  int(device), ctypes.byref(h))
        if rc != 0:
            raise LobsterError(rc, "lobster_group_nccl failed")
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            self._L.lobster_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """One lobster context: program_load -> facts_push* -> run -> output_get*."""

    def __init__(self, program: str, semiring: int, batch_size: int = 1, device: int = 0,
                 stream: Optional[int] = None, max_iters: int = 0, arena_bytes: int = 0, micro_batch: int = 0,
                 rank: int = 0, world_size: int = 1):
        self._L = _lib.load()
        o = _lib.Options()
        o.device = device
        o.cuda_stream = stream or 0
        o.batch_size = batch_size
        o.max_iters = max_iters
        o.arena_bytes = arena_bytes
        o.micro_batch = micro_batch
        o.rank = rank
        o.world_size = world_size
        # samples this context owns: the whole batch, or its shard of the
        # global batch (include/lobster.h `rank`); sample ids stay global
        base, extra = divmod(batch_size, max(world_size, 1))
        self.sample_lo = rank * base + min(rank, extra) if world_size > 1 else 0
        self.local_batch = (base + (1 if rank < extra else 0)) if world_size > 1 else batch_size
        self.batch_size = batch_size
        self.semiring = semiring
        self.device = device
        h = ctypes.c_void_p()
        rc = self._L.lobster_create(ctypes.byref(o), ctypes.byref(h))
        if rc != 0:
            raise LobsterError(rc, "lobster_create failed (no CUDA device?)")
        self._h = h
        self._check(self._L.lobster_program_load(self._h, program.encode(), semiring))
        self._group = None

    def partition(self, group: "Group", rank: int) -> None:
        """Key-partitioned evaluation of this engine's databases as `rank` of `group`
        (lobster_partition): push the same facts on every rank, run every rank."""
        self._check(self._L.lobster_partition(self._h, group._h if group is not None else None, int(rank)))
        self._group = group  # the group must outlive the context

    def _check(self, rc):
        if rc != 0:
            raise LobsterError(rc, self._L.lobster_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.lobster_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ push
    def push(self, relation: str, cols: Sequence, sample_ids=None, probs=None) -> int:
        cols = [_as_i32(c) for c in cols]
        sids = _as_i32(sample_ids)
        pr = _as_f32(probs)
        if cols:
            n = int(cols[0].shape[0])
        elif sids is not None:
            n = int(sids.shape[0])
        else:
            n = 0 if pr is None else int(pr.shape[0])
        keep = []
        colp = (ctypes.c_void_p * max(1, len(cols)))()
        for i, c in enumerate(cols):
            p, k = _ptr(c)
            colp[i] = p
            keep.append(k)
        sp, k1 = _ptr(sids)
        pp, k2 = _ptr(pr)
        first = ctypes.c_int64(0)
        self._check(self._L.lobster_facts_push(self._h, relation.encode(), n, colp, sp, pp, ctypes.byref(first)))
        del keep, k1, k2
        return first.value

    def facts_groups(self, first_fact_id: int, group_ids) -> None:
        """top-1-proof exclusion groups of facts [first, first + n) (-1 = none)."""
        g = _as_i32(group_ids)
        ptr, keep = _ptr(g)
        self._check(self._L.lobster_facts_groups(self._h, int(first_fact_id), int(len(g)), ptr))

    def push_facts(self, facts: Dict[str, object]) -> Dict[str, int]:
        """Push a dict rel -> workloads.Facts (cols, sample_ids, probs) in dict order."""
        return {rel: self.push(rel, f.cols, f.sample_ids, f.probs) for rel, f in facts.items()}

    # ------------------------------------------------------------------- run
    def run(self) -> dict:
        s = _lib.RunStats()
        self._check(self._L.lobster_run(self._h, ctypes.byref(s)))
        return s.as_dict()

    @property
    def num_facts(self) -> int:
        return int(self._L.lobster_num_facts(self._h))

    # ---------------------------------------------------------------- output
    def output(self, relation: str, device: bool = False, copy: bool = True) -> RelationOutput:
        """device=False: numpy arrays of the host copy (lobster_output_get where=0).  With
        copy=False they are read-only views of the context's pinned buffers — no extra host
        copy — valid until the next push / run / close (the C ABI's lifetime rule)."""
        o = _lib.Output()
        self._check(self._L.lobster_output_get(self._h, relation.encode(), 1 if device else 0, ctypes.byref(o)))
        n, ar = int(o.n), int(o.arity)
        if not device:
            if ar and not copy:  # columns are one arity x n block in the context's buffer
                cols = _np_view(o.columns[0], ar * n, np.int32, False).reshape(ar, n)
            elif ar:
                cols = np.stack([_np_view(o.columns[c], n, np.int32) for c in range(ar)])
            else:
                cols = np.zeros((0, n), np.int32)
            out = RelationOutput(n, ar, _np_view(o.sample_ids, n, np.int32, copy), cols,
                                 _np_view(o.probs, n, np.float32, copy) if self.semiring != _lib.UNIT else None,
                                 _np_view(o.sample_offsets, self.local_batch + 1, np.int64, copy))
            if o.grad_offsets or (self.semiring in (_lib.DIFF_MAX_MULT_PROB, _lib.DIFF_MAX_MIN_PROB, _lib.DIFF_TOP1_PROOFS) and n == 0 and o.grad_offsets is not None):
                goff = _np_view(o.grad_offsets, n + 1, np.int64, copy) if n else np.zeros(1, np.int64)
                ng = int(goff[-1]) if n else 0
                out.grad_offsets = goff
                out.grad_fact_ids = _np_view(o.grad_fact_ids, ng, np.int64, copy)
                out.grad_values = _np_view(o.grad_values, ng, np.float32, copy)
            return out
        import torch
        dev = torch.device("cuda", self.device)

        def t(ptr, shape, ts):
            if not ptr or 0 in shape:
                dt = {"<i4": torch.int32, "<i8": torch.int64, "<f4": torch.float32}[ts]
                return torch.zeros(shape, dtype=dt, device=dev)
            return torch.as_tensor(_CudaArray(ptr, shape, ts, self), device=dev)
        out = RelationOutput(n, ar, t(o.sample_ids, (n,), "<i4"), [t(o.columns[c], (n,), "<i4") for c in range(ar)],
                             t(o.probs, (n,), "<f4") if self.semiring != _lib.UNIT else None,
                             t(o.sample_offsets, (self.local_batch + 1,), "<i8"))
        if o.grad_offsets:
            goff = t(o.grad_offsets, (n + 1,), "<i8")
            ng = int(goff[-1].item()) if n else 0
            out.grad_offsets = goff
            out.grad_fact_ids = t(o.grad_fact_ids, (ng,), "<i8")
            out.grad_values = t(o.grad_values, (ng,), "<f4")
        return out

    def backward(self, relation: str, upstream, grad_facts) -> None:
        """grad_facts[f] = Σ_rows upstream[row] · ∂probs[row]/∂p_f (device tensors)."""
        up, k1 = _ptr(upstream)
        gf, k2 = _ptr(grad_facts)
        self._check(self._L.lobster_output_backward(self._h, relation.encode(), up, gf))
