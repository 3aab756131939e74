"""Communication contract of the distributed solver (mirrors btasel/collectives.py:69-79).

A ``Collectives`` endpoint offers exactly two group operations:

* ``all_gather(payload)`` -> list of every rank's payload, rank-ordered,
  identical on every rank;
* ``all_reduce_sum(tensor)`` -> elementwise sum accumulated in FIXED RANK
  ORDER, so the result is bitwise replicated and deterministic
  (collectives.py:149-158).

Transports:

* :class:`TorchCollectives` -- one process per GPU over ``torch.distributed``
  (NCCL over NVLink/NVSwitch on B200; gloo on CPU for host-logic tests).
  Payloads are device tensors packed into one fixed-size slot per rank and
  moved with a single ``all_gather_into_tensor``.  ``all_reduce_sum`` is an
  ``all_gather`` of the (tiny, 2*a*a) tip contributions followed by a
  rank-ordered local sum: same bytes on the wire as an allreduce tree at this
  size, and bitwise-identical, order-fixed results on every rank.  It also
  takes the reference's own numpy payloads (``to_bytes``/``from_bytes``,
  dist.py:73-131) and numpy tip arrays, so the reference's ``dist.py``
  orchestration (``_run_rank``) runs over NCCL unchanged.
* :class:`LocalHub` -- all partitions in one process on one GPU (the
  ``transport=None`` default of ``dist_solve``); rounds are recorded, data
  never leaves the device.

Both record a trace of rounds (``TraceEvent``) for communication-contract
checks (reference tests/test_dist.py:87-133).  ``dist_solve`` also accepts
any other Collectives -- the reference's ``ThreadHub`` (collectives.py:87-133)
or ``SocketCollectives`` -- and then exchanges host payloads by value.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ProtocolError

__all__ = ["TraceEvent", "Collectives", "TorchCollectives", "LocalHub"]


@dataclass
class TraceEvent:
    """One collective round (collectives.py:52-58)."""

    kind: str  # "all_gather" | "all_reduce"
    round_id: int
    payloads: list


def _summary(obj):
    if hasattr(obj, "summary"):
        return obj.summary()
    if isinstance(obj, torch.Tensor):
        return {"nbytes": obj.numel() * obj.element_size(), "elements": obj.numel()}
    if isinstance(obj, np.ndarray):
        return {"nbytes": obj.nbytes, "elements": obj.size}
    return {"nbytes": None}


class Collectives:
    """Abstract endpoint (collectives.py:69-79)."""

    rank: int
    world_size: int

    def all_gather(self, payload) -> list:
        raise NotImplementedError

    def all_reduce_sum(self, array: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError


class TorchCollectives(Collectives):
    """torch.distributed transport; the process group must be initialised.

    ``symmetric`` (default: env ``BSEL_SYMM_EXCHANGE=1``, NCCL groups only):
    the boundary all_gather is one kernel of NVLink peer stores
    (``bsel_publish``) into symmetric-memory receive buffers (torch
    ``_symmetric_memory``), bracketed by device-side group barriers, instead
    of pack + NCCL ``all_gather_into_tensor``.  If the symmetric rendezvous
    fails on any rank, every rank keeps the NCCL path (agreed by one
    all_reduce)."""

    def __init__(self, group=None, symmetric=None):
        import os

        import torch.distributed as dist

        if not dist.is_initialized():
            raise ProtocolError("torch.distributed is not initialised")
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        self.trace: list[TraceEvent] = []
        self._round = 0
        if symmetric is None:
            symmetric = os.environ.get("BSEL_SYMM_EXCHANGE", "0") == "1"
        self.symmetric = bool(symmetric) and dist.get_backend(group) == "nccl" and self.world_size <= 8
        self._symm = {}
        self.exchange_impl = "nccl all_gather"

    def _symm_get(self, slot: int):
        """Receive buffer (world x slot float64) in symmetric memory, its
        handle and the peers' mapped buffer pointers; None if unavailable."""
        st = self._symm.get(slot)
        if st is not None:
            return st
        import ctypes

        dev = torch.device("cuda", torch.cuda.current_device())
        ok, err = 1, None
        try:
            import torch.distributed._symmetric_memory as symm

            grp = self.group or self._dist.group.WORLD
            if hasattr(symm, "enable_symm_mem_for_group"):
                symm.enable_symm_mem_for_group(grp.group_name)
            buf = symm.empty(self.world_size * slot, dtype=torch.float64, device=dev)
            hdl = symm.rendezvous(buf, grp)
            ptrs = (ctypes.c_void_p * self.world_size)(*[int(p) for p in hdl.buffer_ptrs])
        except Exception as exc:  # noqa: BLE001 - decided collectively below
            ok, err = 0, exc
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        self._dist.all_reduce(flag, op=self._dist.ReduceOp.MIN, group=self.group)
        if not int(flag.item()):
            self.symmetric = False
            import warnings

            warnings.warn(f"symmetric-memory exchange unavailable ({err}); using NCCL all_gather")
            return None
        st = self._symm[slot] = (buf, hdl, ptrs)
        self.exchange_impl = "bsel_publish: NVLink peer stores into symmetric memory"
        return st

    def _symm_all_gather(self, payload):
        import ctypes

        from . import _native
        from .dist import _KIND_CODES

        slot = payload.slot_elems()
        st = self._symm_get(slot)
        if st is None:
            return None
        buf, hdl, ptrs = st
        w = self.world_size
        hdl.barrier(channel=0)  # every rank consumed the previous exchange
        blocks = payload.slot_blocks()
        base = self.rank * (slot // 2)  # complex offset of this rank's slot
        nb = len(blocks)
        src = (ctypes.c_void_p * max(nb, 1))(*[t.data_ptr() for t, _ in blocks])
        elems = (ctypes.c_int64 * max(nb, 1))(*[t.numel() for t, _ in blocks])
        offs = (ctypes.c_int64 * max(nb, 1))(*[base + off for _, off in blocks])
        hdr = (ctypes.c_double * 4)(float(payload.rank), float(_KIND_CODES[payload.kind]), float(len(payload.diag)),
                                    float(payload.sym_flags))
        ctx = _native.Context.get(torch.cuda.current_device())
        ctx.bind_stream()
        ctx.call("bsel_publish", src, elems, offs, nb, ptrs, w, base, hdr)
        hdl.barrier(channel=0)  # every slot written everywhere
        allp = buf.view(w, slot)
        hdrs = allp[:, :4].cpu().tolist()
        return [payload.unpack(allp[r], rank=r, header=hdrs[r]) for r in range(w)]

    def _record(self, kind, payloads):
        self.trace.append(TraceEvent(kind=kind, round_id=self._round, payloads=payloads))
        self._round += 1

    def gather_tensor(self, flat: torch.Tensor) -> torch.Tensor:
        """all_gather of equal-size flat tensors -> [world, numel]."""
        out = torch.empty((self.world_size,) + tuple(flat.shape), dtype=flat.dtype, device=flat.device)
        try:
            self._dist.all_gather_into_tensor(out, flat.contiguous(), group=self.group)
        except (RuntimeError, NotImplementedError):  # backends without the fused op (older gloo)
            self._dist.all_gather(list(out.unbind(0)), flat.contiguous(), group=self.group)
        return out

    def _device(self):
        """Where the wire tensors live: CUDA for NCCL, host memory otherwise."""
        if self._dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def _gather_bytes(self, blob: bytes) -> list:
        """all_gather of variable-length byte strings: the lengths first,
        then every blob padded to the longest (two NCCL all_gathers)."""
        dev = self._device()
        sizes = self.gather_tensor(torch.tensor([len(blob)], dtype=torch.int64, device=dev)).view(-1).tolist()
        buf = torch.zeros(max(sizes), dtype=torch.uint8)
        if blob:
            buf[:len(blob)] = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
        allb = self.gather_tensor(buf.to(dev)).cpu().numpy()
        return [allb[r, :sizes[r]].tobytes() for r in range(self.world_size)]

    def all_gather(self, payload) -> list:
        """* device payloads exposing pack()/unpack() (this package's
          BoundaryPayload) travel as one fixed-size slot per rank, all ranks'
          headers read back with ONE device->host copy;
        * payloads exposing to_bytes()/from_bytes() -- the reference's numpy
          BoundaryPayload (dist.py:73-131), or a host payload of this package
          -- travel as bytes, so the reference's own dist.py orchestration
          runs over NCCL;
        * tensors / numpy arrays of identical shape on all ranks."""
        on_dev = getattr(payload, "on_device", None)
        out = None
        if self.symmetric and hasattr(payload, "slot_blocks") and on_dev is not None and on_dev():
            out = self._symm_all_gather(payload)
        if out is not None:
            pass
        elif hasattr(payload, "pack") and (on_dev is None or on_dev()):
            flat = payload.pack()
            allp = self.gather_tensor(flat)
            hdrs = allp[:, :4].cpu().tolist()
            out = [payload.unpack(allp[r], rank=r, header=hdrs[r]) for r in range(self.world_size)]
        elif hasattr(payload, "to_bytes"):
            blobs = self._gather_bytes(payload.to_bytes())
            out = [type(payload).from_bytes(bl) for bl in blobs]
        elif isinstance(payload, np.ndarray):
            allp = self.gather_tensor(torch.from_numpy(np.ascontiguousarray(payload)).to(self._device()))
            out = [allp[r].cpu().numpy() for r in range(self.world_size)]
        else:
            allp = self.gather_tensor(payload)
            out = [allp[r] for r in range(self.world_size)]
        self._record("all_gather", [_summary(p) for p in out])
        return out

    def gather_to_root(self, blob: bytes):
        """Rank 0 receives every rank's bytes (rank order); others get None
        (the reference's SocketCollectives.gather_to_root contract)."""
        blobs = self._gather_bytes(blob)
        return blobs if self.rank == 0 else None

    def all_reduce_sum(self, array):
        """Elementwise sum in FIXED rank order (bitwise replicated).  numpy
        arrays in -> numpy out (the reference's contract), tensors -> tensors."""
        if isinstance(array, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(array)).to(self._device())
            return self.all_reduce_sum(t).cpu().numpy()
        allp = self.gather_tensor(torch.view_as_real(array) if array.is_complex() else array)
        if array.is_complex():
            allp = torch.view_as_complex(allp)
        total = allp[0].clone()
        for r in range(1, self.world_size):
            total += allp[r]
        self._record("all_reduce", [{"nbytes": array.numel() * array.element_size(),
                                     "elements": array.numel()}] * self.world_size)
        return total


class LocalHub:
    """In-process stand-in for P ranks on one device (ThreadHub analogue,
    collectives.py:87-133): the driver hands it the list of per-rank
    contributions; rounds are recorded like a real transport."""

    def __init__(self, world_size: int):
        if world_size < 1:
            raise ValueError("world_size must be positive")
        self.world_size = world_size
        self.trace: list[TraceEvent] = []
        self._round = 0

    def _record(self, kind, payloads):
        self.trace.append(TraceEvent(kind=kind, round_id=self._round, payloads=payloads))
        self._round += 1

    def all_gather_all(self, payloads: list) -> list:
        if len(payloads) != self.world_size:
            raise ProtocolError(f"expected {self.world_size} payloads, got {len(payloads)}")
        self._record("all_gather", [_summary(p) for p in payloads])
        return list(payloads)

    def all_reduce_all(self, arrays: list) -> torch.Tensor:
        total = arrays[0].clone()
        for part in arrays[1:]:
            if part.shape != total.shape:
                raise ProtocolError(f"all_reduce shape mismatch: {tuple(part.shape)} vs {tuple(total.shape)}")
            total += part
        self._record("all_reduce", [{"nbytes": x.numel() * x.element_size(), "elements": x.numel()}
                                    for x in arrays])
        return total
