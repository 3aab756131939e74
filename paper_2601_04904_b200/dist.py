"""Distributed selected inversion / quadratic solution (drop-in for btasel/dist.py).

The paper's scheme: contiguous partitions of diagonal
blocks (partition.py), each eliminated locally on its own GPU by the sm_100a
partition kernels (csrc/partition.cu: first = downward, last = upward,
middle = downward with fill-in to its top boundary); ONE all_gather of the
fixed-layout boundary payload plus (a > 0) ONE rank-ordered all_reduce of the
tip contributions; every rank assembles and solves the small reduced BTA
system (2P-2 diagonal blocks + tip) redundantly; then each partition
back-substitutes locally, seeded from the reduced solution.  Outputs stay
sharded on the devices unless gathered.

Transports: ``TorchCollectives`` (one process per GPU, NCCL over NVLink) or
the in-process ``LocalHub`` (all partitions on one GPU, the default).
"""

from __future__ import annotations

import ctypes
import os
import struct
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .collectives import Collectives, LocalHub, TorchCollectives
from .device import DeviceBta, to_device, to_host
from .errors import ProtocolError, ShapeMismatchError, WorkerError
from .kernels import OpCounter, record_sweep
from .matrix import BtaMatrix, SelectedSolution
from .partition import PartitionPlan, plan_partitions
from .rgf import solve_selected

__all__ = ["BoundaryPayload", "LocalFactors", "ReducedSystem", "local_forward", "assemble_reduced",
           "solve_reduced", "local_backward", "dist_solve", "DistSolver", "InGpuPartitions", "record_partition",
           "owned_slices", "merge_slices"]

_KIND_CODES = {"first": 0, "middle": 1, "last": 2}
_KIND_NAMES = {v: k for k, v in _KIND_CODES.items()}
_FIELDS = ("diag", "coupling", "arrow_row", "arrow_col", "b_diag", "b_coupling", "b_arrow_row", "b_arrow_col")


def _np(t):
    """Host numpy copy of a device/host tensor or array."""
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def _nbytes(t) -> int:
    return t.numel() * t.element_size() if isinstance(t, torch.Tensor) else int(np.asarray(t).nbytes)


def _dev_tensor(x, dev):
    """Device tensor of a numpy array or tensor (no copy when already there)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(dev)


def _native_transport(coll) -> bool:
    """Transports of this package move device tensors; any other
    Collectives (the reference's ThreadHub endpoints / SocketCollectives, a
    user's transport) gets host payloads, by value, like the reference."""
    return isinstance(coll, TorchCollectives)

# Logical per-step product inventory of the partition sweeps (dist.py:211-397,
# 595-742), checked against the reference OpCounter in tests.
_PART_TABLE = {
    ("si", "end", "forward"): {"bbb": 2, "bba": 2, "abb": 1, "aba": 1},
    ("siq", "end", "forward"): {"bbb": 8, "abb": 5, "bba": 5, "aba": 4},
    ("si", "middle", "forward"): {"bbb": 6, "abb": 3, "bba": 2, "aba": 1},
    ("siq", "middle", "forward"): {"bbb": 22, "abb": 10, "bba": 8, "aba": 4},
    ("si", "end", "backward"): {"bbb": 6, "bab": 3, "bba": 2, "baa": 1, "abb": 2, "aab": 1},
    ("siq", "end", "backward"): {"bbb": 26, "bab": 11, "bba": 7, "baa": 3, "abb": 8, "aab": 4},
    ("si", "middle", "backward"): {"bbb": 15, "bab": 5, "bba": 3, "baa": 1, "abb": 3, "aab": 1},
    ("siq", "middle", "backward"): {"bbb": 59, "bab": 18, "bba": 10, "baa": 3, "abb": 12, "aab": 4},
}


def record_partition(counter, kind, length, b, a, mode, phase):
    """Add the reference's logical counts of one partition sweep."""
    if counter is None:
        return
    role = "middle" if kind == "middle" else "end"
    steps = length - 2 if role == "middle" else length - 1
    if steps <= 0:
        return
    dims = {"b": b, "a": a}
    for label, cnt in _PART_TABLE[(mode, role, phase)].items():
        if "a" in label and a == 0:
            continue
        counter.gemm_by_shape["".join(counter._classify(dims[ch]) for ch in label)] += cnt * steps
    if phase == "forward":
        counter.lu_count += steps
        counter.inv_count += steps
        counter.trsm_count += 2 * steps


# ---------------------------------------------------------------------------
# Containers
# ---------------------------------------------------------------------------


@dataclass
class BoundaryPayload:
    """One rank's AllGather contribution (dist.py:73-131), device tensors.

    ``pack``/``unpack`` use one fixed-size slot (the middle-partition
    inventory) so the exchange is a single equal-size all_gather.
    """

    rank: int
    kind: str
    b: int
    a: int
    fused: bool
    diag: list = field(default_factory=list)
    coupling: list = field(default_factory=list)
    arrow_row: list = field(default_factory=list)
    arrow_col: list = field(default_factory=list)
    b_diag: list = field(default_factory=list)
    b_coupling: list = field(default_factory=list)
    b_arrow_row: list = field(default_factory=list)
    b_arrow_col: list = field(default_factory=list)
    # symmetry flags of this rank's check of B (Context.b_symmetry; 3 = none),
    # carried in the slot header: the reduced solve and every local backward
    # take the symmetric path only if ALL of B is (anti-)Hermitian
    sym_flags: int = 3

    def nbytes(self) -> int:
        return sum(_nbytes(t) for f in _FIELDS for t in getattr(self, f))

    def on_device(self) -> bool:
        """True when the blocks are torch tensors (device slot path); False
        for a host (numpy) payload."""
        return bool(self.diag) and isinstance(self.diag[0], torch.Tensor)

    def to_host(self) -> "BoundaryPayload":
        """The same payload with numpy blocks (message passing by value over
        a foreign transport, dist.py:73-131 semantics)."""
        p = BoundaryPayload(rank=self.rank, kind=self.kind, b=self.b, a=self.a, fused=self.fused,
                            sym_flags=self.sym_flags)
        for f in _FIELDS:
            setattr(p, f, [_np(t) for t in getattr(self, f)])
        return p

    def to_bytes(self) -> bytes:
        """Wire form for byte transports (the reference SocketCollectives,
        TorchCollectives' byte path): little-endian u32 rank, u8 kind code;
        per field a u32 block count, then per block u64 rows, u64 cols and
        the row-major complex128 data; a trailing i32 carries sym_flags."""
        out = [struct.pack("<IB", self.rank, _KIND_CODES[self.kind])]
        for f in _FIELDS:
            blocks = [_np(t) for t in getattr(self, f)]
            out.append(struct.pack("<I", len(blocks)))
            for blk in blocks:
                out.append(struct.pack("<QQ", *blk.shape))
                out.append(np.ascontiguousarray(blk, dtype="<c16").tobytes())
        out.append(struct.pack("<i", int(self.sym_flags)))
        return b"".join(out)

    @classmethod
    def from_bytes(cls, buf: bytes) -> "BoundaryPayload":
        rank, code = struct.unpack_from("<IB", buf, 0)
        if code not in _KIND_NAMES:
            raise ProtocolError(f"payload carries unknown kind code {code}")
        off = 5
        fields = {}
        for f in _FIELDS:
            (count,) = struct.unpack_from("<I", buf, off)
            off += 4
            blocks = []
            for _ in range(count):
                r, c = struct.unpack_from("<QQ", buf, off)
                off += 16
                blocks.append(np.frombuffer(buf, dtype="<c16", count=r * c, offset=off).reshape(r, c).copy())
                off += 16 * r * c
            fields[f] = blocks
        (sym,) = struct.unpack_from("<i", buf, off) if len(buf) >= off + 4 else (3,)
        d = fields["diag"]
        b = d[0].shape[0] if d else 0
        a = fields["arrow_row"][0].shape[0] if fields["arrow_row"] else 0
        return cls(rank=rank, kind=_KIND_NAMES[code], b=b, a=a, fused=bool(fields["b_diag"]), sym_flags=sym,
                   **fields)

    def summary(self) -> dict:
        blocks = {f: [tuple(t.shape) for t in getattr(self, f)] for f in _FIELDS if getattr(self, f)}
        return {"rank": self.rank, "kind": self.kind, "nbytes": self.nbytes(), "blocks": blocks}

    def _layout(self):
        b, a = self.b, self.a
        shapes = {"diag": (b, b), "coupling": (b, b), "arrow_row": (a, b), "arrow_col": (b, a)}
        sides = ("",) + (("b_",) if self.fused else ())
        return [(s + f, shapes[f]) for s in sides for f in ("diag", "coupling", "arrow_row", "arrow_col")]

    def slot_elems(self) -> int:
        return 4 + sum(2 * 2 * r * c for _, (r, c) in self._layout())  # 2 blocks per field

    def slot_blocks(self) -> list:
        """(block tensor, complex offset within the slot) of every block, in
        ``pack``'s layout (header = the first 2 complex)."""
        out, off = [], 2
        for name, (r, c) in self._layout():
            for j in range(2):
                lst = getattr(self, name)
                if j < len(lst):
                    out.append((lst[j], off))
                off += r * c
        return out

    def pack(self) -> torch.Tensor:
        dev = self.diag[0].device
        out = torch.zeros(self.slot_elems(), dtype=torch.float64, device=dev)
        out[0], out[1], out[2] = float(self.rank), float(_KIND_CODES[self.kind]), len(self.diag)
        out[3] = float(self.sym_flags)
        off = 4
        for name, (r, c) in self._layout():
            for t in getattr(self, name):
                out[off:off + 2 * r * c] = torch.view_as_real(t.contiguous()).reshape(-1)
                off += 2 * r * c
            off += 2 * r * c * (2 - len(getattr(self, name)))
        return out

    def unpack(self, flat: torch.Tensor, rank: int, header=None) -> "BoundaryPayload":
        """``header``: the slot's first 4 values already on the host
        (TorchCollectives reads all ranks' headers with ONE device->host
        copy); read from ``flat`` otherwise."""
        hdr = flat[:4].tolist() if header is None else list(header)
        kind = _KIND_NAMES.get(int(hdr[1]))
        if kind is None or int(hdr[0]) != rank:
            raise ProtocolError(f"payload {rank} carries rank {int(hdr[0])} kind code {int(hdr[1])}")
        nbnd = int(hdr[2])
        p = BoundaryPayload(rank=rank, kind=kind, b=self.b, a=self.a, fused=self.fused, sym_flags=int(hdr[3]))
        off = 4
        for name, (r, c) in self._layout():
            count = nbnd if not name.endswith("coupling") else (2 if kind == "middle" else 0)
            lst = []
            for j in range(2):
                if j < count:
                    lst.append(torch.view_as_complex(flat[off:off + 2 * r * c].view(r, c, 2)))
                off += 2 * r * c
            setattr(p, name, lst)
        return p


@dataclass
class LocalFactors:
    """Per-rank retained elimination data (dist.py:134-151), device tensors."""

    kind: str
    lo: int
    hi: int
    mode: str
    tensors: dict = field(default_factory=dict)
    work_a: object = None
    work_b: object = None

    def eliminated(self) -> range:
        """Global indices of the blocks this partition eliminated."""
        lo, hi = self.lo, self.hi
        return {"first": range(lo, hi - 1), "last": range(lo + 1, hi), "middle": range(lo + 1, hi - 1)}[self.kind]

    @property
    def s_a(self) -> dict:
        """{global block index: inverted pivot} like the reference's
        LocalFactors.s_a (dist.py:134-151); device tensors (views)."""
        t = self.tensors.get("s_a")
        return {g: t[g - self.lo] for g in self.eliminated()} if t is not None else {}

    def desc(self) -> _native.LocalFactors:
        f = _native.LocalFactors()
        f.lo, f.hi, f.kind, f.fused = self.lo, self.hi, _KIND_CODES[self.kind], int(self.mode == "siq")
        for k in ("s_a", "s_b", "fill_row", "fill_col", "b_fill_row", "b_fill_col", "elim_f", "elim_g", "elim_q",
                  "elim_k", "elim_fr", "elim_qr", "elim_h", "elim_ha", "elim_eq", "elim_ek"):
            t = self.tensors.get(k)
            setattr(f, k, t.data_ptr() if (t is not None and t.numel()) else None)
        return f


@dataclass
class ReducedSystem:
    """The boundary-coupling system, replicated on every rank (dist.py:154-169)."""

    matrix_a: DeviceBta
    matrix_b: DeviceBta | None
    provenance: list
    index: dict
    # backward path for the quadratic solve decided from every rank's check of
    # B: +1 / -1 when B = +-B^H exactly, 0 otherwise (Context.set_b_symmetry)
    b_symmetry: int = 0

    def to_host(self) -> "ReducedSystem":
        """Host BtaMatrix form (the reference's ReducedSystem types)."""
        host = lambda m: m if (m is None or not isinstance(m, DeviceBta)) else to_host(m)  # noqa: E731
        return ReducedSystem(matrix_a=host(self.matrix_a), matrix_b=host(self.matrix_b), provenance=self.provenance,
                             index=self.index, b_symmetry=self.b_symmetry)


class _Strips:
    """Partition working arrays: diag / arrow strips (+ tip contribution)."""

    def __init__(self, length, b, a, device):
        c128 = dict(dtype=torch.complex128, device=device)
        self.n, self.b, self.a = length, b, a
        self.diag = torch.empty((length, b, b), **c128)
        self.arrow_row = torch.empty((length, a, b), **c128)
        self.arrow_col = torch.empty((length, b, a), **c128)
        self.tip = torch.zeros((a, a), **c128)

    def desc(self) -> _native.Bta:
        d = _native.Bta()
        d.n, d.b, d.a = self.n, self.b, self.a
        for k in ("diag", "arrow_row", "arrow_col", "tip"):
            t = getattr(self, k)
            setattr(d, k, t.data_ptr() if t.numel() else None)
        return d


# ---------------------------------------------------------------------------
# Phases
# ---------------------------------------------------------------------------


def _as_device(m, device=None):
    if m is None or isinstance(m, DeviceBta):
        return m
    return to_device(m, device)


def _alloc_factors(kind, lo, hi, fused, bs, asz, dev) -> "LocalFactors":
    length = hi - lo
    c128 = dict(dtype=torch.complex128, device=dev)
    t = {"s_a": torch.empty((length, bs, bs), **c128)}
    # elimination products retained for the backward (bsel_local_factors_t)
    t["elim_f"] = torch.empty((length, bs, bs), **c128)
    t["elim_g"] = torch.empty((length, asz, bs), **c128)
    t["elim_h"] = torch.empty((length, bs, bs), **c128)
    # steps.cuh fwd_backward_products; middle partitions always form them
    extra = os.environ.get("BSEL_FWD_BWD_PRODUCTS", "0") not in ("", "0") or kind == "middle"
    if extra or not fused:
        t["elim_ha"] = torch.empty((length, bs, asz), **c128)
    if fused:
        t["s_b"] = torch.empty((length, bs, bs), **c128)
        t["elim_q"] = torch.empty((length, bs, bs), **c128)
        t["elim_k"] = torch.empty((length, bs, asz), **c128)
        if extra:
            t["elim_eq"] = torch.empty((length, bs, bs), **c128)
            t["elim_ek"] = torch.empty((length, bs, asz), **c128)
    if kind == "middle":
        t["fill_row"] = torch.empty((length, bs, bs), **c128)
        t["fill_col"] = torch.empty((length, bs, bs), **c128)
        t["elim_fr"] = torch.empty((length, bs, bs), **c128)
        if fused:
            t["b_fill_row"] = torch.empty((length, bs, bs), **c128)
            t["b_fill_col"] = torch.empty((length, bs, bs), **c128)
            t["elim_qr"] = torch.empty((length, bs, bs), **c128)
    return LocalFactors(kind=kind, lo=lo, hi=hi, mode="siq" if fused else "si", tensors=t,
                        work_a=_Strips(length, bs, asz, dev), work_b=_Strips(length, bs, asz, dev) if fused else None)


def local_forward(a, b, plan: PartitionPlan, rank: int, counter: OpCounter | None = None, *, _factors=None,
                  _ctx=None, _sync=None):
    """Eliminate one partition's interior blocks on the GPU (dist.py:172-416).

    Returns ``(payload, tip_delta, factors)``; inputs are never mutated.
    """
    A = _as_device(a)
    B = _as_device(b, A.device) if b is not None else None
    lo, hi = plan.ranges[rank]
    kind = plan.kinds[rank]
    fused = B is not None
    n, bs, asz = A.shape_params
    length = hi - lo
    dev = A.device
    fac = _factors or _alloc_factors(kind, lo, hi, fused, bs, asz, dev)
    WA, WB = fac.work_a, fac.work_b
    ctx = _ctx or _native.Context.get(dev.index)
    ad, wad, fd = A.desc(), WA.desc(), fac.desc()
    bd = B.desc() if fused else None
    wbd = WB.desc() if fused else None
    ctx.bind_stream()
    ctx.call("bsel_local_forward", ctypes.byref(ad), ctypes.byref(bd) if fused else None, ctypes.byref(wad),
             ctypes.byref(wbd) if fused else None, ctypes.byref(fd), ctypes.byref(_sync) if _sync else None)
    record_partition(counter, kind, length, bs, asz, fac.mode, "forward")
    bnd = {"first": [hi - 1], "last": [lo], "middle": [lo, hi - 1]}[kind]
    pay = BoundaryPayload(rank=rank, kind=kind, b=bs, a=asz, fused=fused,
                          sym_flags=ctx.b_symmetry()[0] if fused else 3)
    pay.diag = [WA.diag[g - lo] for g in bnd]
    pay.arrow_row = [WA.arrow_row[g - lo] for g in bnd]
    pay.arrow_col = [WA.arrow_col[g - lo] for g in bnd]
    if kind == "middle":
        pay.coupling = [fac.tensors["fill_row"][length - 1], fac.tensors["fill_col"][length - 1]]
    if fused:
        pay.b_diag = [WB.diag[g - lo] for g in bnd]
        pay.b_arrow_row = [WB.arrow_row[g - lo] for g in bnd]
        pay.b_arrow_col = [WB.arrow_col[g - lo] for g in bnd]
        if kind == "middle":
            pay.b_coupling = [fac.tensors["b_fill_row"][length - 1], fac.tensors["b_fill_col"][length - 1]]
    tip_delta = torch.stack([WA.tip, WB.tip]) if fused else WA.tip.unsqueeze(0)
    if not isinstance(a, DeviceBta):
        # host inputs -> host payload / tip delta (reference types); the
        # factors stay on the device for local_backward
        return pay.to_host(), _np(tip_delta), fac
    return pay, tip_delta, fac


def _assemble(gathered, a, b, plan: PartitionPlan, tip_sum, dev=None) -> ReducedSystem:
    """Reduced system from all payloads (dist.py:440-504), on device ``dev``
    (payload blocks may be device tensors or host arrays)."""
    fused = b is not None
    if len(gathered) != plan.num_parts:
        raise ProtocolError(f"expected {plan.num_parts} payloads, got {len(gathered)}")
    prov, d, r, c, bd, br, bc = [], [], [], [], [], [], []
    for p, pay in enumerate(gathered):
        if pay.rank != p or pay.kind != plan.kinds[p]:
            raise ProtocolError(f"payload {p} carries rank {pay.rank} kind {pay.kind!r}")
        expected = 2 if pay.kind == "middle" else 1
        if len(pay.diag) != expected or (fused and len(pay.b_diag) != expected):
            raise ProtocolError(f"payload {p} has malformed boundary blocks")
        if pay.kind == "middle" and (len(pay.coupling) != 2 or (fused and len(pay.b_coupling) != 2)):
            raise ProtocolError(f"payload {p} lacks its fill-in coupling pair")
        sides = {"first": ("bottom",), "last": ("top",), "middle": ("top", "bottom")}[pay.kind]
        for j, side in enumerate(sides):
            prov.append((p, side))
            d.append(pay.diag[j])
            r.append(pay.arrow_row[j])
            c.append(pay.arrow_col[j])
            if fused:
                bd.append(pay.b_diag[j])
                br.append(pay.b_arrow_row[j])
                bc.append(pay.b_arrow_col[j])
    nr = len(d)
    up, lw, bup, blw = [], [], [], []
    for k in range(nr - 1):
        p1, p2 = prov[k][0], prov[k + 1][0]
        if p1 == p2:
            up.append(gathered[p1].coupling[0])
            lw.append(gathered[p1].coupling[1])
            if fused:
                bup.append(gathered[p1].b_coupling[0])
                blw.append(gathered[p1].b_coupling[1])
        else:  # original separator owned by the upper-side rank
            g = plan.ranges[p1][1] - 1
            up.append(a.upper[g])
            lw.append(a.lower[g])
            if fused:
                bup.append(b.upper[g])
                blw.append(b.lower[g])
    asz, bs = a.a, a.b
    if dev is None:
        dev = d[0].device if isinstance(d[0], torch.Tensor) else torch.device("cuda", torch.cuda.current_device())

    def stack(lst, shape):
        if lst:
            return torch.stack([_dev_tensor(x, dev) for x in lst]).contiguous()
        return torch.empty((0,) + shape, dtype=torch.complex128, device=dev)

    flags = 0
    for pay in gathered:
        flags |= int(pay.sym_flags)
    sym = 0 if not fused else (1 if not flags & 1 else -1 if not flags & 2 else 0)
    if tip_sum is not None:
        tip_sum = _dev_tensor(tip_sum, dev)
    tip = (_dev_tensor(a.tip, dev) + tip_sum[0]) if asz else torch.empty((0, 0), dtype=torch.complex128, device=dev)
    ra = DeviceBta(nr, bs, asz, {"diag": stack(d, (bs, bs)), "lower": stack(lw, (bs, bs)),
                                 "upper": stack(up, (bs, bs)), "arrow_row": stack(r, (asz, bs)),
                                 "arrow_col": stack(c, (bs, asz)), "tip": tip.contiguous()})
    rb = None
    if fused:
        btip = (_dev_tensor(b.tip, dev) + tip_sum[1]) if asz else torch.empty((0, 0), dtype=torch.complex128,
                                                                             device=dev)
        rb = DeviceBta(nr, bs, asz, {"diag": stack(bd, (bs, bs)), "lower": stack(blw, (bs, bs)),
                                     "upper": stack(bup, (bs, bs)), "arrow_row": stack(br, (asz, bs)),
                                     "arrow_col": stack(bc, (bs, asz)), "tip": btip.contiguous()})
    return ReducedSystem(matrix_a=ra, matrix_b=rb, provenance=prov, index={key: k for k, key in enumerate(prov)},
                         b_symmetry=sym)


def assemble_reduced(coll: Collectives, a, b, plan: PartitionPlan, payload: BoundaryPayload,
                     tip_delta) -> ReducedSystem:
    """Exchange boundary data and build the replicated reduced system
    (dist.py:419-504): one all_gather, plus one all_reduce when a > 0.

    ``coll``: a TorchCollectives endpoint (device payload slots over NCCL)
    or any other Collectives (the reference's ThreadHub endpoints /
    SocketCollectives): those receive host payloads and a numpy tip delta,
    by value, as in the reference.  Host inputs give a host ReducedSystem.
    """
    if _native_transport(coll):
        gathered = coll.all_gather(payload)
        tip_sum = coll.all_reduce_sum(tip_delta) if a.a > 0 else None
    else:
        host_pay = payload.to_host() if isinstance(payload, BoundaryPayload) and payload.on_device() else payload
        gathered = coll.all_gather(host_pay)
        tip_sum = coll.all_reduce_sum(_np(tip_delta)) if a.a > 0 else None
    dev = a.device if isinstance(a, DeviceBta) else torch.device("cuda", torch.cuda.current_device())
    reduced = _assemble(gathered, a, b, plan, tip_sum, dev)
    return reduced if isinstance(a, DeviceBta) else reduced.to_host()


def solve_reduced(reduced: ReducedSystem, mode: str, counter=None, recursive_parts=None, *, _pipe=0):
    """Solve the replicated reduced system (dist.py:507-523) on the GPU."""
    if recursive_parts and reduced.matrix_a.n >= 2 * recursive_parts:
        return dist_solve(reduced.matrix_a, reduced.matrix_b, num_parts=recursive_parts, mode=mode)
    return solve_selected(reduced.matrix_a, reduced.matrix_b if mode == "siq" else None, mode, counter=counter,
                          _b_symmetry=reduced.b_symmetry, _pipe=_pipe)


def local_backward(a, b, plan: PartitionPlan, rank: int, factors: LocalFactors, reduced: ReducedSystem,
                   red_sol: SelectedSolution, counter=None, *, out=None, _ctx=None, _sync=None):
    """Back-substitute one partition seeded with the reduced solution
    (dist.py:542-744).  Writes this rank's pattern blocks (and, on rank 0,
    the tip) into ``out`` = (x_a, x_b) full-size DeviceBta (allocated zeroed
    if None) and returns it."""
    host = not isinstance(a, DeviceBta)
    A = _as_device(a)
    B = _as_device(b, A.device) if b is not None else None
    lo, hi = plan.ranges[rank]
    fused = factors.mode == "siq"
    if fused and B is None:
        raise ProtocolError("fused factors require the right-hand side")
    if not isinstance(red_sol.x_a, DeviceBta):  # host reduced solution (reference types)
        red_sol = SelectedSolution(x_a=to_device(red_sol.x_a, A.device),
                                   x_b=to_device(red_sol.x_b, A.device) if red_sol.x_b is not None else None,
                                   mode=red_sol.mode)
    if red_sol.x_a.shape_params != reduced.matrix_a.shape_params:
        raise ProtocolError("reduced solution shape disagrees with reduced system")
    n, bs, asz = A.shape_params
    if out is None:
        out = (DeviceBta.empty(n, bs, asz, A.device), DeviceBta.empty(n, bs, asz, A.device) if fused else None)
    XA, XB = out
    kind = plan.kinds[rank]
    k_top = reduced.index.get((rank, "top"), -1)
    k_bot = reduced.index.get((rank, "bottom"), -1)
    ctx = _ctx or _native.Context.get(A.device.index)
    ad, fd, wad = A.desc(), factors.desc(), factors.work_a.desc()
    xrd, xad = red_sol.x_a.desc(), XA.desc()
    bd = B.desc() if fused else None
    wbd = factors.work_b.desc() if fused else None
    zrd = red_sol.x_b.desc() if fused else None
    xbd = XB.desc() if fused else None
    ref = lambda x: ctypes.byref(x) if x is not None else None  # noqa: E731
    ctx.bind_stream()
    ctx.set_b_symmetry(reduced.b_symmetry)
    try:
        ctx.call("bsel_local_backward", ref(ad), ref(bd), ref(fd), ref(wad), ref(wbd), ref(xrd), ref(zrd),
                 k_top, k_bot, int(rank == 0), ref(xad), ref(xbd), ref(_sync))
    finally:
        ctx.set_b_symmetry(ctx.SYM_AUTO)
    record_partition(counter, kind, hi - lo, bs, asz, factors.mode, "backward")
    if host:
        return owned_slices(out, plan, rank)
    return out


def owned_slices(out, plan: PartitionPlan, rank: int) -> dict:
    """Host slice of the blocks partition ``rank`` owns, in the reference's
    local_backward return form (dist.py:551-560): ``{"x_a": {kind: {g: blk}},
    "x_b": ... | None}`` -- its diagonal blocks and arrow strips, its interior
    off-diagonals and (except the last rank) its separator, and on rank 0
    the tip."""
    lo, hi = plan.ranges[rank]
    last = rank == plan.num_parts - 1
    offd = range(lo, hi - 1 if last else hi)

    def one(X):
        if X is None:
            return None
        h = {k: _np(getattr(X, k)[lo:hi]) for k in ("diag", "arrow_row", "arrow_col")}
        o = {k: _np(getattr(X, k)[offd.start:offd.stop]) for k in ("lower", "upper")}
        sl = {k: {g: h[k][g - lo] for g in range(lo, hi)} for k in h}
        sl.update({k: {g: o[k][g - offd.start] for g in offd} for k in o})
        sl["tip"] = _np(X.tip) if rank == 0 else None
        return sl

    return {"x_a": one(out[0]), "x_b": one(out[1])}


def merge_slices(n, b, a, mode, slices) -> SelectedSolution:
    """Host solution from every rank's owned slices (dist.py:752-780)."""
    fused = mode == "siq"
    xs = {"x_a": BtaMatrix.zeros(n, b, a), "x_b": BtaMatrix.zeros(n, b, a) if fused else None}
    seen = set()
    for sl in slices:
        seen.update(sl["x_a"]["diag"].keys())
        for side, m in xs.items():
            if m is None:
                continue
            part = sl[side]
            for kind in ("diag", "lower", "upper", "arrow_row", "arrow_col"):
                for g, blk in part[kind].items():
                    getattr(m, kind)[g][...] = blk
            if part["tip"] is not None:
                m.tip[...] = part["tip"]
    if seen != set(range(n)):
        raise ProtocolError(f"incomplete solution coverage: missing {sorted(set(range(n)) - seen)}")
    return SelectedSolution(x_a=xs["x_a"], x_b=xs["x_b"], mode=mode)


def _slices_to_bytes(sl: dict) -> bytes:
    import io

    arrays = {}
    for side in ("x_a", "x_b"):
        part = sl[side]
        if part is None:
            continue
        for kind, blocks in part.items():
            if kind == "tip":
                if blocks is not None:
                    arrays[f"{side}/tip/0"] = blocks
                continue
            for g, blk in blocks.items():
                arrays[f"{side}/{kind}/{g}"] = blk
    buf = io.BytesIO()
    np.savez(buf, **arrays)
    return buf.getvalue()


def _slices_from_bytes(blob: bytes, fused: bool) -> dict:
    import io

    z = np.load(io.BytesIO(blob))
    sl = {"x_a": None, "x_b": None}
    for side in ("x_a", "x_b") if fused else ("x_a",):
        sl[side] = {k: {} for k in ("diag", "lower", "upper", "arrow_row", "arrow_col")}
        sl[side]["tip"] = None
    for key in z.files:
        side, kind, g = key.split("/")
        if kind == "tip":
            sl[side]["tip"] = z[key]
        else:
            sl[side][kind][int(g)] = z[key]
    return sl


# ---------------------------------------------------------------------------
# Facade
# ---------------------------------------------------------------------------


class _Lanes:
    """Run one callable per partition concurrently on one GPU: each partition
    gets its own native context (lane) and CUDA stream and runs in its own
    thread; the lanes start after, and the caller's stream waits for, all
    work previously queued on the caller's stream."""

    def __init__(self, device, count, base=0):
        self.device = device
        self.count = count
        self.base = base  # lane contexts base .. base + count - 1 (concurrent runners use disjoint lanes)
        self.streams = [torch.cuda.Stream(device) for _ in range(count)]
        # Concurrent chains share the SMs: each block inverse gets fewer CTAs
        # (cfg4, 2 lanes, current sweeps: 32 / 36 / 40 / 44 / 48 / 64 CTAs ->
        # 1070 / 1045 / 1019-1023 / 1028 / 1035 / 1060 ms per energy point).
        self.inverse_grid = int(os.environ.get("BSEL_LANE_INV_GRID", "40")) if count > 1 else 0
        # SMs the lanes' forward aux levels leave to the chains (experiment; 0 = off)
        self.avoid_sms = int(os.environ.get("BSEL_LANE_AVOID_SMS", "0"))

    def run(self, fn) -> list:
        import threading

        main = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(main)
        errors = []

        def work(rank):
            try:
                with torch.cuda.device(self.device), torch.cuda.stream(self.streams[rank]):
                    self.streams[rank].wait_event(start)
                    ctx = _native.Context.get(self.device.index, lane=self.base + rank)
                    ctx.set_inverse_grid(self.inverse_grid)
                    ctx.set_aux_avoid_sms(self.avoid_sms)
                    try:
                        fn(rank, ctx)
                    finally:
                        ctx.set_inverse_grid(0)
                        ctx.set_aux_avoid_sms(0)
            except Exception as exc:  # noqa: BLE001 - rank attribution
                errors.append((rank, exc))

        threads = [threading.Thread(target=work, args=(r,)) for r in range(self.count)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for s in self.streams:
            main.wait_stream(s)
        return errors


class HostWindow:
    """Pinned host storage for the blocks of a full-size BTA matrix that ONE
    rank of the distributed solve touches: its partition's diagonal / arrow
    blocks and couplings, the separators of the other partitions (the
    replicated reduced system needs them) and the tip.  Its descriptor
    (``desc()``) addresses blocks by their GLOBAL index, so it can stand in
    for a full-size host matrix in ``DistSolver.solve`` without pinning the
    whole matrix on every rank (only the window's blocks are ever touched)."""

    def __init__(self, n, b, a, lo, hi, separators=()):
        self.n, self.b, self.a, self.lo, self.hi = n, b, a, lo, hi
        self.c_hi = min(hi, n - 1)
        pin = dict(dtype=torch.complex128, pin_memory=torch.cuda.is_available())
        self.diag = torch.empty((hi - lo, b, b), **pin)
        self.arrow_row = torch.empty((hi - lo, a, b), **pin)
        self.arrow_col = torch.empty((hi - lo, b, a), **pin)
        self.lower = torch.empty((max(self.c_hi - lo, 0), b, b), **pin)
        self.upper = torch.empty((max(self.c_hi - lo, 0), b, b), **pin)
        self.tip = torch.empty((a, a), **pin)
        self.separators = {g: (torch.empty((b, b), **pin), torch.empty((b, b), **pin))
                           for g in separators if not lo <= g < self.c_hi}

    @property
    def shape_params(self):
        return self.n, self.b, self.a

    def fill_from(self, m: DeviceBta, *, non_blocking=False, tip=True) -> "HostWindow":
        """Copy the window's blocks out of a full-size device matrix."""
        lo, hi, c = self.lo, self.hi, self.c_hi
        nb = dict(non_blocking=non_blocking)
        self.diag.copy_(m.diag[lo:hi], **nb)
        self.arrow_row.copy_(m.arrow_row[lo:hi], **nb)
        self.arrow_col.copy_(m.arrow_col[lo:hi], **nb)
        if c > lo:
            self.lower.copy_(m.lower[lo:c], **nb)
            self.upper.copy_(m.upper[lo:c], **nb)
        if tip:
            self.tip.copy_(m.tip, **nb)
        for g, (lw, up) in self.separators.items():
            lw.copy_(m.lower[g], **nb)
            up.copy_(m.upper[g], **nb)
        return self

    def copy_to(self, m: DeviceBta) -> DeviceBta:
        """Copy the window's blocks into a full-size device matrix (current
        stream, asynchronous: the window is pinned)."""
        lo, hi, c = self.lo, self.hi, self.c_hi
        m.diag[lo:hi].copy_(self.diag, non_blocking=True)
        m.arrow_row[lo:hi].copy_(self.arrow_row, non_blocking=True)
        m.arrow_col[lo:hi].copy_(self.arrow_col, non_blocking=True)
        if c > lo:
            m.lower[lo:c].copy_(self.lower, non_blocking=True)
            m.upper[lo:c].copy_(self.upper, non_blocking=True)
        m.tip.copy_(self.tip, non_blocking=True)
        for g, (lw, up) in self.separators.items():
            m.lower[g].copy_(lw, non_blocking=True)
            m.upper[g].copy_(up, non_blocking=True)
        return m

    def separator(self, g):
        if self.lo <= g < self.c_hi:
            return self.lower[g - self.lo], self.upper[g - self.lo]
        return self.separators[g]

    def desc(self) -> _native.Bta:
        d = _native.Bta()
        d.n, d.b, d.a = self.n, self.b, self.a
        for k in ("diag", "arrow_row", "arrow_col", "lower", "upper"):
            t = getattr(self, k)
            per = t[0].numel() * 16 if t.numel() else 0
            # global block g lives at base + (g - lo) * per
            setattr(d, k, (t.data_ptr() - self.lo * per) if t.numel() else None)
        d.tip = self.tip.data_ptr() if self.tip.numel() else None
        return d

    @property
    def nbytes(self):
        ts = [self.diag, self.arrow_row, self.arrow_col, self.lower, self.upper, self.tip]
        ts += [x for pair in self.separators.values() for x in pair]
        return sum(t.numel() * 16 for t in ts)


def _host_io(chunk, a=None, b=None, x_a=None, x_b=None, copy_tip=False, stream=None):
    """bsel_host_io_t for local_forward / local_backward end-to-end mode
    (the descriptors are kept alive on the returned struct)."""
    io = _native.HostIo()
    keep = []
    for k, m in (("a", a), ("b", b), ("x_a", x_a), ("x_b", x_b)):
        if m is not None:
            d = m.desc() if isinstance(m, HostWindow) else _native.host_desc(m)
            keep.append(d)
            setattr(io, k, ctypes.pointer(d))
    io.chunk_blocks = int(chunk)
    io.copy_tip = int(bool(copy_tip))
    io.copy_stream = stream.cuda_stream if stream is not None else None
    io._keep = keep
    return io


class InGpuPartitions:
    """The paper's partitioned scheme with every partition on ONE GPU, the
    partitions running concurrently (one lane = native context + stream +
    thread each).  With 2 partitions (first + last, no middle-partition work
    inflation) the two Schur chains run side by side, which fills the SMs the
    latency-bound chain of a single sweep leaves idle.  Factor buffers are
    kept between runs for repeated solves of one shape."""

    def __init__(self, shape, mode, parts, device, plan=None, local=None, lane_base=0, pipe=0):
        """``local``: the partition indices this process runs (default: all
        ``parts``, the single-GPU scheme); with a subset -- k partitions per
        GPU of a multi-GPU job -- ``run`` needs a hub that exchanges with the
        other ranks (_RankHub)."""
        self.n, self.b, self.a = shape
        self.mode = mode
        self.parts = parts
        self.device = device
        self.plan = plan or plan_partitions(self.n, parts, mode)
        self.local = list(range(parts)) if local is None else list(local)
        self.lanes = _Lanes(device, len(self.local), base=lane_base)
        self.pipe = pipe  # the reduced solve's context (concurrent runners: disjoint)
        self._factors = [None] * len(self.local)
        self.chunk = None
        self.copy_stream = torch.cuda.Stream(device)  # shared by the partitions' input chunks
        self.counters = []
        self.reduced = None
        self._tm = None

    def run(self, A, B, out=None, hub=None, recursive_parts=None, host_in=None, host_out=None):
        """One solve.  ``host_in`` = (a, b) host BtaMatrix (pinned for full
        overlap): the inputs are streamed in chunk by chunk behind the
        forward sweeps instead of being resident in A/B beforehand (A/B then
        only provide device storage for the couplings and the tip);
        ``host_out`` = (x_a, x_b) host BtaMatrix receiving the solution,
        streamed out behind the backward sweeps."""
        st = self.run_forward(A, B, hub=hub, recursive_parts=recursive_parts, host_in=host_in)
        return self.run_backward(st, out=out, host_out=host_out)

    def run_forward(self, A, B, hub=None, recursive_parts=None, host_in=None) -> dict:
        """Forward half of ``run``: the partitions' eliminations, the exchange
        and the reduced solve.  Returns the state ``run_backward`` consumes;
        this runner's factor buffers stay in use until that backward ran
        (EnergySweep overlaps one energy's backward with the next energy's
        forward on a second runner).  Blocks the host until the reduced
        solve is done."""
        plan, parts, mode = self.plan, self.parts, self.mode
        B = B if mode == "siq" else None
        # Chunk of the host transfers (blocks): small enough that the first
        # chunk arrives fast, large enough to amortise the copy calls.
        chunk = self.chunk or int(os.environ.get("BSEL_STREAM_CHUNK", "8"))
        hub = hub or LocalHub(parts)
        tm = _PhaseTimer(("forward", "communication", "reduced", "backward"))
        loc = self.local
        self.counters = counters = [OpCounter(b=A.b, a=A.a) for _ in loc]
        results = [None] * len(loc)
        tm.start("forward")

        def fwd(lane, ctx):
            rank = loc[lane]
            sync = None
            if host_in is not None:
                sync = _host_io(chunk, a=host_in[0], b=host_in[1] if B is not None else None,
                                copy_tip=rank == loc[0], stream=self.copy_stream)
            results[lane] = local_forward(A, B, plan, rank, counters[lane], _factors=self._factors[lane], _ctx=ctx,
                                          _sync=sync)
            self._factors[lane] = results[lane][2]

        errors = self.lanes.run(fwd)
        tm.stop("forward")
        if errors:
            primary = [e for e in errors if not isinstance(e[1], ProtocolError)]
            lane, exc = min(primary or errors, key=lambda e: e[0])
            raise WorkerError(loc[lane], exc) from exc
        tm.start("communication")
        gathered = hub.all_gather_all([r[0] for r in results])
        tip_sum = hub.all_reduce_all([r[1] for r in results]) if A.a > 0 else None
        self.reduced = reduced = _assemble(gathered, A, B, plan, tip_sum)
        tm.stop("communication")
        tm.start("reduced")
        red_sol = solve_reduced(reduced, mode, None, recursive_parts, _pipe=self.pipe)
        tm.stop("reduced")
        return {"A": A, "B": B, "results": results, "reduced": reduced, "red_sol": red_sol, "tm": tm,
                "counters": counters, "chunk": chunk}

    def run_backward(self, st: dict, out=None, host_out=None):
        """Backward half of ``run`` (enqueues the back-substitutions; returns
        without waiting for the GPU)."""
        A, B, results, tm, loc = st["A"], st["B"], st["results"], st["tm"], self.local
        tm.start("backward")
        if out is None:
            out = (DeviceBta.empty(A.n, A.b, A.a, self.device),
                   DeviceBta.empty(A.n, A.b, A.a, self.device) if B is not None else None)
        io_out = None
        if host_out is not None:
            io_out = _host_io(st["chunk"], x_a=host_out[0], x_b=host_out[1] if B is not None else None)
        errors = self.lanes.run(lambda lane, ctx: local_backward(
            A, B, self.plan, loc[lane], results[lane][2], st["reduced"], st["red_sol"], st["counters"][lane],
            out=out, _ctx=ctx, _sync=io_out))
        if errors:
            lane, exc = min(errors, key=lambda e: e[0])
            raise WorkerError(loc[lane], exc) from exc
        tm.stop("backward")
        self._tm = tm
        return out

    def phase_seconds(self):
        return self._tm.seconds()


class _PhaseTimer:
    def __init__(self, names):
        self.ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in names}

    def start(self, k):
        self.ev[k][0].record()

    def stop(self, k):
        self.ev[k][1].record()

    def seconds(self):
        torch.cuda.synchronize()
        return {k: s.elapsed_time(e) / 1e3 for k, (s, e) in self.ev.items()}


def _reduced_counts(reduced, mode):
    c = OpCounter(b=reduced.matrix_a.b, a=reduced.matrix_a.a)
    record_sweep(c, reduced.matrix_a.n, reduced.matrix_a.b, reduced.matrix_a.a, mode, "forward")
    record_sweep(c, reduced.matrix_a.n, reduced.matrix_a.b, reduced.matrix_a.a, mode, "backward")
    return c


def dist_solve(a, b=None, num_parts=2, mode=None, transport=None, *, counter=None, timings=None,
               rank_counters=None, recursive_parts=None, gather=True):
    """Distributed selected solve (dist.py:804-896).

    ``transport=None`` (or a LocalHub): every partition runs on the current
    GPU in this process and the full solution is returned.  A
    ``TorchCollectives`` endpoint makes this process one rank of a
    one-process-per-GPU job: with ``gather`` rank 0 returns the merged
    solution and other ranks None; without, every rank returns its sharded
    (zero-elsewhere) device solution.  ``num_parts=1`` delegates to
    ``solve_selected``.
    """
    if mode is None:
        mode = "si" if b is None else "siq"
    if mode == "siq" and b is None:
        raise ValueError("mode 'siq' requires a right-hand side")
    if mode == "si":
        b = None
    if num_parts == 1:
        return solve_selected(a, b, mode, counter=counter, timings=timings)
    host = not isinstance(a, DeviceBta)
    plan = plan_partitions(a.n, num_parts, mode)
    if isinstance(transport, TorchCollectives):
        if transport.world_size != num_parts:
            raise ProtocolError(f"transport world size {transport.world_size} != num_parts {num_parts}")
        dev = torch.device("cuda", torch.cuda.current_device())
        A = _as_device(a, dev)
        B = _as_device(b, dev) if b is not None else None
        rank = transport.rank
        tm = _PhaseTimer(("forward", "communication", "reduced", "backward"))
        cnt = OpCounter(b=A.b, a=A.a)
        try:
            tm.start("forward")
            ctx = _native.Context.get(dev.index)
            ctx.set_aux_avoid_sms(AUX_AVOID_SMS)
            try:
                pay, delta, fac = local_forward(A, B, plan, rank, cnt, _ctx=ctx)
            finally:
                ctx.set_aux_avoid_sms(0)
            tm.stop("forward")
        except Exception as exc:  # rank attribution (dist.py:875-885)
            raise WorkerError(rank, exc) from exc
        tm.start("communication")
        reduced = assemble_reduced(transport, A, B, plan, pay, delta)
        tm.stop("communication")
        tm.start("reduced")
        red_sol = solve_reduced(reduced, mode, None, recursive_parts)
        tm.stop("reduced")
        tm.start("backward")
        XA, XB = local_backward(A, B, plan, rank, fac, reduced, red_sol, cnt)
        tm.stop("backward")
        if timings is not None:
            timings.update(tm.seconds())
        if counter is not None:
            counter.merge(cnt)
            if rank == 0:
                counter.merge(_reduced_counts(reduced, mode))
        if rank_counters is not None:
            rank_counters.append(cnt)
        if not gather:
            return SelectedSolution(x_a=XA, x_b=XB, mode=mode)
        import torch.distributed as tdist

        # pattern blocks are owned by exactly one rank (zeros elsewhere):
        # a sum-reduce to rank 0 is an exact merge.
        for m in (XA, XB) if XB is not None else (XA,):
            for t in m.tensors().values():
                if t.numel():
                    tdist.reduce(torch.view_as_real(t), dst=0, group=transport.group)
        if rank != 0:
            return None
        if host:
            return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if XB is not None else None, mode=mode)
        return SelectedSolution(x_a=XA, x_b=XB, mode=mode)

    if transport is not None and not isinstance(transport, LocalHub):
        if transport.world_size != num_parts:
            raise ProtocolError(f"transport world size {transport.world_size} != num_parts {num_parts}")
        if hasattr(transport, "endpoint"):
            return _solve_over_hub(a, b, plan, transport, mode, counter, timings, rank_counters, recursive_parts)
        return _solve_as_rank(a, b, plan, transport, mode, counter, timings, recursive_parts)

    hub = transport if transport is not None else LocalHub(num_parts)
    if hub.world_size != num_parts:
        raise ProtocolError(f"transport world size {hub.world_size} != num_parts {num_parts}")
    dev = a.device if isinstance(a, DeviceBta) else torch.device("cuda", torch.cuda.current_device())
    A = _as_device(a, dev)
    B = _as_device(b, dev) if b is not None else None
    runner = InGpuPartitions(A.shape_params, mode, num_parts, dev, plan=plan)
    out = runner.run(A, B, hub=hub, recursive_parts=recursive_parts)
    if timings is not None:
        timings.update(runner.phase_seconds())
    if counter is not None:
        for c in runner.counters:
            counter.merge(c)
        counter.merge(_reduced_counts(runner.reduced, mode))
    if rank_counters is not None:
        rank_counters.extend(runner.counters)
    XA, XB = out
    if host:
        return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if XB is not None else None, mode=mode)
    return SelectedSolution(x_a=XA, x_b=XB, mode=mode)


_REDUCED_LOCK = threading.Lock()


def _solve_over_hub(a, b, plan, hub, mode, counter, timings, rank_counters, recursive_parts):
    """dist_solve over a foreign in-process hub (``hub.endpoint(rank)``, e.g.
    the reference's ThreadHub, collectives.py:87-133): every rank is a lane
    on this GPU running the reference's per-rank pipeline (dist.py:787-801)
    -- local forward, exchange through its endpoint (host payloads by
    value), redundant reduced solve, local backward -- so the hub records
    exactly the reference's rounds."""
    num_parts = plan.num_parts
    host = not isinstance(a, DeviceBta)
    dev = a.device if not host else torch.device("cuda", torch.cuda.current_device())
    A = _as_device(a, dev)
    B = _as_device(b, dev) if b is not None else None
    out = (DeviceBta.empty(A.n, A.b, A.a, dev), DeviceBta.empty(A.n, A.b, A.a, dev) if B is not None else None)
    cnts = [OpCounter(b=A.b, a=A.a) for _ in range(num_parts)]
    red_cnt = OpCounter(b=A.b, a=A.a)
    timers = [None] * num_parts

    def work(rank, ctx):
        try:
            tm = timers[rank] = _PhaseTimer(("forward", "communication", "reduced", "backward"))
            tm.start("forward")
            pay, delta, fac = local_forward(A, B, plan, rank, cnts[rank], _ctx=ctx)
            tm.stop("forward")
            tm.start("communication")
            reduced = assemble_reduced(hub.endpoint(rank), A, B, plan, pay, delta)
            tm.stop("communication")
            tm.start("reduced")
            with _REDUCED_LOCK:  # the reduced solves share the device's default context
                red_sol = solve_reduced(reduced, mode, red_cnt if rank == 0 else None, recursive_parts)
                torch.cuda.current_stream().synchronize()
            tm.stop("reduced")
            tm.start("backward")
            local_backward(A, B, plan, rank, fac, reduced, red_sol, cnts[rank], out=out, _ctx=ctx)
            tm.stop("backward")
        except BaseException:
            abort = getattr(hub, "abort", None)
            if abort is not None:
                abort()  # release peers blocked inside a collective round
            raise

    errors = _Lanes(dev, num_parts).run(work)
    if errors:
        primary = [e for e in errors if not isinstance(e[1], ProtocolError)]
        rank, exc = min(primary or errors, key=lambda e: e[0])
        raise WorkerError(rank, exc) from exc
    if counter is not None:
        for c in cnts:
            counter.merge(c)
        counter.merge(red_cnt)
    if rank_counters is not None:
        rank_counters.extend(cnts)
    if timings is not None:
        timings.update(timers[0].seconds())
    XA, XB = out
    if host:
        return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if XB is not None else None, mode=mode)
    return SelectedSolution(x_a=XA, x_b=XB, mode=mode)


def _solve_as_rank(a, b, plan, coll, mode, counter, timings, recursive_parts):
    """dist_solve as ONE rank of a multi-process job over a foreign
    Collectives endpoint (e.g. the reference's SocketCollectives,
    collectives.py:187-331): this rank's partition on this process's GPU,
    host payloads on the wire; with ``gather_to_root`` rank 0 returns the
    merged host solution and the others None (dist.py:839-855), else every
    rank returns its sharded device solution."""
    rank = coll.rank
    dev = torch.device("cuda", torch.cuda.current_device())
    A = _as_device(a, dev)
    B = _as_device(b, dev) if b is not None else None
    cnt, red_cnt = OpCounter(b=A.b, a=A.a), OpCounter(b=A.b, a=A.a)
    tm = _PhaseTimer(("forward", "communication", "reduced", "backward"))
    tm.start("forward")
    pay, delta, fac = local_forward(A, B, plan, rank, cnt)
    tm.stop("forward")
    tm.start("communication")
    reduced = assemble_reduced(coll, A, B, plan, pay, delta)
    tm.stop("communication")
    tm.start("reduced")
    red_sol = solve_reduced(reduced, mode, red_cnt, recursive_parts)
    tm.stop("reduced")
    tm.start("backward")
    out = local_backward(A, B, plan, rank, fac, reduced, red_sol, cnt)
    tm.stop("backward")
    if timings is not None:
        timings.update(tm.seconds())
    if counter is not None:
        counter.merge(cnt)
        if rank == 0:
            counter.merge(red_cnt)
    if not hasattr(coll, "gather_to_root"):
        return SelectedSolution(x_a=out[0], x_b=out[1], mode=mode)
    blobs = coll.gather_to_root(_slices_to_bytes(owned_slices(out, plan, rank)))
    if rank != 0 or blobs is None:
        return None
    fused = B is not None
    return merge_slices(A.n, A.b, A.a, mode, [_slices_from_bytes(bl, fused) for bl in blobs])


# SMs the forward's throughput GEMM levels leave to a single lane's chain.
# Round 1 (real-embedding GEMM): 32 helped (n=512 one lane: forward 343 ->
# 322 ms).  Round 2 (persistent 3M TMA GEMM): 0 is best (2 GPUs 496 vs 520 ms,
# 4 GPUs 352 vs 369 ms; profiles/sweeps_r02.md).
AUX_AVOID_SMS = int(os.environ.get("BSEL_AUX_AVOID_SMS", "0"))


class _RankHub:
    """The exchange of k partitions per rank over a TorchCollectives endpoint
    (InGpuPartitions with ``local``): this rank's k payload slots travel in
    ONE NCCL all_gather (rank-major = partition order), the k tip deltas are
    summed locally in partition order and then across ranks in rank order
    (one rank-ordered all_reduce): still exactly one all_gather + one
    all_reduce per solve (test_acceptance.py:201-243)."""

    def __init__(self, coll: TorchCollectives, k: int):
        self.coll, self.k = coll, k
        self.world_size = coll.world_size * k

    def all_gather_all(self, payloads: list) -> list:
        if len(payloads) != self.k:
            raise ProtocolError(f"expected {self.k} local payloads, got {len(payloads)}")
        slot = payloads[0].slot_elems()
        allp = self.coll.gather_tensor(torch.cat([p.pack() for p in payloads])).view(-1, slot)
        hdrs = allp[:, :4].cpu().tolist()
        out = [payloads[0].unpack(allp[q], rank=q, header=hdrs[q]) for q in range(allp.shape[0])]
        self.coll._record("all_gather", [p.summary() for p in out])
        return out

    def all_reduce_all(self, arrays: list):
        total = arrays[0].clone()
        for part in arrays[1:]:
            total += part
        return self.coll.all_reduce_sum(total)


class DistSolver:
    """Repeated distributed solves of one energy point on this rank with all
    device buffers preallocated (the bench / multi-GPU production path).

    ``parts_per_rank`` = k: the plan has world x k partitions and this rank
    runs partitions [rank k, rank k + k) concurrently as lanes on its GPU
    (k Schur chains per GPU instead of one; e.g. the reference's 8-partition
    plan on 4 GPUs)."""

    def __init__(self, A: DeviceBta, B: DeviceBta | None, mode: str, world: int, rank: int, device,
                 transport: TorchCollectives | None = None, plan_costs=None, parts_per_rank: int = 1):
        self.A, self.B, self.mode = A, B if mode == "siq" else None, mode
        self.k = int(parts_per_rank)
        # plan_costs: per-block (end, middle) costs for the partition sizes
        # (default: the reference's plan, partition.py:52-90)
        self.plan = plan_partitions(A.n, world * self.k, mode, costs=plan_costs)
        self.rank = rank
        # the bench / production path publishes boundaries by NVLink peer stores
        # into symmetric memory (BSEL_SYMM_EXCHANGE=0: NCCL all_gather)
        self.coll = transport or TorchCollectives(symmetric=os.environ.get("BSEL_SYMM_EXCHANGE", "1") != "0")
        self.out = (DeviceBta.empty(A.n, A.b, A.a, device),
                    DeviceBta.empty(A.n, A.b, A.a, device) if self.B is not None else None)
        self._fac = None
        self.timings = {}
        self._runner = None
        if self.k > 1:
            local = list(range(rank * self.k, (rank + 1) * self.k))
            self._runner = InGpuPartitions(A.shape_params, mode, world * self.k, device, plan=self.plan, local=local)
            self._hub = _RankHub(self.coll, self.k)

    def owned_range(self):
        """[lo, hi) of the diagonal blocks this rank's partitions cover."""
        r = self.plan.ranges
        return r[self.rank * self.k][0], r[self.rank * self.k + self.k - 1][1]

    def solve(self, host_in=None, host_out=None):
        if self._runner is not None:
            if host_in is not None:
                self._copy_separators(host_in)
            out = self._runner.run(self.A, self.B, out=self.out, hub=self._hub, host_in=host_in, host_out=host_out)
            self._tm = self._runner._tm
            return out
        """One distributed solve.  ``host_in`` = (a, b) full-size pinned host
        BtaMatrix: this rank's partition streams in behind its forward sweep
        (plus the separators and tip every rank needs for the replicated
        reduced system); ``host_out`` = (x_a, x_b) full-size host BtaMatrix:
        the blocks this rank owns stream out behind its backward sweep."""
        chunk = int(os.environ.get("BSEL_STREAM_CHUNK", "8"))
        fused = self.B is not None
        io_in = io_out = None
        if host_in is not None:
            io_in = _host_io(chunk, a=host_in[0], b=host_in[1] if fused else None, copy_tip=True)
            self._copy_separators(host_in)
        if host_out is not None:
            io_out = _host_io(chunk, x_a=host_out[0], x_b=host_out[1] if fused else None)
        tm = _PhaseTimer(("forward", "communication", "reduced", "backward", "step"))
        tm.start("step")
        tm.start("forward")
        if self._fac is None:
            lo, hi = self.plan.ranges[self.rank]
            self._fac = _alloc_factors(self.plan.kinds[self.rank], lo, hi, fused, self.A.b, self.A.a,
                                       self.A.device)
        # one partition per GPU: its Schur chain is the forward's critical
        # path, so the throughput levels leave the inverse SMs of its own
        ctx = _native.Context.get(self.A.device.index)
        ctx.set_aux_avoid_sms(AUX_AVOID_SMS)
        try:
            pay, delta, self._fac = local_forward(self.A, self.B, self.plan, self.rank, _factors=self._fac,
                                                  _ctx=ctx, _sync=io_in)
        finally:
            ctx.set_aux_avoid_sms(0)
        tm.stop("forward")
        tm.start("communication")
        reduced = assemble_reduced(self.coll, self.A, self.B, self.plan, pay, delta)
        tm.stop("communication")
        tm.start("reduced")
        red_sol = solve_reduced(reduced, self.mode)
        tm.stop("reduced")
        tm.start("backward")
        local_backward(self.A, self.B, self.plan, self.rank, self._fac, reduced, red_sol, out=self.out,
                       _sync=io_out)
        tm.stop("backward")
        tm.stop("step")
        self._tm = tm
        return self.out

    def solve_energies(self, inputs, outputs):
        """Pipelined end-to-end form of ``solve`` for a sequence of energy
        points: ``inputs[k]`` = (a, b) and ``outputs[k]`` = (x_a, x_b) are
        HostWindow pairs of this rank (the blocks it reads / owns).  Energy
        k+1's window is copied into a second device input slot while energy k
        solves, energy k's owned outputs are copied to the host from a second
        device output slot while energy k+1 solves (the multi-GPU analogue of
        HostEnergySweep); energy 0 loads whole.  Needs two more full-size
        input and output sets on the device: raises torch.OutOfMemoryError
        when they do not fit (callers fall back to ``solve(host_in,
        host_out)`` per energy).  One partition per rank only."""
        if self._runner is not None:
            raise ValueError("solve_energies: one partition per rank only")
        if len(inputs) != len(outputs):
            raise ValueError("inputs and outputs differ in length")
        if not inputs:
            return 0
        A, B = self.A, self.B
        dev = A.device
        if getattr(self, "_slot1", None) is None:
            mk = lambda: DeviceBta.empty(A.n, A.b, A.a, dev, zero=False)  # noqa: E731
            self._slot1 = ((mk(), mk() if B is not None else None), (mk(), mk() if B is not None else None))
            self._h2d, self._d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ins = [(A, B), self._slot1[0]]
        outs = [self.out, self._slot1[1]]
        main = torch.cuda.current_stream(dev)
        h2d, d2h = self._h2d, self._d2h
        in_free, out_free = [None, None], [None, None]

        def load(win, slot):
            with torch.cuda.stream(h2d):
                if in_free[slot] is not None:
                    h2d.wait_event(in_free[slot])
                for w, D in zip(win, ins[slot]):
                    if w is not None and D is not None:
                        w.copy_to(D)
                ev = torch.cuda.Event()
                ev.record(h2d)
            return ev

        h2d.wait_stream(main)
        d2h.wait_stream(main)
        ready = load(inputs[0], 0)
        try:
            for k in range(len(inputs)):
                s = k & 1
                nxt = load(inputs[k + 1], s ^ 1) if k + 1 < len(inputs) else None
                main.wait_event(ready)
                if out_free[s] is not None:
                    main.wait_event(out_free[s])
                self.A, self.B = ins[s]
                self.out = outs[s]
                self.solve()
                done = torch.cuda.Event()
                done.record(main)
                in_free[s] = done
                with torch.cuda.stream(d2h):
                    d2h.wait_event(done)
                    for w, X in zip(outputs[k], outs[s]):
                        if w is not None and X is not None:
                            w.fill_from(X, non_blocking=True, tip=self.rank == 0)
                    ev = torch.cuda.Event()
                    ev.record(d2h)
                out_free[s] = ev
                ready = nxt
        finally:
            self.A, self.B = ins[0]
            self.out = outs[0]
        main.wait_stream(d2h)
        main.wait_stream(h2d)
        return len(inputs)

    def _copy_separators(self, host_in):
        """Couplings at the other partitions' boundaries (the reduced system
        is assembled on every rank)."""
        lo, hi = self.owned_range()
        for p in range(self.plan.num_parts - 1):
            g = self.plan.ranges[p][1] - 1
            if lo <= g < hi:
                continue  # streamed with this rank's own chunks
            for hm, D in zip(host_in, (self.A, self.B)):
                if hm is None or D is None:
                    continue
                if isinstance(hm, HostWindow):
                    lw, up = hm.separator(g)
                else:
                    h = hm.stacked()
                    lw, up = torch.from_numpy(h["lower"][g]), torch.from_numpy(h["upper"][g])
                D.lower[g].copy_(lw, non_blocking=True)
                D.upper[g].copy_(up, non_blocking=True)

    def phase_seconds(self):
        return self._tm.seconds()
