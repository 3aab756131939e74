"""B200-native fused BT/BTA selected inversion (SI) and selected quadratic
solution (SQ): a drop-in for the hot path of `btasel` (arXiv 2601.04904).

Public API mirrors btasel/__init__.py for the hot path:

* containers / generators: BtaMatrix, SelectedSolution, generate_dd_bta,
  hermitianize, to_dense, mask_to_pattern; DeviceBta (device fast path)
* sequential solver: solve_selected, bt_forward, bt_backward, bta_forward,
  bta_backward, RgfFactors
* distributed solver: dist_solve, local_forward, assemble_reduced,
  solve_reduced, local_backward, plan_partitions, Collectives
* kernels: OpCounter, block_multiply_acc, mm, block_inverse
* BTA1 files: read_bta, write_bta, read_bta_header (+ read_bta_device)
* dense GPU oracle: dense_solve (baselines.py)
* energy-point sweeps (config 5): EnergySweep; host-buffer pipelined sweep: HostEnergySweep
* errors: the reference's exception hierarchy

Every numerical call runs in libbtasel_b200.so (sm_100a); there is no CPU
fallback.
"""

from .errors import (
    BadMagicError,
    BtaselError,
    DenseGuardError,
    FormatError,
    NativeUnavailableError,
    ProtocolError,
    ShapeMismatchError,
    ShapeInconsistencyError,
    SingularBlockError,
    TruncatedPayloadError,
    WorkerError,
)
from .matrix import BtaMatrix, SelectedSolution, generate_dd_bta, hermitianize, mask_to_pattern, to_dense
from .partition import PartitionPlan, plan_partitions
from .kernels import OpCounter, block_inverse, block_multiply_acc, mm
from .device import (DeviceBta, bind_host_to_device, generate_dd_bta_device, hermitianize_device, kernel_launches,
                     to_device, to_host)
from .rgf import (RgfFactors, bt_backward, bt_forward, bta_backward, bta_forward, default_partitions,
                  release_caches, solve_selected)
from .collectives import Collectives, LocalHub, TorchCollectives, TraceEvent
from .dist import (BoundaryPayload, DistSolver, HostWindow, InGpuPartitions, LocalFactors, ReducedSystem,
                   assemble_reduced, dist_solve, local_backward, local_forward, solve_reduced)
from .fileio import read_bta, read_bta_device, read_bta_header, write_bta
from .dense import dense_solve
from .energy import EnergySweep, HostEnergySweep, energy_seeds, rank_energies

__version__ = "0.1.0"

__all__ = [
    "BtaMatrix", "SelectedSolution", "RgfFactors", "OpCounter", "PartitionPlan", "DeviceBta",
    "bind_host_to_device",
    "generate_dd_bta", "hermitianize", "to_dense", "mask_to_pattern", "to_device", "to_host",
    "block_multiply_acc", "mm", "block_inverse",
    "bt_forward", "bt_backward", "bta_forward", "bta_backward", "solve_selected", "default_partitions",
    "release_caches", "InGpuPartitions",
    "plan_partitions", "dist_solve", "local_forward", "assemble_reduced", "solve_reduced", "local_backward",
    "BoundaryPayload", "LocalFactors", "ReducedSystem", "DistSolver", "HostWindow", "Collectives", "TorchCollectives",
    "LocalHub", "TraceEvent", "generate_dd_bta_device", "hermitianize_device", "kernel_launches",
    "BtaselError", "ShapeMismatchError", "SingularBlockError", "DenseGuardError", "ProtocolError",
    "WorkerError", "NativeUnavailableError", "FormatError", "BadMagicError", "TruncatedPayloadError",
    "ShapeInconsistencyError", "read_bta", "write_bta", "read_bta_header", "read_bta_device", "dense_solve",
    "EnergySweep", "HostEnergySweep", "energy_seeds", "rank_energies",
]
