"""Test shim: ``import btasel`` resolves to the B200 package, so the
reference's OWN test files (pkg/tests/test_rgf.py, test_dist.py,
test_acceptance.py) run unmodified against the GPU implementation
(tests/test_gpu_reference_suite.py).  Not part of the product.

Hot-path modules map to this repository's package:
    btasel, btasel.rgf, btasel.dist, btasel.kernels, btasel.matrix,
    btasel.partition, btasel.errors, btasel.fileio
Harness-only modules that are out of scope (the click CLI,
the bench report, BLAS thread pools, the CPU dense/batched oracles, the
in-process ThreadHub and TCP SocketCollectives transports) are the
reference's own, loaded from the offline install ``baseline/_ref`` under
the private name ``_btasel_ref`` and sharing THIS package's exception
classes (so ``except ProtocolError`` / ``WorkerError`` attribution works
across both).  The transports then drive this package's ``dist_solve``
exactly as they drive the reference's.
"""

import importlib.util
import os
import sys
import types

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2601_04904_b200 as _pkg  # noqa: E402
from paper_2601_04904_b200 import (collectives as _coll, dist as _dist, errors as _errors, fileio as _fileio,  # noqa: E402
                                   kernels as _kernels, matrix as _matrix, partition as _partition, rgf as _rgf)


def _load_reference():
    ref = os.environ.get("BTASEL_REF_DIR", os.path.join(_ROOT, "baseline", "_ref", "btasel"))
    if "_btasel_ref" in sys.modules:
        return sys.modules["_btasel_ref"]
    sys.modules["_btasel_ref.errors"] = _errors  # one exception hierarchy for both
    spec = importlib.util.spec_from_file_location("_btasel_ref", os.path.join(ref, "__init__.py"),
                                                  submodule_search_locations=[ref])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_btasel_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


_ref = _load_reference()
for _sub in ("threads", "bench", "cli", "baselines", "collectives"):
    importlib.import_module(f"_btasel_ref.{_sub}")

# package namespace: the B200 package first, reference harness names after
for _name in dir(_ref):
    if not _name.startswith("__"):
        globals()[_name] = getattr(_ref, _name)
for _name in dir(_pkg):
    if not _name.startswith("__"):
        globals()[_name] = getattr(_pkg, _name)

# submodules
_collectives = types.ModuleType("btasel.collectives")
_collectives.__dict__.update({k: v for k, v in vars(_ref.collectives).items() if not k.startswith("__")})
_collectives.__dict__.update({k: getattr(_coll, k) for k in ("Collectives", "TraceEvent", "TorchCollectives", "LocalHub")})

for _sub, _mod in {"rgf": _rgf, "dist": _dist, "kernels": _kernels, "matrix": _matrix, "partition": _partition,
                   "errors": _errors, "fileio": _fileio, "collectives": _collectives,
                   "threads": _ref.threads, "bench": _ref.bench, "cli": _ref.cli,
                   "baselines": _ref.baselines}.items():
    sys.modules[f"{__name__}.{_sub}"] = _mod
    globals()[_sub] = _mod

# the reference's CPU oracles stay the oracles (acceptance criteria 1-3 compare
# the solver against them): an independent check, not the GPU dense path
dense_solve = _ref.dense_solve
batched_solve = _ref.batched_solve
