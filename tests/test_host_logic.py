"""CPU tests of the host-side logic and the C-ABI library (no GPU calls)."""

import ctypes
import os
import re

import numpy as np
import pytest
from conftest import ROOT, load_case, manifest

import oracle
import paper_2601_04904_b200 as bs
from paper_2601_04904_b200 import _native
from paper_2601_04904_b200.kernels import record_sweep

M = manifest()


# ---- partition plan (partition.py:52-90) ----------------------------------

@pytest.mark.parametrize("mode", ["si", "siq"])
def test_plan_matches_oracle_exhaustive(mode):
    for parts in range(2, 10):
        for n in range(2 * parts, 2 * parts + 60):
            ranges, kinds = oracle.plan_partitions(n, parts, mode)
            plan = bs.plan_partitions(n, parts, mode)
            assert list(plan.ranges) == ranges and list(plan.kinds) == kinds


def test_plan_reference_values_and_errors():
    assert bs.plan_partitions(1024, 8, "siq").ranges[1] == (218, 316)
    assert [bs.plan_partitions(1024, 4, "siq").size(r) for r in range(4)] == [354, 158, 158, 354]
    with pytest.raises(ValueError):
        bs.plan_partitions(7, 4)
    with pytest.raises(ValueError):
        bs.plan_partitions(8, 1)


# ---- logical op counts (OpCounter parity, test_acceptance.py:149-198) -----

@pytest.mark.parametrize("key", sorted(M["op_counts"]))
def test_record_sweep_matches_reference_counts(key):
    mode, n, a = key.split("_")
    n, a = int(n[1:]), int(a[1:])
    ref = M["op_counts"][key]
    c = bs.OpCounter(b=8, a=a)
    record_sweep(c, n, 8, a, mode, "forward")
    assert c.as_dict() == ref["forward"]
    record_sweep(c, n, 8, a, mode, "backward")
    assert c.as_dict() == ref["total"]


@pytest.mark.parametrize("name", sorted(k for k, v in M["cases"].items() if v["kind"] == "seq"))
def test_record_sweep_matches_golden_cases(name):
    meta = M["cases"][name]
    c = bs.OpCounter(b=meta["b"], a=meta["a"])
    record_sweep(c, meta["n"], meta["b"], meta["a"], meta["mode"], "forward")
    assert c.as_dict() == meta["forward_counts"]
    record_sweep(c, meta["n"], meta["b"], meta["a"], meta["mode"], "backward")
    assert c.as_dict() == meta["counts"]


@pytest.mark.parametrize("n,b,a,mode", [(9, 4, 4, "siq"), (3, 2, 2, "si"), (1, 5, 5, "siq"), (4, 3, 1, "siq")])
def test_record_sweep_vs_oracle_counter_any_shape(n, b, a, mode):
    from collections import Counter
    A = oracle.generate_dd_bta(n, b, a, seed=3)
    B = oracle.generate_dd_bta(n, b, a, seed=4) if mode == "siq" else None
    cnt = Counter()
    oracle.solve_selected(A, B, mode, counts=cnt)
    # oracle counts in its own classes; re-classify against (b, a) like OpCounter
    c = bs.OpCounter(b=b, a=a)
    record_sweep(c, n, b, a, mode, "forward")
    record_sweep(c, n, b, a, mode, "backward")
    assert dict(c.gemm_by_shape) == dict(cnt)


# ---- containers / generator (matrix.py) ------------------------------------

def test_generator_bitwise_vs_reference_inputs():
    for name in ("seq_bta_siq_5_4_2", "seq_bt_si_16_8", "dist_siq_24_8_4_p4"):
        meta, A, B, _, _ = load_case(name)
        g = bs.generate_dd_bta(meta["n"], meta["b"], meta["a"], seed=meta["seed"])
        for (_, _, x), (_, _, y) in zip(g.pattern_blocks(), A.blocks()):
            np.testing.assert_array_equal(x, y)
        if B is not None and meta.get("hermitian_rhs", meta["kind"] == "dist"):
            h = bs.hermitianize(bs.generate_dd_bta(meta["n"], meta["b"], meta["a"], seed=meta["seed"] + 1))
            for (_, _, x), (_, _, y) in zip(h.pattern_blocks(), B.blocks()):
                np.testing.assert_array_equal(x, y)


def test_block_list_views_and_validation():
    m = bs.BtaMatrix.zeros(3, 2, 1)
    m.diag[1] = np.eye(2)
    assert m.stacked()["diag"][1, 0, 0] == 1
    m.diag[2][:] = 5.0
    assert np.all(m.stacked()["diag"][2] == 5)
    assert len(m.lower) == 2 and m.tip.shape == (1, 1)
    with pytest.raises(bs.ShapeMismatchError):
        m.diag[0] = np.eye(3)
    with pytest.raises(bs.ShapeMismatchError):
        bs.BtaMatrix(2, 2, 0, [np.eye(2)], [np.eye(2)], [np.eye(2)])
    c = m.copy()
    c.diag[0][0, 0] = 9
    assert m.diag[0][0, 0] == 0
    assert bs.BtaMatrix.identity(2, 3, 1).equals_exact(bs.mask_to_pattern(np.eye(7), (2, 3, 1)))
    d = bs.to_dense(bs.generate_dd_bta(3, 2, 2, seed=1))
    assert d.shape == (8, 8)


def test_hermitianize_matches_oracle():
    g = bs.generate_dd_bta(4, 3, 2, seed=9)
    h1 = bs.hermitianize(g)
    h2 = oracle.hermitianize(oracle.generate_dd_bta(4, 3, 2, seed=9))
    for (_, _, x), (_, _, y) in zip(h1.pattern_blocks(), h2.blocks()):
        np.testing.assert_array_equal(x, y)


# ---- C ABI: library loads, exports every declared symbol --------------------

def _header_symbols():
    with open(os.path.join(ROOT, "include", "btasel_b200.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"\b(bsel_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    declared = _header_symbols()
    assert set(declared) == set(_native.EXPORTS)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert lib.bsel_abi_version() == 3


def test_abi_struct_layouts():
    import shutil
    import subprocess
    import tempfile
    names = {"Status": "bsel_status_t", "Bta": "bsel_bta_t", "Factors": "bsel_factors_t",
             "LocalFactors": "bsel_local_factors_t", "Profile": "bsel_profile_t", "HostIo": "bsel_host_io_t"}
    sizes = {"Status": 272, "Bta": 72, "Factors": 104, "LocalFactors": 96, "Profile": 80, "HostIo": 56}
    if shutil.which("gcc"):
        fmt = " ".join(["%zu"] * len(names))
        src = ('#include <stdio.h>\n#include "btasel_b200.h"\nint main(void){printf("' + fmt + '",'
               + ", ".join(f"sizeof({c})" for c in names.values()) + ');return 0;}')
        with tempfile.TemporaryDirectory() as d:
            open(os.path.join(d, "t.c"), "w").write(src)
            subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "t"),
                            os.path.join(d, "t.c")], check=True)
            out = subprocess.run([os.path.join(d, "t")], capture_output=True, text=True, check=True).stdout
        sizes = dict(zip(names, map(int, out.split())))
    for name, size in sizes.items():
        assert ctypes.sizeof(getattr(_native, name)) == size, name
    size = ctypes.c_size_t()
    lib = _native.load_library()
    assert lib.bsel_solve_workspace_size(4, 8, 2, 1, ctypes.byref(size)) == 0
    assert size.value > 16 * (4 * 8 * 8)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(bs.NativeUnavailableError):
        _native.load_library(str(tmp_path / "nope.so"))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bs.NativeUnavailableError):
        bs.solve_selected(bs.generate_dd_bta(2, 2, 0, seed=1))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2601_04904_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_dense_expansion_and_mask_roundtrip():
    """dense.py expansion / masking (plain tensor indexing, runs on CPU
    tensors too) agree with the host to_dense / mask_to_pattern."""
    import torch
    from paper_2601_04904_b200 import DeviceBta, generate_dd_bta
    from paper_2601_04904_b200.dense import dense_device, mask_device
    from paper_2601_04904_b200.matrix import to_dense
    for shape in [(4, 3, 2), (1, 2, 0), (3, 1, 4), (2, 5, 0)]:
        m = generate_dd_bta(*shape, seed=1)
        d = DeviceBta(*shape, {k: torch.from_numpy(v) for k, v in m.stacked().items()})
        dd = dense_device(d)
        assert np.array_equal(dd.numpy(), to_dense(m))
        back = mask_device(dd, shape)
        for k, v in m.stacked().items():
            assert np.array_equal(getattr(back, k).numpy(), v)


def test_energy_assignment():
    from paper_2601_04904_b200 import energy_seeds, rank_energies
    assert energy_seeds(0) == (0, 1) and energy_seeds(5) == (10, 11)
    es = list(range(64))
    parts = [rank_energies(es, 8, r) for r in range(8)]
    assert sorted(sum(parts, [])) == es and all(len(p) == 8 for p in parts)
    assert rank_energies(range(3), 4, 3) == []
