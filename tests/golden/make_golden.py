"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src,
solves a grid of small BT/BTA systems with `solve_selected` and `dist_solve`,
records the reference's OpCounter tallies and known-answer results, and
writes the inputs and outputs as compressed .npz files next to this script.
The fixtures are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

SEQ_CASES = [
    # (name, n, b, a, mode, seed, hermitian_rhs)
    ("seq_bta_siq_5_4_2", 5, 4, 2, "siq", 11, False),
    ("seq_bta_si_5_4_2", 5, 4, 2, "si", 12, False),
    ("seq_bt_siq_7_3", 7, 3, 0, "siq", 13, False),
    ("seq_bt_si_7_3", 7, 3, 0, "si", 14, False),
    ("seq_bta_siq_6_8_4_herm", 6, 8, 4, "siq", 15, True),
    ("seq_bt_siq_4_16", 4, 16, 0, "siq", 16, True),
    ("seq_bta_siq_3_1_1", 3, 1, 1, "siq", 17, False),
    ("seq_bt_siq_1_4", 1, 4, 0, "siq", 18, False),
    ("seq_bta_siq_1_3_2", 1, 3, 2, "siq", 19, False),
    ("seq_bta_siq_2_5_3", 2, 5, 3, "siq", 20, True),
    ("seq_bta_siq_5_16_12", 5, 16, 12, "siq", 21, True),
    ("seq_bt_si_16_8", 16, 8, 0, "si", 0, False),
]

DIST_CASES = [
    # (name, n, b, a, mode, seed, parts)
    ("dist_siq_12_3_2_p3", 12, 3, 2, "siq", 31, 3),
    ("dist_si_12_3_0_p3", 12, 3, 0, "si", 32, 3),
    ("dist_siq_16_3_2_p8", 16, 3, 2, "siq", 33, 8),
    ("dist_siq_24_8_4_p4", 24, 8, 4, "siq", 34, 4),
    ("dist_si_8_2_0_p4", 8, 2, 0, "si", 35, 4),
    ("dist_siq_20_2_1_p8", 20, 2, 1, "siq", 36, 8),
    ("dist_siq_10_5_3_p2", 10, 5, 3, "siq", 37, 2),
    ("dist_siq_14_6_0_p3", 14, 6, 0, "siq", 38, 3),
]

KINDS = ("diag", "lower", "upper", "arrow_row", "arrow_col")


def stack(m, prefix, out):
    for kind in KINDS:
        blocks = getattr(m, kind)
        shape = {"diag": (m.b, m.b), "lower": (m.b, m.b), "upper": (m.b, m.b),
                 "arrow_row": (m.a, m.b), "arrow_col": (m.b, m.a)}[kind]
        arr = np.zeros((len(blocks),) + shape, np.complex128)
        for i, blk in enumerate(blocks):
            arr[i] = blk
        out[f"{prefix}_{kind}"] = arr
    out[f"{prefix}_tip"] = np.asarray(m.tip, np.complex128)


def main():
    sys.path.insert(0, REF)
    import btasel  # noqa: E402
    from btasel import (OpCounter, dist_solve, generate_dd_bta, hermitianize,  # noqa: E402
                        solve_selected, bta_forward, BtaMatrix)
    from btasel.threads import set_blas_threads  # noqa: E402

    set_blas_threads(1)
    manifest = {"reference": REF, "btasel_version": btasel.__version__, "numpy": np.__version__,
                "cases": {}}

    for name, n, b, a, mode, seed, herm in SEQ_CASES:
        A = generate_dd_bta(n, b, a, seed=seed)
        Braw = generate_dd_bta(n, b, a, seed=seed + 1)
        B = hermitianize(Braw) if herm else Braw
        cnt = OpCounter(b=b, a=a)
        sol = solve_selected(A, B if mode == "siq" else None, mode, counter=cnt)
        fwd = OpCounter(b=b, a=a)
        bta_forward(A.copy(), B.copy() if mode == "siq" else None, fwd)
        out = {}
        stack(A, "a", out)
        if mode == "siq":
            stack(B, "b", out)
        stack(sol.x_a, "xa", out)
        if sol.x_b is not None:
            stack(sol.x_b, "xb", out)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        manifest["cases"][name] = {
            "kind": "seq", "n": n, "b": b, "a": a, "mode": mode, "seed": seed, "hermitian_rhs": herm,
            "counts": cnt.as_dict(), "forward_counts": fwd.as_dict(),
        }

    for name, n, b, a, mode, seed, parts in DIST_CASES:
        A = generate_dd_bta(n, b, a, seed=seed)
        B = hermitianize(generate_dd_bta(n, b, a, seed=seed + 1))
        cnt = OpCounter(b=b, a=a)
        hub = btasel.ThreadHub(parts)
        sol = dist_solve(A, B if mode == "siq" else None, num_parts=parts, mode=mode, transport=hub,
                         counter=cnt)
        out = {}
        stack(A, "a", out)
        if mode == "siq":
            stack(B, "b", out)
        stack(sol.x_a, "xa", out)
        if sol.x_b is not None:
            stack(sol.x_b, "xb", out)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        plan = btasel.plan_partitions(n, parts, mode)
        manifest["cases"][name] = {
            "kind": "dist", "n": n, "b": b, "a": a, "mode": mode, "seed": seed, "parts": parts,
            "ranges": [list(r) for r in plan.ranges], "counts": cnt.as_dict(),
            "trace": [{"kind": e.kind, "payloads": [
                {k: (v if k != "blocks" else {kk: [list(s) for s in vv] for kk, vv in v.items()})
                 for k, v in p.items()} if isinstance(p, dict) else p for p in e.payloads]}
                for e in hub.trace],
        }

    # Config 1 of BASELINE.json (BT SI n=16 b=64, bench protocol seed 0):
    # per-block Frobenius norms and corner entries of X_A as a digest.
    A = generate_dd_bta(16, 64, 0, seed=0)
    sol = solve_selected(A, None, "si")
    digest = {k: [] for k in ("norm", "e00", "elast")}
    for kind, i, blk in sol.x_a.pattern_blocks():
        if blk.size == 0:
            continue
        digest["norm"].append(float(np.linalg.norm(blk)))
        digest["e00"].append([float(blk[0, 0].real), float(blk[0, 0].imag)])
        digest["elast"].append([float(blk[-1, -1].real), float(blk[-1, -1].imag)])
    manifest["config1_digest"] = digest
    a_stream = generate_dd_bta(3, 4, 2, seed=123)
    manifest["generator_probe"] = {
        "n": 3, "b": 4, "a": 2, "seed": 123,
        "diag0_row0": [[float(z.real), float(z.imag)] for z in a_stream.diag[0][0]],
        "tip": [[[float(z.real), float(z.imag)] for z in row] for row in a_stream.tip],
    }
    # Known answers (tests/test_rgf.py:31-35, 74-79, 109-119).
    two = BtaMatrix(2, 1, 0, [[[2.0]], [[2.0]]], [[[1.0]]], [[[1.0]]])
    manifest["known"] = {
        "two_by_two_inverse": [[2 / 3, -1 / 3], [-1 / 3, 2 / 3]],
        "two_block_s_a": [0.5, 1 / 1.5],
        "scalar_arrow_tip_schur_inv": 1 / 2.5,
        "scalar_arrow_inverse": [[0.6, -0.2], [-0.2, 0.4]],
        "two_block_xa_diag": [float(x[0, 0].real) for x in solve_selected(two).x_a.diag],
    }
    for counts_n in (5, 6):
        for mode in ("si", "siq"):
            for a in (0, 4):
                A = generate_dd_bta(counts_n, 8, a, seed=6)
                B = generate_dd_bta(counts_n, 8, a, seed=7)
                c = OpCounter(b=8, a=a)
                solve_selected(A, B if mode == "siq" else None, mode, counter=c)
                f = OpCounter(b=8, a=a)
                bta_forward(A.copy(), B.copy() if mode == "siq" else None, f)
                manifest.setdefault("op_counts", {})[f"{mode}_n{counts_n}_a{a}"] = {
                    "total": c.as_dict(), "forward": f.as_dict()}
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("wrote", len(manifest["cases"]), "cases")


if __name__ == "__main__":
    main()
