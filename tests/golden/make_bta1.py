"""BTA1 golden files written by the REFERENCE (fileio.write_bta).

Run in the build container (where /root/reference exists):

    python tests/golden/make_bta1.py

Writes tests/golden/bta1_*.bta (reference-generated matrices and one
reference solution) and bta1_manifest.json (shape, sha256).  The GPU box only
reads the committed files.
"""

import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [("gen_3_2_1", 3, 2, 1, 0), ("gen_2_1_5", 2, 1, 5, 8), ("gen_1_1_0", 1, 1, 0, 1), ("gen_4_3_0", 4, 3, 0, 2)]


def main():
    sys.path.insert(0, REF)
    import btasel

    man = {}
    for name, n, b, a, seed in CASES:
        path = os.path.join(HERE, f"bta1_{name}.bta")
        btasel.write_bta(btasel.generate_dd_bta(n, b, a, seed=seed), path)
        man[name] = {"n": n, "b": b, "a": a, "seed": seed}
    A = btasel.generate_dd_bta(5, 4, 2, seed=3)
    B = btasel.hermitianize(btasel.generate_dd_bta(5, 4, 2, seed=4))
    sol = btasel.solve_selected(A, B, "siq")
    btasel.write_bta(sol.x_b, os.path.join(HERE, "bta1_sol_xb_5_4_2.bta"))
    man["sol_xb_5_4_2"] = {"n": 5, "b": 4, "a": 2, "seeds": [3, 4], "what": "solve_selected(A, B, 'siq').x_b"}
    for name in man:
        with open(os.path.join(HERE, f"bta1_{name}.bta"), "rb") as f:
            man[name]["sha256"] = hashlib.sha256(f.read()).hexdigest()
    with open(os.path.join(HERE, "bta1_manifest.json"), "w") as f:
        json.dump(man, f, indent=1)


if __name__ == "__main__":
    main()
