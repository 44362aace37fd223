"""E^H E applies/s over a shape sweep on one GPU (device times, CUDA events).

    python tools/sweep_e.py --out profiles/r1_sweep_e.json [--precisions f16x3,fp32] [--quick]

Random basis tables with a realistic phase range (row 0: time in s x B0 in rad/s, the other rows
O(1) coefficients), random coil maps.  Each point: plan + tables + one warm-up E^H E, then
`nfs_kernel_times` (forward + split reduction + adjoint + reduction, back to back, L2 warm).
A point whose device buffers do not fit is recorded as skipped, not fatal.
"""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_09233_b200 import _native  # noqa: E402
from paper_2604_09233_b200.errors import EngineError  # noqa: E402


def tables(K, L, P1, rng):
    temporal = np.empty((K, P1))
    temporal[:, 0] = np.linspace(0.0, 0.03, K)                        # t (s)
    if P1 > 1:
        temporal[:, 1:] = rng.uniform(-1.0, 1.0, (K, P1 - 1)) * 40.0  # k_p(t) (rad per unit basis)
    spatial = np.empty((P1, L))
    spatial[0] = rng.uniform(-1.0, 1.0, L) * 2 * np.pi * 100.0          # B0 (rad/s)
    if P1 > 1:
        spatial[1:] = rng.uniform(-1.0, 1.0, (P1 - 1, L))
    return temporal, spatial


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r1_sweep_e.json")
    ap.add_argument("--precisions", default="f16x3,fp32")
    ap.add_argument("--quick", action="store_true", help="3 points per precision (smoke)")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    Ls = [2 ** e for e in (12, 14, 16, 18, 20)]
    Ks = [2 ** e for e in (14, 16, 18)]
    rows = []
    for prec in a.precisions.split(","):
        if prec == "f16x3":
            grid = list(itertools.product(Ls, Ks, (8, 32), (3, 16)))
        else:   # the CUDA-core modes are ~5x slower: coil/term extremes only at the largest sizes
            grid = list(itertools.product(Ls, Ks, (32,), (16,))) + [(2 ** 16, 2 ** 16, 8, 3)]
        if a.quick:
            grid = grid[:3]
        for (L, K, G, P1) in grid:
            rec = {"precision": prec, "L_R": L, "K": K, "coils": G, "P1": P1}
            t0 = time.time()
            try:
                temporal, spatial = tables(K, L, P1, rng)
                sens = (rng.standard_normal((L, G)) + 1j * rng.standard_normal((L, G))) / np.sqrt(G)
                plan = _native.Plan(K, L, G, P1, prec, 0)
                try:
                    plan.set_tables(temporal, spatial)
                    plan.set_sens(sens)
                    plan.apply_EHE(rng.standard_normal(L) + 1j * rng.standard_normal(L))
                    kt = plan.kernel_times(a.reps)
                    ehe = sum(kt)
                    rec.update(EHE_ms=ehe, forward_ms=kt[0], adjoint_ms=kt[2], applies_per_s=1e3 / ehe,
                               pairs_per_s_per_op=K * L / (0.5 * ehe * 1e-3), plan=plan.describe())
                finally:
                    plan.close()
            except EngineError as e:
                rec["skipped"] = str(e)
            rec["wall_s"] = round(time.time() - t0, 2)
            rows.append(rec)
            print(json.dumps({k: v for k, v in rec.items() if k != "plan"}), flush=True)
    with open(a.out, "w") as f:
        json.dump({"_doc": __doc__.strip().splitlines()[0], "points": rows}, f, indent=1)


if __name__ == "__main__":
    main()
