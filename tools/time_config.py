"""Per-operator device times (CUDA events, L2 not flushed) for a config and precision list.

    python tools/time_config.py --config D --precisions f16x3,fp32
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09233_b200 import _native, simulate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="B")
ap.add_argument("--precisions", default="f16x3,fp32")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
prob = simulate.make_problem(a.config)
K, L, G, P1 = prob.temporal.shape[0], prob.spatial.shape[1], prob.sens.shape[1], prob.spatial.shape[0]
out = {"config": a.config, "K": K, "L_R": L, "coils": G, "P1": P1, "pairs": K * L}
for prec in a.precisions.split(","):
    plan = _native.Plan(K, L, G, P1, prec, 0)
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    plan.apply_EHE(prob.rho_true)
    kt = plan.kernel_times(a.reps)
    ehe = sum(kt)
    out[prec] = {"forward_ms": kt[0], "adjoint_ms": kt[2], "reduce_ms": kt[1] + kt[3], "EHE_ms": ehe,
                 "pairs_per_s_per_op": K * L / (0.5 * ehe * 1e-3)}
    plan.close()
print(json.dumps(out, indent=1))
