"""Per-operator device times of the tensor-core kernels for config B (PREC env = precision).

Profiling switches are compile-time: build a variant with tools/build_variant.sh NAME
-DNFS_TCI_DEBUG=m (f16x3) and point NFS_B200_LIB at it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09233_b200 import _native, simulate
prob = simulate.make_problem("B")
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
plan = _native.Plan(K, L, 32, 16, os.environ.get("PREC", "tf32x3"), 0)
plan.set_tables(prob.temporal, prob.spatial)
plan.set_sens(prob.sens, prob.intensity)
plan.apply_EHE(prob.rho_true)
kt = plan.kernel_times(3)
print("mode", os.environ.get("NFS_TC_DEBUG", "0"), "fwd ms %.3f adj ms %.3f" % (kt[0], kt[2]))
