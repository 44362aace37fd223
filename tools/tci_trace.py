import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200 import _native, simulate
lib = _native.load_library()
lib.nfs_tci_trace_enable.restype = ctypes.POINTER(ctypes.c_longlong)
tr = lib.nfs_tci_trace_enable()
prob = simulate.make_problem("B")
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
plan = _native.Plan(K, L, 32, 16, "f16x3", 0)
plan.set_tables(prob.temporal, prob.spatial); plan.set_sens(prob.sens, prob.intensity)
plan.apply_EHE(prob.rho_true)
plan.kernel_times(1)
a = np.ctypeslib.as_array(tr, shape=(64, 12)).copy()
a -= a[0, 0]
print("chunk phIssued itStart emptyAok genArrA cmmaGo cmmaCommit | pfWait pfGot mathEnd phEmptyArr | dEmptyOk drainDone")
for c in range(24):
    print(c, *a[c][:6], '|', *a[c][6:10], '|', *a[c][10:12])
d = np.diff(a[4:60, 4])
print("mean cycles per chunk (issuer start to start):", d.mean())
b = np.ctypeslib.as_array(tr, shape=(64 * 12 + 64 * 8,)).copy()[768:].reshape(64, 8)
b = np.where(b > 0, b - np.ctypeslib.as_array(tr, shape=(768,))[0], 0)
print("per-quadrant: chunk | phase got q0..q3 | phase released q0..q3 | next phIssued")
for c in range(4, 24):
    print(c, *b[c][4:], '|', *b[c][:4], '|', a[c + 4][0] if c + 4 < 64 else '')
