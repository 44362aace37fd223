"""Per-CTA fixed-cost stamps of CTA (0,0) from a -DNFS_TCI_TRACE build (1- and N-chunk problems):
kernel entry, setup done, owner image landed (phase issuer), first phase MMA, first / last
contraction, last drain load, epilogue written, end, TMEM freed (clock64 cycles)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200 import _native
lib = _native.load_library()
import ctypes
lib.nfs_tci_trace_enable.restype = ctypes.POINTER(ctypes.c_longlong)
tr = lib.nfs_tci_trace_enable()
rng = np.random.default_rng(0)
K, G, P1 = 65536, 32, 16
for L in (32, 32 * 12):
    temporal = rng.standard_normal((K, P1)) * 0.5
    spatial = rng.standard_normal((P1, L)) * 0.5
    sens = rng.standard_normal((L, G)) + 1j * rng.standard_normal((L, G))
    plan = _native.Plan(K, L, G, P1, "f16x3", 0)
    plan.set_tables(temporal, spatial); plan.set_sens(sens)
    p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    for _ in range(3):   # no host access in between: the managed trace pages stay on the GPU
        plan.apply_E(p)
    a = np.ctypeslib.as_array(tr, shape=(64 * 12,)).copy()
    t0 = a[756]
    names = ["entry", "setup", "owner img", "last drain ld", "epilogue", "roles end", "syncthreads", "dealloc"]
    fx = {n: a[756 + i] - t0 for i, n in enumerate(names)}
    n_ch = L // 32
    print(f"L={L} ({n_ch} chunks/CTA):", " ".join(f"{k}={v}" for k, v in fx.items()),
          f"| phIssued0={a[0]-t0} cmmaGo0={a[4]-t0} cmmaCommit_last={a[(n_ch-1)*12+5]-t0}")
    plan.close()
