"""Wall-clock breakdown of one recon_full on config B (plan, uploads, CG, finalize)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200 import engine, simulate
prec = os.environ.get("PREC", "f16x3")
from paper_2604_09233_b200._native import Plan
prob = simulate.make_problem("B")
K, L, G = prob.temporal.shape[0], prob.spatial.shape[1], prob.sens.shape[1]
pl = Plan(K, L, G, prob.spatial.shape[0], "fp32"); pl.set_tables(prob.temporal, prob.spatial)
pl.set_sens(prob.sens, prob.intensity); sig = pl.apply_E(prob.rho_true / prob.intensity); pl.close()
for rep in range(2):
    inputs = engine.EncodingInputs(sigma=sig, spatial=prob.spatial,
                                   temporal=prob.temporal, sens=prob.sens, intensity=prob.intensity,
                                   kfilter=None, mask_r=prob.mask_r, grid=prob.grid, n_iter=20)
    t0 = time.perf_counter()
    img, log = engine.recon_full(inputs, precision=prec)
    wall = time.perf_counter() - t0
    tim = dict(log.timings) if hasattr(log, "timings") else {}
    cg = sum(v for k, v in tim.items() if k.startswith("cg_iteration"))
    print(f"rep {rep}: wall {wall*1e3:.1f} ms | " + " ".join(f"{k}={v*1e3:.1f}" for k, v in tim.items()
          if not k.startswith("cg_iteration")) + f" cg_total={cg*1e3:.1f}")
for rep in range(3):
    t0 = time.perf_counter(); p = Plan(K, L, G, prob.spatial.shape[0], prec); t1 = time.perf_counter()
    p.set_sens(prob.sens, prob.intensity); t2 = time.perf_counter()
    p.set_tables(prob.temporal, prob.spatial); t3 = time.perf_counter()
    p.set_samples(sig); t4 = time.perf_counter()
    p.close(); t5 = time.perf_counter()
    print(f"plan {1e3*(t1-t0):.1f} sens {1e3*(t2-t1):.1f} tables {1e3*(t3-t2):.1f} samples {1e3*(t4-t3):.1f} close {1e3*(t5-t4):.1f} ms")
