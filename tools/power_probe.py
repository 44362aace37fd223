"""Sustained E^H E applies on config B with nvidia-smi sampling (clocks, power) -- which part of
the f16x3 kernel the power cap is paid for.  NFS_B200_LIB selects a variant build.

    python tools/power_probe.py [n_applies]
"""
import os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_09233_b200 import _native, simulate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
prob = simulate.make_problem("B")
K, L, G, P1 = prob.temporal.shape[0], prob.spatial.shape[1], prob.sens.shape[1], prob.spatial.shape[0]
plan = _native.Plan(K, L, G, P1, os.environ.get("PREC", "f16x3"), 0)
plan.set_tables(prob.temporal, prob.spatial)
plan.set_sens(prob.sens, prob.intensity)
plan.apply_EHE(prob.rho_true)
plan.apply_EHE_resident(5)
torch.cuda.synchronize()
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        try:
            c, p, cap = [x.strip() for x in out.split(",")]
            samples.append((float(c), float(p), cap))
        except ValueError:
            pass
        time.sleep(0.05)


th = threading.Thread(target=sampler, daemon=True)
th.start()
t0 = time.perf_counter()
plan.apply_EHE_resident(n)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
stop.set(); th.join()
c = np.array([s[0] for s in samples]); p = np.array([s[1] for s in samples])
print(f"{n} applies: {dt / n * 1e3:.3f} ms each; sm MHz median {np.median(c):.0f} (min {c.min():.0f}); "
      f"power median {np.median(p):.0f} W (max {p.max():.0f}); power-cap samples {sum(1 for s in samples if 'Active' in s[2])}/{len(samples)}")
