#!/usr/bin/env python
"""Benchmark: E^H E applies/s (and end-to-end CG seconds) on SURVEY.md config B.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision f16x3|tf32x3|fp32|fp64]
    python bench.py --impl reference ...      # CPU reference arm (oracle port, host cores)

A step = one E^H E apply (forward + adjoint, phase regenerated on the fly) over config B:
2D 256x256 spiral, L_R = 41,684 voxels, K = 65,536 samples (71.5 ms readout, R=4),
32 coils, B0 + 15 third-order field terms (P+1 = 16).  `value` is device-timed with inputs
resident in HBM; `e2e` is the same metric through the public API (`recon_full` from host
numpy arrays, 20 CG iterations, host<->device copies inside the timed region).
For N > 1 (torchrun) the samples are sharded across ranks with one NCCL all-reduce of the
adjoint image per apply (strong scaling of the fixed config-B job).
"""

from __future__ import annotations

import os

# The CPU legs must size the BLAS pool before numpy is imported (nfs/cli.py:19 quirk).
_NCPU = len(os.sched_getaffinity(0))
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, str(_NCPU))

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = ("config B: 2D 256x256 single-shot spiral, L_R=41684 (disc mask), K=65536 samples "
            "(71.5 ms, R=4), 32 coils, B0 + 15 third-order field terms (P+1=16)")
METRIC = "E^H E applies/s (config B)"
CPU_SAMPLE_ROWS = 1206   # 3 reference split blocks of 402 rows (budget 2^28 B, nfs/pipeline.py:221)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.perf_counter(), parts))

    def window(self, t0, t1):
        """Keep the samples taken inside [t0, t1] (the timed region; nvidia-smi was started
        before the warm-up so it is sampling by then)."""
        self.t0, self.t1 = t0, t1

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        rows = [r for t, r in self.rows if t0 is None or t0 <= t <= t1]
        if not rows:   # region shorter than one sampling period: nearest samples
            rows = [r for _, r in sorted(self.rows, key=lambda tr: abs(tr[0] - (t0 or 0)))[:3]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self_rows = rows
        sm = [float(r[0]) for r in self_rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self_rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self_rows for n, v in zip(names, r[3:]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self_rows)}


# ------------------------------------------------------------------ CPU legs
def cpu_reference_sample(prob, rows=CPU_SAMPLE_ROWS):
    """Time the reference algorithm (oracle port of nfs/engine.py:217-223 recon_split inner
    loop, P recomputed per 402-row block) on `rows` sample rows; return extrapolated
    full-config applies/s and the sample seconds."""
    from oracle import nfs_oracle as orc   # CPU baseline leg only

    s_eff = prob.sens * prob.intensity[:, None]
    temporal = prob.temporal[:rows]
    starts = orc.choose_block_starts(rows, prob.spatial.shape[1], 2**28)
    p = (prob.rho_true / prob.intensity).astype(np.complex128)
    t0 = time.perf_counter()
    orc.split_normal_apply(p, s_eff, prob.spatial, temporal, starts)
    dt = time.perf_counter() - t0
    full_s = dt * prob.temporal.shape[0] / rows
    return 1.0 / full_s, dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2604_09233_b200 import simulate

    prob = simulate.make_problem("B")
    for _ in range(max(args.warmup, 0) and 1):
        cpu_reference_sample(prob, rows=402)
    vals, secs = [], []
    for _ in range(args.steps):
        v, dt = cpu_reference_sample(prob)
        vals.append(v)
        secs.append(dt)
    value = float(np.median(vals))
    sample = (f"{CPU_SAMPLE_ROWS} of 65536 sample rows (3 reference split blocks of 402 rows), "
              f"extrapolated linearly to the full apply; numpy+OpenBLAS, {_NCPU} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "applies/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": WORKLOAD, "variant": "recon_split (P recomputed per block)",
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": "applies/s", "cores": _NCPU, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_seconds": secs,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default=os.environ.get("NFS_BENCH_PRECISION", "f16x3"),
                    choices=["f16x3", "tf32x3", "fp32", "fp64"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["NFS_B200_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2604_09233_b200 import _native, engine, simulate

    prob = simulate.make_problem("B")
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
    lo, hi = engine.shard_rows(K, rank, world)

    plan = _native.Plan(hi - lo, L, G, P1, args.precision, local)
    stream = torch.cuda.Stream()
    plan.set_stream(stream.cuda_stream)
    if world > 1:
        plan.attach_comm(engine._nccl_unique_id(dist, rank), rank, world)
    plan.set_tables(prob.temporal[lo:hi], prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    # synthetic raw data = E rho_true through the device forward operator
    sigma = plan.apply_E(prob.rho_true / prob.intensity)
    plan.set_samples(sigma)
    plan.apply_EHE(prob.rho_true)   # places p on the device for the resident applies

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    launches = plan.launches_per_apply()

    clk = ClockSampler(local).__enter__()   # sampling from before the warm-up
    try:
        t_wait = time.perf_counter()
        while not clk.rows and time.perf_counter() - t_wait < 3.0 and clk.proc is not None:
            time.sleep(0.01)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                plan.apply_EHE_resident(1)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            t_start = time.perf_counter()
            for i in range(args.steps):
                flush.fill_(float(i))            # evict L2 between steps (outside the events)
                ev[i][0].record(stream)
                plan.apply_EHE_resident(1)
                ev[i][1].record(stream)
            stream.synchronize()
            torch.cuda.synchronize()
            clk.window(t_start, time.perf_counter())
            if world > 1:
                dist.barrier()
    finally:
        clk.__exit__(None, None, None)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1e3 / ms_per_step

    # per-kernel durations on the plan stream (CUDA events), roofline of the dominant kernel
    kt = plan.kernel_times(reps=3)
    k_loc = hi - lo
    flops_1 = float(k_loc) * L * (8 * G + 2 * P1)
    dom = int(np.argmax([kt[0], kt[2]]))
    dom_ms = [kt[0], kt[2]][dom]
    pk = peaks()
    clocks = clk.summary()
    if args.precision == "fp64":
        peak = 148 * 64 * 2 * 1.965e9 / 1e12
        bound, peak_src = "fp64", "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1965 MHz"
    elif args.precision == "tf32x3":
        peak = pk.get("bf16_tflops", 1590.0) / 2
        bound, peak_src = "tensor", "measured bf16 dense (MEASURED_PEAKS.json) / 2 = tf32 dense"
    elif args.precision == "f16x3":
        peak = pk.get("bf16_tflops", 1590.0)
        bound, peak_src = "tensor", ("measured bf16 dense burst (MEASURED_PEAKS.json); fp16 MMA runs at "
                                     "the same rate")
    else:
        peak = 148 * 128 * 2 * 1.965e9 / 1e12
        bound, peak_src = "fp32", ("nominal 148 SM x 128 FP32 lanes x 2 flop x sm_max 1965 MHz "
                                   "(MEASURED_PEAKS.json carries no FP32-pipe figure)")
    achieved = flops_1 / (dom_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
            traffic = json.load(fh).get(args.precision, {}).get(["forward", "adjoint"][dom])
    except (OSError, ValueError):
        pass
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": "profiles/r1_traffic.json (ncu --set full, dram read+write bytes per launch)",
                "kernel": ["contract_forward", "contract_adjoint"][dom],
                "kernel_ms": dom_ms, "algorithmic_flop_per_launch": flops_1,
                "peak_source": peak_src,
                "kernel_ms_all": {"forward": kt[0], "forward_reduce": kt[1], "adjoint": kt[2],
                                  "adjoint_reduce": kt[3]}}
    if clocks.get("sm_mhz"):
        roofline["frac_at_observed_clock"] = achieved / (peak * clocks["sm_mhz"] / 1965.0)
    # the phasor e^{i phi} costs 2 MUFU ops (sin, cos) per pair in every mode: the SFU floor
    # (16 MUFU lane-ops / clk / SM, tools/ubench/mufu_rate.cu) is the binding resource of the
    # tensor-core modes
    if args.precision != "fp64":
        mufu_peak = 148 * 16 * 1.965e9
        roofline["mufu_frac"] = 2.0 * float(k_loc) * L / (dom_ms * 1e-3) / mufu_peak
        # the highest `frac` this algorithm can reach: the phasor's 2 MUFU ops per pair at the
        # SFU peak bound the time per launch from below, whatever the tensor cores do
        t_floor = 2.0 * float(k_loc) * L / mufu_peak
        roofline["frac_ceiling_mufu"] = flops_1 / t_floor / 1e12 / peak
        if clocks.get("sm_mhz"):   # against the SFU peak at the clock the run actually had
            roofline["mufu_frac_at_observed_clock"] = roofline["mufu_frac"] * 1965.0 / clocks["sm_mhz"]
    if args.precision in ("f16x3", "tf32x3"):
        # the split MMA executes 3 products on the real-ified operands: 3 x 2 x (2 x 2G) per pair
        executed = float(k_loc) * L * 3 * 2 * 2 * (2 * G) * 2 / 2
        roofline["tensor_flop_executed_per_launch"] = executed
        roofline["tensor_frac_executed"] = executed / (dom_ms * 1e-3) / 1e12 / peak
        roofline["fp32_cuda_core_equiv_frac"] = achieved / (148 * 128 * 2 * 1.965e9 / 1e12)

    # end-to-end through the public API (host arrays in, image out)
    inputs = engine.EncodingInputs(sigma=np.empty((K, G), np.complex128), spatial=prob.spatial,
                                   temporal=prob.temporal, sens=prob.sens,
                                   intensity=prob.intensity, kfilter=None, mask_r=prob.mask_r,
                                   grid=prob.grid, n_iter=prob.n_iter)
    if world > 1:
        full = [None] * world
        dist.all_gather_object(full, sigma)
        inputs.sigma = np.concatenate(full, 0)
    else:
        inputs.sigma = sigma
    e2e_times = []
    img = log = None
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        img, log = engine.recon_full(inputs, precision=args.precision)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = min(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    iters = len(log.residual_norms)
    h2d = (prob.temporal.nbytes + prob.spatial.nbytes + prob.sens.nbytes + prob.intensity.nbytes
           + inputs.sigma.nbytes)
    d2h = L * 16 + 2 * 8 * iters
    rel_truth = float(np.linalg.norm(img.values[prob.mask_r] - prob.rho_true)
                      / np.linalg.norm(prob.rho_true))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # ~10 s of CPU work: three samples of 8 reference split blocks (402 rows each)
        rows = 8 * 402
        runs = [cpu_reference_sample(prob, rows=rows) for _ in range(3)]
        cpu = {"value": float(np.median([v for v, _ in runs])), "unit": "applies/s", "cores": _NCPU,
               "kind": "port",
               "sample": (f"3 x {rows} of {K} sample rows (8 reference split blocks of 402 rows) of one "
                          f"E^H E, {sum(dt for _, dt in runs):.1f} s of CPU work, extrapolated linearly; "
                          "oracle port of nfs/engine.py:217-223, numpy+OpenBLAS")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value * 1.0, "unit": "applies/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": {"fp32": "fp32", "fp64": "fp64", "tf32x3": "tf32x3 (fp32 accumulate)",
                      "f16x3": "f16x3 split contraction (exact int8 phase, fp32 accumulate)"}[args.precision],
            "data": "synthetic (disc phantom, synthetic coils, linear B0; raw data from the device forward model)",
            "config": {"workload": WORKLOAD, "precision": args.precision,
                       "l2": "flushed between steps (256 MiB device write outside the timed events)",
                       "parallelism": f"sample-sharded x{world}" if world > 1 else "1 GPU",
                       "plan": plan.describe()},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": iters / e2e_s, "unit": "applies/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "recon_seconds": e2e_s, "cg_iterations": iters,
                    "api": "paper_2604_09233_b200.recon_full (host numpy in/out)",
                    "rel_l2_vs_truth": rel_truth},
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
