#!/usr/bin/env python
"""Benchmark: E^H E applies/s (and end-to-end CG seconds) on SURVEY.md config B (or D).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision f16x3|tf32x3|fp32|fp64]
                    [--config B|D]
    python bench.py --impl reference ...      # the reference's own CPU path on the host cores

A step = one E^H E apply (forward + adjoint, phase regenerated on the fly; for N > 1 plus the
NCCL all-reduce of the adjoint image) over the configuration's full problem:
  B  2D 256x256 spiral, L_R = 41,684, K = 65,536 (71.5 ms, R=4), 32 coils, P+1 = 16
  D  3D 128x128x64 stack of spirals, L_R = 532,872, K = 299,648 (R~7), 32 coils, P+1 = 16
`value` is device-timed (CUDA events on the plan stream, inputs resident in HBM, L2 flushed by a
256 MiB device write before every step, outside the events); the dominant kernel is timed with
events around each of its launches INSIDE the same steps (roofline).  `e2e` is the same metric
through the public API: `recon_full` from host numpy arrays (20 CG iterations for B, 50 for D),
host<->device copies inside the timed region.  `sustained` repeats the apply back to back for a
few seconds (power-capped clock) against the sustained tensor peak.
For N > 1 (torchrun) the samples are sharded across ranks (strong scaling of the fixed job).

The reference arm and the `cpu_baseline` leg run the reference's OWN code: the `nfsense`
package staged unmodified in baseline/_ref (tools/stage_reference.sh): `engine.recon_split`
(nfs/engine.py:182-241) with the pipeline's 2^28-byte blocks on a row sample of the
configuration (one CG iteration = one E^H E over those rows, read from its CGLog
`cg_iteration_1` label), extrapolated linearly to all K rows; plus a fully timed config-A
`recon_full` (20 iterations) next to the GPU's config-A solve.  Without baseline/_ref the
oracle port (oracle/nfs_oracle.py) stands in (`kind: "port"`).
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
REF_PKG = os.path.join(ROOT, "baseline", "_ref")

WORKLOADS = {
    "B": ("config B: 2D 256x256 single-shot spiral, L_R=41684 (disc mask), K=65536 samples "
          "(71.5 ms, R=4), 32 coils, B0 + 15 third-order field terms (P+1=16)"),
    "C": ("config C: stack of 40 config-B slices (z = +-39 mm, 2 mm apart; third-order harmonics at each "
          "slice's z), shared 65536-sample trajectory, 32 coils, P+1=16; slices are independent "
          "replicas across ranks (no collective)"),
    "D": ("config D: 3D 128x128x64 stack of 64 spirals, L_R=532872 (ellipsoid mask), K=299648 samples "
          "(R~7), 32 coils, B0 + 15 third-order field terms (P+1=16)"),
}
ITERS = {"B": 20, "C": 20, "D": 50}
N_SLICES = 40
METRIC = "E^H E applies/s"
FLUSH_BYTES = 256 << 20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def bench_config(cfg: str) -> dict:
    """The config dict both arms print (identical keys and values)."""
    return {"workload": WORKLOADS[cfg], "cg_iterations_e2e": ITERS[cfg],
            "l2": "flushed before every step (256 MiB device write outside the timed events)"}


def host_info() -> dict:
    info = {"cores": _NCPU}
    try:
        with open("/proc/cpuinfo") as fh:
            names = [ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")]
        info["cpu_model"] = names[0] if names else None
    except OSError:
        info["cpu_model"] = None
    try:
        import threadpoolctl
        info["threadpools"] = [{k: p.get(k) for k in ("internal_api", "num_threads", "version")}
                               for p in threadpoolctl.threadpool_info()]
    except Exception as exc:   # threadpoolctl missing: say so
        info["threadpools"] = f"unavailable: {exc}"
    return info


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

    def wait_first(self, timeout=3.0):
        t = time.perf_counter()
        while not self.rows and self.proc is not None and time.perf_counter() - t < timeout:
            time.sleep(0.01)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Samples taken inside [t0, t1] (the nearest three if the region is shorter than the
        sampling period)."""
        rows = [r for t, r in self.rows if t0 is None or t0 <= t <= t1]
        if not rows:
            rows = [r for _, r in sorted(self.rows, key=lambda tr: abs(tr[0] - (t0 or 0)))[:3]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU legs (reference code)
def load_reference():
    """The unmodified reference package from baseline/_ref, or None."""
    if os.path.isdir(os.path.join(REF_PKG, "nfsense")):
        if REF_PKG not in sys.path:
            sys.path.insert(0, REF_PKG)
        try:
            import nfsense.engine as ref_engine
            return ref_engine
        except Exception:
            return None
    return None


def _problem(cfg):
    """The configuration's problem; for C the most off-centre slice (z = +39 mm) stands for every
    slice (all slices have the same sizes and per-pair cost)."""
    from paper_2604_09233_b200 import simulate
    if cfg == "C":
        return simulate.make_slices(N_SLICES, which=[N_SLICES - 1])[0]
    return simulate.make_problem(cfg)


def cpu_apply_sample(prob, rows: int):
    """One E^H E of the reference over the first `rows` sample rows, through its own public API:
    recon_split (nfs/engine.py:182-241) with n_iter=1 and the pipeline's 2^28-byte blocks --
    its CGLog `cg_iteration_1` is exactly one blocked E^H E (phase blocks recomputed, as the
    reference does every iteration).  Returns (extrapolated full-K applies/s, sample seconds,
    kind)."""
    ref = load_reference()
    k_full = prob.temporal.shape[0]
    temporal = prob.temporal[:rows]
    sigma = np.zeros((rows, prob.sens.shape[1]), np.complex128)
    sigma[:, :] = 1.0 + 0.5j    # any finite data: the timed iteration's cost is data independent
    if ref is not None:
        starts = ref.choose_block_starts(rows, prob.spatial.shape[1], 2 ** 28)
        inputs = ref.EncodingInputs(sigma=sigma, spatial=prob.spatial, temporal=temporal, sens=prob.sens,
                                    intensity=prob.intensity, kfilter=None, mask_r=prob.mask_r,
                                    grid=_ref_grid(prob.grid), n_iter=1, block_starts=starts)
        _, log = ref.recon_split(inputs)
        dt = dict(log.timings)["cg_iteration_1"]
        kind = "reference"
    else:
        from oracle import nfs_oracle as orc   # CPU baseline leg only (no staged reference)
        s_eff = prob.sens * prob.intensity[:, None]
        starts = orc.choose_block_starts(rows, prob.spatial.shape[1], 2 ** 28)
        t0 = time.perf_counter()
        orc.split_normal_apply(prob.rho_true.astype(np.complex128), s_eff, prob.spatial, temporal, starts)
        dt = time.perf_counter() - t0
        kind = "port"
    return 1.0 / (dt * k_full / rows), dt, kind


def _ref_grid(grid):
    import nfsense
    return nfsense.Grid(grid.dims, grid.fov_m)


def cpu_config_a_recon():
    """A fully timed (not extrapolated) reference recon_full at config A, 20 iterations."""
    ref = load_reference()
    if ref is None:
        return None
    from paper_2604_09233_b200 import simulate
    prob = simulate.make_problem("A")
    sigma = config_a_sigma(prob)
    inputs = ref.EncodingInputs(sigma=sigma, spatial=prob.spatial, temporal=prob.temporal, sens=prob.sens,
                                intensity=prob.intensity, kfilter=None, mask_r=prob.mask_r,
                                grid=_ref_grid(prob.grid), n_iter=20)
    t0 = time.perf_counter()
    img, log = ref.recon_full(inputs)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "iterations": len(log.residual_norms),
            "api": "nfsense.engine.recon_full (baseline/_ref, unmodified reference)",
            "final_residual": float(log.residual_norms[-1])}


def config_a_sigma(prob):
    """Config A raw data: the golden fixture made by the reference's forward_signal."""
    return np.load(os.path.join(ROOT, "tests", "golden", "config_a.npz"))["sigma"]


def cpu_sample_rows(cfg):
    # a bounded sample of the workload: whole 2^28-byte phase blocks of the reference's
    # recon_split (402 rows each at config B/C), ~4 s of timed CPU E^H E per sample on the
    # 16-core GPU host (~7 s of wall time with the sample's initial adjoint; np.exp dominates,
    # single-threaded: SURVEY Appendix B), so the cpu_baseline leg (two samples) takes ~15 s and a
    # 20-step reference arm ~2.5 minutes
    return {"B": 10 * 402, "C": 10 * 402, "D": 256}[cfg]


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    prob = _problem(args.config)
    rows = cpu_sample_rows(args.config)
    if args.warmup > 0:
        cpu_apply_sample(prob, rows=min(rows, 64))
    vals, secs, kind = [], [], "port"
    for _ in range(args.steps):
        v, dt, kind = cpu_apply_sample(prob, rows)
        vals.append(v)
        secs.append(dt)
    value = float(np.median(vals))
    k = prob.temporal.shape[0]
    sample = (f"{rows} of {k} sample rows per step: reference recon_split, one CG iteration (one E^H E, "
              f"2^28-byte phase blocks) timed from its CGLog, extrapolated linearly to all rows; "
              f"numpy+OpenBLAS, {_NCPU} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "applies/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak" if args.config == "C" else "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": bench_config(args.config),
        "cpu_baseline": {"value": value, "unit": "applies/s", "cores": _NCPU, "kind": kind,
                         "sample": sample, "extrapolated": True},
        "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_seconds": secs,
        "host": host_info(),
    }
    if not args.no_config_a:
        line["config_a_recon"] = cpu_config_a_recon()
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def e2e_slices(args, engine, simulate, dist, world, rank, n_coils):
    """Config C end to end: the 40-slice stack through engine.recon_slices (slice i on rank
    i mod world, host arrays in and out); raw data of each slice synthesised once, outside the
    timing, by the FP64 device forward operator."""
    import torch
    from paper_2604_09233_b200 import _native
    slices = simulate.make_slices(N_SLICES)
    inputs = []
    for i, prob in enumerate(slices):
        sigma = np.zeros((prob.temporal.shape[0], n_coils), np.complex128)
        if i % world == rank:
            pl = _native.Plan(prob.temporal.shape[0], prob.spatial.shape[1], n_coils, prob.spatial.shape[0], "fp64",
                              int(os.environ.get("LOCAL_RANK", "0")))
            pl.set_tables(prob.temporal, prob.spatial)
            pl.set_sens(prob.sens)
            sigma = pl.apply_E(prob.rho_true)
            pl.close()
        inputs.append(engine.EncodingInputs(sigma=sigma, spatial=prob.spatial, temporal=prob.temporal,
                                            sens=prob.sens, intensity=prob.intensity, kfilter=None,
                                            mask_r=prob.mask_r, grid=prob.grid, n_iter=ITERS["C"]))
    times = []
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        out = engine.recon_slices(inputs, precision=args.precision, gather=world > 1)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    e2e_s = min(times)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    mine = [i for i in range(N_SLICES) if i % world == rank]
    iters = sum(len(out[i][1].residual_norms) for i in mine) * world
    per = inputs[0]
    h2d = len(mine) * (per.temporal.nbytes + per.spatial.nbytes + per.sens.nbytes + per.intensity.nbytes
                       + per.sigma.nbytes)
    rel = [float(np.linalg.norm(out[i][0].values[p.mask_r] - p.rho_true) / np.linalg.norm(p.rho_true))
           for i, p in zip(range(N_SLICES), slices) if out[i] is not None]
    return {"value": iters / e2e_s, "unit": "applies/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(len(mine) * (per.spatial.shape[1] * 16 + 16 * ITERS["C"])),
            "recon_seconds": e2e_s, "slices": N_SLICES, "cg_iterations": ITERS["C"],
            "api": "paper_2604_09233_b200.recon_slices (host numpy in/out, slices as replicas)",
            "rel_l2_vs_truth_max": max(rel) if rel else None}


def roofline_for(args, kern_ms, k_loc, L, G, P1, clocks, sustained_peak=False):
    pk = peaks()
    flops_1 = float(k_loc) * L * (8 * G + 2 * P1)      # SURVEY 8d F1 per operator launch
    dom = int(np.argmax(kern_ms))
    dom_ms = kern_ms[dom]
    if args.precision == "fp64":
        peak, bound, src = 148 * 64 * 2 * 1.965e9 / 1e12, "fp64", "nominal 148 SM x 64 FP64 FMA/clk x 2 x 1965 MHz"
    elif args.precision in ("f16x3", "tf32x3"):
        key = "bf16_tflops_sustained" if sustained_peak else "bf16_tflops"
        peak = pk.get(key, pk.get("bf16_tflops", 1590.0)) / (2 if args.precision == "tf32x3" else 1)
        bound = "tensor"
        src = f"MEASURED_PEAKS.json {key}" + (" / 2 (tf32)" if args.precision == "tf32x3" else
                                             " (fp16 MMA runs at the bf16 rate)")
    else:
        peak, bound = 148 * 128 * 2 * 1.965e9 / 1e12, "fp32"
        src = "nominal 148 SM x 128 FP32 lanes x 2 flop x 1965 MHz (no measured FP32-pipe figure)"
    achieved = flops_1 / (dom_ms * 1e-3) / 1e12
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "kernel": ["tci_kernel<32,fwd> (E)", "tci_kernel<32,adj> (E^H)"][dom] if args.precision == "f16x3"
            else ["forward contraction", "adjoint contraction"][dom],
            "kernel_ms": dom_ms, "kernel_ms_fwd_adj": list(kern_ms), "algorithmic_flop_per_launch": flops_1,
            "peak_source": src}
    if clocks.get("sm_mhz"):
        roof["frac_at_observed_clock"] = achieved / (peak * clocks["sm_mhz"] / 1965.0)
    if args.precision != "fp64":
        # the phasor costs 2 MUFU ops per (k, l) pair in every mode: the SFU floor (16 lane-ops
        # / clk / SM) bounds the launch from below whatever the tensor cores do (DESIGN 3.3)
        mufu_peak = 148 * 16 * 1.965e9
        roof["mufu_frac"] = 2.0 * float(k_loc) * L / (dom_ms * 1e-3) / mufu_peak
        roof["frac_ceiling_mufu"] = flops_1 / (2.0 * float(k_loc) * L / mufu_peak) / 1e12 / peak
        if clocks.get("sm_mhz"):
            roof["mufu_frac_at_observed_clock"] = roof["mufu_frac"] * 1965.0 / clocks["sm_mhz"]
    return roof


def traffic_for(args, dom):
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as fh:
            t = json.load(fh)
        return t.get(args.config, {}).get(args.precision, {}).get(["forward", "adjoint"][dom])
    except (OSError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=os.environ.get("NFS_BENCH_CONFIG", "B"), choices=["B", "C", "D"])
    ap.add_argument("--precision", default=os.environ.get("NFS_BENCH_PRECISION", "f16x3"),
                    choices=["f16x3", "tf32x3", "fp32", "fp64"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--sustain-seconds", type=float, default=3.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config-a", action="store_true")
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

    replicas = args.config == "C"   # slices: every rank runs whole, independent problems
    prob = _problem(args.config)
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
    lo, hi = (0, K) if replicas else engine.shard_rows(K, rank, world)

    plan = _native.Plan(hi - lo, L, G, P1, args.precision, local)
    stream = torch.cuda.Stream()
    plan.set_stream(stream.cuda_stream)
    if world > 1 and not replicas:
        plan.attach_comm(engine._nccl_unique_id(dist, rank), rank, world)
    plan.set_tables(prob.temporal[lo:hi], prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    # synthetic raw data = E rho_true through the device forward operator
    sigma = plan.apply_E(prob.rho_true / prob.intensity)
    plan.set_samples(sigma)
    plan.apply_EHE(prob.rho_true)   # places p on the device for the resident applies
    launches = plan.launches_per_apply()

    def run_e2e():
        """end-to-end through the public API (host arrays in, image out); run right after the
        timed steps, before the sustained leg heats the board to its power cap"""
        if replicas:
            e2e = e2e_slices(args, engine, simulate, dist, world, rank, G)
        else:
            inputs = engine.EncodingInputs(sigma=np.empty((K, G), np.complex128), spatial=prob.spatial,
                                           temporal=prob.temporal, sens=prob.sens,
                                           intensity=prob.intensity, kfilter=None, mask_r=prob.mask_r,
                                           grid=prob.grid, n_iter=ITERS[args.config])
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
            e2e = {"value": iters / e2e_s, "unit": "applies/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "recon_seconds": e2e_s, "cg_iterations": iters,
                   "api": "paper_2604_09233_b200.recon_full (host numpy in/out)",
                   "rel_l2_vs_truth": rel_truth}

        return e2e

    clk = ClockSampler(local).__enter__()   # sampling from before the warm-up
    try:
        clk.wait_first()
        with torch.cuda.stream(stream):
            plan.apply_EHE_resident(args.warmup)
            stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        step_ms, kern_ms = plan.bench_applies(args.steps, FLUSH_BYTES)   # events on the plan stream
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        if world > 1:
            dist.barrier()
        clocks = clk.summary(t_start, t_end)
        t_e0 = time.perf_counter()
        e2e = run_e2e()
        e2e["clocks"] = clk.summary(t_e0, time.perf_counter())
        # sustained: back-to-back applies (no flush) for a few seconds at the power-capped clock
        sus = None
        if args.sustain_seconds > 0:
            n_sus = max(1, int(args.sustain_seconds * 1e3 / max(np.mean(step_ms), 1e-3)))
            t0 = time.perf_counter()
            sus_steps, sus_kern = plan.bench_applies(n_sus, 0)
            t1 = time.perf_counter()
            sus = {"applies": n_sus, "ms_per_apply": float(np.mean(sus_steps)),
                   "applies_per_s": 1e3 / float(np.mean(sus_steps)),
                   "kernel_ms_fwd_adj": [k / n_sus for k in sus_kern],
                   "clocks": clk.summary(t0 + 0.25 * (t1 - t0), t1)}
    finally:
        clk.__exit__(None, None, None)
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1e3 / ms_per_step * (world if replicas else 1)   # replicas: every rank applies its own
    kern_mean = [k / args.steps for k in kern_ms]
    roofline = roofline_for(args, kern_mean, hi - lo, L, G, P1, clocks)
    roofline["traffic"] = traffic_for(args, int(np.argmax(kern_mean)))
    roofline["traffic_source"] = "profiles/r2_traffic.json (ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    roofline["kernel_share_of_step"] = float(sum(kern_mean) / ms_per_step)
    if sus is not None:
        sus["roofline"] = roofline_for(args, sus["kernel_ms_fwd_adj"], hi - lo, L, G, P1, sus["clocks"],
                                       sustained_peak=True)

    # config A through the public API, next to the reference arm's fully timed config-A solve
    cfg_a = None
    if rank == 0 and not args.no_config_a:
        pa = simulate.make_problem("A")
        ia = engine.EncodingInputs(sigma=config_a_sigma(pa), spatial=pa.spatial, temporal=pa.temporal,
                                   sens=pa.sens, intensity=pa.intensity, kfilter=None, mask_r=pa.mask_r,
                                   grid=pa.grid, n_iter=20)
        cfg_a = {"api": "paper_2604_09233_b200.recon_full (host numpy in/out, one GPU), best of 3"}
        for prec in dict.fromkeys(["fp64", args.precision]):   # fp64 = the reference's arithmetic
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                _, la = engine._recon_full(ia, None, prec, shard=False)
                ts.append(time.perf_counter() - t0)
            cfg_a[prec] = {"seconds": min(ts), "iterations": len(la.residual_norms),
                           "final_residual": float(la.residual_norms[-1])}
        cfg_a["seconds"] = cfg_a[args.precision]["seconds"]

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rows = cpu_sample_rows(args.config)
        runs = [cpu_apply_sample(prob, rows) for _ in range(2)]
        cpu = {"value": float(np.median([v for v, _, _ in runs])), "unit": "applies/s", "cores": _NCPU,
               "kind": runs[0][2], "extrapolated": True,
               "sample": (f"2 x {rows} of {K} sample rows of one E^H E ({sum(dt for _, dt, _ in runs):.1f} s "
                          "of CPU work), reference recon_split one CG iteration, 2^28-byte blocks, "
                          "extrapolated linearly to all rows")}
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak" if replicas else "strong", "vs_baseline": None,
            "dtype": {"fp32": "fp32", "fp64": "fp64", "tf32x3": "tf32x3 (fp32 accumulate)",
                      "f16x3": "f16x3 split contraction (exact int8 phase, fp32 accumulate)"}[args.precision],
            "data": "synthetic (disc phantom, synthetic coils, linear B0; raw data from the device forward model)",
            "config": bench_config(args.config),
            "precision": args.precision,
            "parallelism": (f"slice replicas x{world}" if replicas else f"sample-sharded x{world}")
                           if world > 1 else "1 GPU",
            "plan": plan.describe(),
            "roofline": roofline,
            "sustained": sus,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "config_a_recon": cfg_a,
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
            "step_ms_min_max": [float(np.min(step_ms)), float(np.max(step_ms))],
            "host": host_info() if cpu else None,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
