#!/usr/bin/env python
"""Benchmark: Striped UniFrac full distance matrix on B200 (BASELINE.json metric).

Metric: node x pair updates/s (U = E * stripes * n, the reference's unit of
work, kernels.hpp:202-207) for a full distance matrix, plus full-DM seconds.
Default workload: C3, the 25k-sample EMP-shape synthetic (seed 3, n=25,000,
300,000-tip random tree, table density 0.002), unweighted, fp64.

One step = one full stripe computation on device from the resident problem:
zero stripes -> K1 embedding -> K2 stripe update -> K3 finalize. Inputs are
larger than L2 (the embedding alone is GBs), so no L2 flush is needed.
Multi-GPU (torchrun): stripes are split over ranks with the reference's
worker formula; no collective on the data path; time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
  python bench.py --impl reference ...   # the reference CPU path, rank 0 only
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c2": dict(seed=2, n=5000, leaves=50000, density=0.002, subset=0,
               metric="weighted-normalized", precision="fp64",
               workload="C2: WN fp64, synthetic 5k samples x 50k-tip random tree"),
    "c3": dict(seed=3, n=25000, leaves=300000, density=0.002, subset=0,
               metric="unweighted", precision="fp64",
               workload="C3: EMP-shape synthetic, 25k samples x 300k-tip tree, density 0.002, UW fp64"),
    "c3f32": dict(seed=3, n=25000, leaves=300000, density=0.002, subset=0,
                  metric="unweighted", precision="fp32",
                  workload="C3: EMP-shape synthetic, 25k samples x 300k-tip tree, density 0.002, UW fp32"),
    "c4": dict(seed=3, n=25000, leaves=300000, density=0.002, subset=0,
               metric="generalized", alpha=0.5, precision="fp64",
               workload="C4: generalized UniFrac alpha=0.5 fp64 on the C3 synthetic (25k samples x 300k tips)"),
    "c4f32": dict(seed=3, n=25000, leaves=300000, density=0.002, subset=0,
                  metric="generalized", alpha=0.5, precision="fp32",
                  workload="C4: generalized UniFrac alpha=0.5 fp32 on the C3 synthetic (25k samples x 300k tips)"),
    "c3wn": dict(seed=3, n=25000, leaves=300000, density=0.002, subset=0,
                 metric="weighted-normalized", precision="fp64",
                 workload="C3 shape, weighted normalized fp64 (25k samples x 300k tips)"),
    "c5": dict(seed=5, n=113721, leaves=300000, density=0.002, subset=0,
               metric="unweighted", precision="fp32",
               workload="C5: 113,721-sample synthetic, 300k-tip tree, density 0.002, UW fp32"),
    "small": dict(seed=7, n=4000, leaves=40000, density=0.002, subset=0,
                  metric="unweighted", precision="fp64", workload="small UW fp64 (quick check)"),
}
KERNELS = {"auto": 0, "dense": 1, "sparse": 2, "split": 10, "wsparse": 11, "uwalk": 12}
METRIC_CODE = {"unweighted": 1, "weighted-unnormalized": 2, "weighted-normalized": 3, "generalized": 4}
# algorithmic FP64/FP32 flops per update of update_entry (kernels.hpp:55-66),
# FMA counted as 2: UW = sub, fma, max, fma; WN = sub, fma, add, fma; WU = sub, fma
FLOPS_PER_UPDATE = {1: 6, 2: 3, 3: 6, 4: 7}  # generalized: add, sub, div, mul, fma, add + pow (counted as 1)

THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _pump(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[3], 16)
            except ValueError:
                continue
            for b, nm in THROTTLE_BITS.items():
                if bits & b and nm != "gpu_idle":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_problem(cfg):
    from paper_2005_05826_b200 import stripefrac as sf
    t0 = time.perf_counter()
    inst = sf.random_instance(cfg["seed"], cfg["n"], cfg["leaves"], cfg["density"], cfg["subset"],
                              finalize_tree=False)
    t1 = time.perf_counter()
    problem = sf.flatten(inst.tree, inst.table)
    t2 = time.perf_counter()
    log(f"instance: gen {t1 - t0:.1f}s flatten {t2 - t1:.1f}s  E={problem.n_rows} n={problem.n_samples} "
        f"nnz={problem.nnz}")
    return problem


def measured_fp_peak(device: int, prec: str) -> float:
    """FMA/s of this device's FP64 (or FP32) pipe from tools/fp_peaks.cu."""
    lib = C.CDLL(str(ROOT / "tools" / "libsf_peaks.so"))
    fn = lib.sfp_dfma_per_s if prec == "fp64" else lib.sfp_ffma_per_s
    fn.restype = C.c_double
    fn.argtypes = [C.c_int, C.c_int]
    return max(fn(device, 4000) for _ in range(3))


def run_ours(args, cfg):
    from paper_2005_05826_b200 import _native as N
    from paper_2005_05826_b200 import shard
    world, rank, local = dist_env()
    torch = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = N.lib()
    if L.sf_device_count() < 1:
        raise SystemExit("bench: no sm_100 device visible")
    metric = METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    problem = make_problem(cfg)
    n, E = problem.n_samples, problem.n_rows
    S = n // 2
    stop_all = min(S, args.stripes) if args.stripes else S
    a, b = shard.rank_range(0, stop_all, rank, world)
    kernel = KERNELS[args.kernel]
    ex, _keep = N.make_exec([local], kernel, alpha=cfg.get("alpha", 1.0))
    plan = C.c_void_p()
    t0 = time.perf_counter()
    N.check(L.sf_plan_create(problem.ref, metric, prec, a, b, C.byref(ex), C.byref(plan)))
    log(f"rank {rank}: plan stripes [{a},{b}) created in {time.perf_counter() - t0:.2f}s")
    st = N.sf_stats()

    def one_step():
        N.check(L.sf_plan_run(plan, 1))
        N.check(L.sf_plan_sync(plan))
        N.check(L.sf_plan_stats(plan, C.byref(st)))
        return st.total_ms, st.stripe_ms, st.embed_ms, st.updates_exec, st.launches, st.fp64_ops

    for i in range(args.warmup):
        r = one_step()
        log(f"rank {rank}: warmup {i}: {r[0]:.1f} ms (stripe {r[1]:.1f}, prep {r[2]:.1f})")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    dev_ms, str_ms, emb_ms, uexec, launches, fp64_ops = [], [], [], 0, 0, 0
    with ClockSampler(local) as clocks:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            tms, sms, ems, ue, ln, fo = one_step()
            dev_ms.append(tms)
            str_ms.append(sms)
            emb_ms.append(ems)
            uexec += ue
            launches += ln
            fp64_ops += fo
        barrier()
        wall = time.perf_counter() - w0
    total_dev_s = sum(dev_ms) / 1e3
    dev = "cuda" if world > 1 else None
    total_dev_s = shard.max_over_ranks(total_dev_s, dev)
    wall = shard.max_over_ranks(wall, dev)
    uexec_all = shard.sum_over_ranks(float(uexec), dev)
    u_alg_step = E * stop_all * n
    value = u_alg_step * args.steps / total_dev_s
    ms_per_step = total_dev_s * 1e3 / args.steps

    L.sf_plan_destroy(plan)  # free the resident plan before the end-to-end calls
    plan = None

    # ---- e2e through the public C ABI: host problem in, host stripes out
    e2e = None
    if not args.no_e2e:
        import torch as _t
        w = 8 if prec == 8 else 4
        dt = _t.float64 if prec == 8 else _t.float32
        dist_h = _t.empty(((b - a) * n,), dtype=dt, pin_memory=True).numpy()
        tot_h = _t.empty(((b - a) * n,), dtype=dt, pin_memory=True).numpy() if metric != 2 else None
        st2 = N.sf_stats()
        times = []
        # one untimed call first (first-touch of the pinned pages, allocator)
        N.check(L.sf_compute_stripes(problem.ref, metric, prec, a, b, N.ptr(dist_h),
                                     N.ptr(tot_h) if tot_h is not None else None, 1,
                                     C.byref(ex), C.byref(st2)))
        for _ in range(max(1, args.e2e_steps)):
            barrier()
            t1 = time.perf_counter()
            N.check(L.sf_compute_stripes(problem.ref, metric, prec, a, b, N.ptr(dist_h),
                                         N.ptr(tot_h) if tot_h is not None else None, 1,
                                         C.byref(ex), C.byref(st2)))
            times.append(time.perf_counter() - t1)
        e2e_s = max(times) if len(times) == 1 else statistics.median(times)
        e2e_s = shard.max_over_ranks(e2e_s, "cuda" if world > 1 else None)
        h2d = (problem.parent_row.nbytes + problem.lengths.nbytes + problem.leaf_feature.nbytes +
               problem.feat_ptr.nbytes + problem.sample_idx.nbytes + problem.counts.nbytes +
               problem.sample_totals.nbytes)
        d2h = (b - a) * n * w * (2 if metric != 2 else 1)
        e2e = {"value": u_alg_step / e2e_s, "unit": "updates/s", "seconds_per_dm": e2e_s,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return None

    # ---- roofline of the dominant kernel (K2 stripe update)
    # the split kernel (unweighted) accumulates exact limbs with DFMA in every
    # output precision: its pipe is FP64 for the fp32 lines too
    peak_fma = measured_fp_peak(local, "fp64" if (metric == 1 and fp64_ops > 0) else cfg["precision"])
    stripe_s = sum(str_ms) / 1e3
    peak_tf = peak_fma * 2 / 1e12
    if metric == 1 and fp64_ops > 0:
        # split kernel (10): the heavy walk issues 2 DFMA (4 flops) per u bit per
        # live slot; the kernel counts them (stats.fp64_ops = DFMA lane-ops)
        achieved_tf = fp64_ops * 2 / stripe_s / 1e12 if stripe_s else 0.0
        roofline = {
            "bound": "fp64", "achieved": round(achieved_tf, 3), "peak": round(peak_tf, 3),
            "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4) if peak_tf else None,
            # dram__bytes_read+write of one `ncu --set full` capture of this kernel
            # (profiles/r01_ncu_split_c3_1024stripes.txt: 0.685 GB + 0.406 GB for
            # 1024 stripes at C3, heavy threshold 0.03), per launch: scaled by
            # the stripes it covers
            "traffic": (round((0.685215e9 + 0.406339e9) / 1024 * stop_all / max(world, 1))
                        if cfg is CONFIGS["c3"] else None),
            "traffic_unit": "bytes per launch",
            "kernel": "stripe_split_kernel (heavy-row walk)",
            "peak_source": "measured DFMA loop (tools/fp_peaks.cu) on this device, x2 flops/FMA",
            "work": "fp64_ops = DFMA lane-ops counted by the kernel (2 per u bit per live slot)",
            "dfma_per_step": int(fp64_ops / args.steps),
            "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "prep_ms_per_step": round(sum(emb_ms) / args.steps, 3),
            "algorithmic_speedup_vs_dense_fp64_roofline": round(
                (E * stop_all * n * args.steps / (sum(dev_ms) / 1e3)) / (peak_fma / 4), 2),
        }
    else:
        fl = FLOPS_PER_UPDATE[metric]
        achieved_tf = (uexec / max(world, 1) if world > 1 else uexec) * fl / stripe_s / 1e12 if stripe_s else 0.0
        roofline = {
            "bound": "fp64" if prec == 8 else "fp32",
            "achieved": round(achieved_tf, 3), "peak": round(peak_tf, 3), "unit": "TFLOP/s",
            "frac": round(achieved_tf / peak_tf, 4) if peak_tf else None, "traffic": None,
            "kernel": ("stripe_dense_kernel" if kernel == 1 else
                       "stripe_wsparse_kernel (present-row walk)" if metric != 1 else "stripe walk"),
            "peak_source": "measured DFMA/FFMA loop (tools/fp_peaks.cu) on this device",
            "flops_per_update": fl, "updates_exec_per_step": int(uexec_all / args.steps),
            "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "embed_ms_per_step": round(sum(emb_ms) / args.steps, 3),
        }

    # ---- CPU baseline (oracle restatement, bounded sample, all host threads)
    cpu = None
    if not args.no_cpu_baseline and world == 1 and metric != 4:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_port
        threads = os.cpu_count() or 1
        rows = 64
        stripes = max(1, min(S, 64))
        secs, upd = oracle_port.time_sample(problem, metric, prec, rows, 0, stripes, threads)
        # scale the sample toward ~10 s of CPU work
        scale = max(1, min(S // stripes, int(10.0 / max(secs, 1e-3))))
        if scale > 1:
            stripes = min(S, stripes * scale)
            secs, upd = oracle_port.time_sample(problem, metric, prec, rows, 0, stripes, threads)
        cpu = {"value": upd / secs, "unit": "updates/s", "cores": threads, "kind": "port",
               "sample": f"first {rows} postorder rows x stripes [0,{stripes}) x {n} samples "
                         f"({upd:.3g} updates, {secs:.2f}s), oracle/stripefrac_oracle.c, -O2 no FMA"}

    clk = clocks.summary()
    line = {
        "metric": "UniFrac node x pair updates/s (full distance matrix)",
        "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "full_dm_seconds": ms_per_step / 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if prec == 8 else "f32", "data": "synthetic (reference random_instance, seeded)",
        "config": {"workload": cfg["workload"], "seed": cfg["seed"], "n_samples": n,
                   "tree_tips": cfg["leaves"], "rows_E": E, "density": cfg["density"],
                   "metric": cfg["metric"], "stripes": [0, stop_all],
                   **({"alpha": cfg["alpha"]} if "alpha" in cfg else {}),
                   "parallelism": f"stripe-range x{world}", "kernel": args.kernel,
                   "l2": "inputs larger than L2 (no flush)"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": int(launches), "wall_seconds_timed": wall,
    }
    if world > 1:
        torch.distributed.destroy_process_group()
    return line


def run_reference(args, cfg):
    """The reference's own CPU implementation (oracle/_ref/ref_driver, built
    from the reference sources) on a bounded sample, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    metric = cfg["metric"]
    if metric == "generalized":
        return {"impl": "reference", "unavailable": "the reference implements no generalized UniFrac "
                                                    "(common.hpp:19); C4 is an extension"}
    n = cfg["n"]
    threads = os.cpu_count() or 1
    driver = ROOT / "oracle" / "_ref" / "ref_driver"
    stripes = max(1, min(n // 2, args.ref_stripes))
    reps = args.warmup + args.steps
    if driver.exists():
        cmd = [str(driver), "bench", str(cfg["seed"]), str(n), str(cfg["leaves"]), str(cfg["density"]),
               str(cfg["subset"]), metric, cfg["precision"], str(stripes), str(reps), str(threads), "64"]
        log("reference:", " ".join(cmd))
        out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
        rec = json.loads(out.strip().splitlines()[-1])
        secs = rec["seconds"][args.warmup:] or rec["seconds"]
        upd = rec["updates_per_rep"]
        kind = "reference"
        sample = (f"reference compute_unifrac hot loop (Embedder::next_batch + accumulate_stripes, "
                  f"{threads} std::threads): one 64-row batch x stripes [0,{stripes}) x {n} samples "
                  f"per step; setup (instance + Embedder) {rec['setup_s']:.1f}s untimed")
    else:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_port
        problem = make_problem(cfg)
        secs = []
        upd = 0
        for i in range(reps):
            s, upd = oracle_port.time_sample(problem, METRIC_CODE[metric],
                                             8 if cfg["precision"] == "fp64" else 4, 64, 0, stripes, threads)
            if i >= args.warmup:
                secs.append(s)
        kind = "port"
        sample = f"oracle port: 64 rows x stripes [0,{stripes}) x {n} samples per step"
    med = statistics.median(secs)
    value = upd / med
    return {
        "impl": "reference", "metric": "UniFrac node x pair updates/s (full distance matrix)",
        "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if cfg["precision"] == "fp64" else "f32",
        "data": "synthetic (reference random_instance, seeded)",
        "config": {"workload": cfg["workload"], "seed": cfg["seed"], "n_samples": n,
                   "tree_tips": cfg["leaves"], "density": cfg["density"], "metric": metric,
                   "parallelism": f"{threads} CPU threads"},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--kernel", choices=sorted(KERNELS), default="auto")
    ap.add_argument("--stripes", type=int, default=0, help="limit to stripes [0, N) (debug)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-stripes", type=int, default=256)
    args = ap.parse_args()
    if args.warmup < 3 and not os.environ.get("BENCH_ALLOW_SHORT"):
        args.warmup = 3
    cfg = CONFIGS[args.config]
    line = run_reference(args, cfg) if args.impl == "reference" else run_ours(args, cfg)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
