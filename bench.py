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
KERNELS = {"auto": 0, "dense": 1, "sparse": 2, "split": 10, "wsparse": 11, "uwalk": 12, "wsplit": 13}
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

    def __init__(self, index):
        self.index = index if isinstance(index, str) else str(index)
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.index,
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


def host_description() -> dict:
    """CPU model, host threads and RAM of the machine the CPU legs ran on."""
    model, ram = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 1048576, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count(), "ram_gib": ram}


def resolve_devices(gpus: int, world: int, visible: int):
    """Devices this process drives. Under torchrun each rank drives its
    LOCAL_RANK device (returns None) and --gpus must equal WORLD_SIZE; a
    single process with --gpus N > 1 shards the stripes over devices
    0..N-1 in-process (sf_exec.devices). Asking for more GPUs than are
    visible fails loudly."""
    if gpus < 1:
        raise SystemExit(f"bench: --gpus must be >= 1 (got {gpus})")
    if world > 1:
        if gpus != world:
            raise SystemExit(f"bench: --gpus {gpus} but WORLD_SIZE={world}: launch one rank per GPU")
        return None
    if gpus > visible:
        raise SystemExit(f"bench: --gpus {gpus} requested but only {visible} sm_100 device(s) are visible")
    return list(range(gpus))


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


def ncu_traffic(cfg_name: str, kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of the dominant kernel from the committed `ncu --set full` capture of
    this config (profiles/ncu_traffic.json, written by tools/ncu_summary.py
    --traffic), with the stripes it covered; None when there is none."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    rec = json.loads(p.read_text()).get(f"{cfg_name}:{kernel}")
    return rec


def run_ours(args, cfg):
    from paper_2005_05826_b200 import _native as N
    from paper_2005_05826_b200 import shard
    world, rank, local = dist_env()
    torch = None
    t_ctx = time.perf_counter()
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = N.lib()
    visible = L.sf_device_count()  # first CUDA call of the process: context creation
    t_ctx = time.perf_counter() - t_ctx
    if visible < 1:
        raise SystemExit("bench: no sm_100 device visible")
    devices = resolve_devices(args.gpus, world, visible)
    my_devs = devices if devices is not None else [local]
    n_gpus = world if world > 1 else len(my_devs)
    metric = METRIC_CODE[cfg["metric"]]
    prec = 8 if cfg["precision"] == "fp64" else 4
    problem = make_problem(cfg)
    n, E = problem.n_samples, problem.n_rows
    S = n // 2
    stop_all = min(S, args.stripes) if args.stripes else S
    a, b = shard.rank_range(0, stop_all, rank, world)
    kernel = KERNELS[args.kernel]
    ex, _keep = N.make_exec(my_devs, kernel, alpha=cfg.get("alpha", 1.0))
    plan = C.c_void_p()
    t0 = time.perf_counter()
    N.check(L.sf_plan_create(problem.ref, metric, prec, a, b, C.byref(ex), C.byref(plan)))
    cold_plan_s = time.perf_counter() - t0
    log(f"rank {rank}: plan stripes [{a},{b}) on devices {my_devs} created in {cold_plan_s:.2f}s "
        f"(context {t_ctx:.2f}s)")
    st = N.sf_stats()
    tens = []  # (tensor ops, tensor ms) per step

    def one_step():
        w0 = time.perf_counter()
        N.check(L.sf_plan_run(plan, 1))
        N.check(L.sf_plan_sync(plan))
        wall_ms = (time.perf_counter() - w0) * 1e3
        N.check(L.sf_plan_stats(plan, C.byref(st)))
        tens.append((st.tensor_ops, st.tensor_ms))
        return st.total_ms, st.stripe_ms, st.embed_ms, st.updates_exec, st.launches, st.fp64_ops, wall_ms

    for i in range(args.warmup):
        r = one_step()
        log(f"rank {rank}: warmup {i}: {r[0]:.1f} ms (stripe {r[1]:.1f}, prep {r[2]:.1f}, host wall {r[6]:.1f})")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    tens.clear()
    dev_ms, str_ms, emb_ms, wall_ms, uexec, launches, fp64_ops = [], [], [], [], 0, 0, 0
    with ClockSampler(",".join(str(d) for d in my_devs)) as clocks:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            tms, sms, ems, ue, ln, fo, wms = one_step()
            dev_ms.append(tms)
            str_ms.append(sms)
            emb_ms.append(ems)
            wall_ms.append(wms)
            uexec += ue
            launches += ln
            fp64_ops += fo
        barrier()
        wall = time.perf_counter() - w0
    # one device: CUDA events on the plan's stream; several devices in one
    # process: the host clock around run + sync (it includes the launch
    # stagger between devices, which per-device events would hide); torchrun:
    # each rank's device time, max over ranks
    step_s = (sum(wall_ms) if len(my_devs) > 1 else sum(dev_ms)) / 1e3
    dev = "cuda" if world > 1 else None
    total_dev_s = shard.max_over_ranks(step_s, dev)
    wall = shard.max_over_ranks(wall, dev)
    uexec_all = shard.sum_over_ranks(float(uexec), dev)
    u_alg_step = E * stop_all * n
    value = u_alg_step * args.steps / total_dev_s
    ms_per_step = total_dev_s * 1e3 / args.steps

    L.sf_plan_destroy(plan)  # free the resident plan before the end-to-end calls
    plan = None

    # ---- e2e through the public C ABI: host problem in, host stripes out
    e2e = None
    dm_leg = None
    if not args.no_e2e:
        w = 8 if prec == 8 else 4
        dist_h = pinned_empty((b - a) * n, prec)
        tot_h = pinned_empty((b - a) * n, prec) if metric != 2 else None
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
               "calls": len(times), "host_buffers": "pinned",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        del dist_h, tot_h
        # compute_distance_matrix (kernels.hpp:319-326) into a pageable n x n
        # matrix (what the C++/Python API hands out): condense on device
        if world == 1 and not args.stripes and metric != 4 and not args.no_dm:
            mat = np.empty((n, n), dtype=np.float64)
            tms = []
            for i in range(3):
                t1 = time.perf_counter()
                N.check(L.sf_compute_distance_matrix(problem.ref, metric, prec, N.ptr(mat), C.byref(ex),
                                                     C.byref(st2)))
                tms.append(time.perf_counter() - t1)
            dm_leg = {"seconds": statistics.median(tms[1:]), "first_call_seconds": tms[0],
                      "host_buffer": "pageable n x n fp64", "bytes_d2h": n * n * 8,
                      "api": "sf_compute_distance_matrix (stripes stay on device; condense on device)"}
            del mat

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return None

    roofline = roofline_record(args, cfg, metric, prec, my_devs[0], world, stop_all, E, n, str_ms, emb_ms,
                               dev_ms, fp64_ops, uexec, uexec_all, kernel, tens)

    # ---- CPU baseline (oracle restatement, bounded sample, all host threads)
    cpu = None
    if not args.no_cpu_baseline and world == 1 and len(my_devs) == 1 and metric != 4:
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
                         f"({upd:.3g} updates, {secs:.2f}s), oracle/stripefrac_oracle.c, -O2 no FMA",
               "host": host_description()}

    clk = clocks.summary()
    line = {
        "metric": "UniFrac node x pair updates/s (full distance matrix)",
        "value": value, "unit": "updates/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        # host to host, in-memory problem -> finalized stripes in host memory
        "full_dm_seconds": e2e["seconds_per_dm"] if e2e else None,
        "device_seconds_per_dm": ms_per_step / 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if prec == 8 else "f32", "data": "synthetic (reference random_instance, seeded)",
        "config": {"workload": cfg["workload"], "seed": cfg["seed"], "n_samples": n,
                   "tree_tips": cfg["leaves"], "rows_E": E, "density": cfg["density"],
                   "metric": cfg["metric"], "stripes": [0, stop_all],
                   **({"alpha": cfg["alpha"]} if "alpha" in cfg else {}),
                   "parallelism": (f"stripe ranges over {world} ranks (torchrun, one GPU each)" if world > 1
                                   else f"stripe ranges over {len(my_devs)} device(s) in one process"),
                   "kernel": args.kernel, "l2": "inputs larger than L2 (no flush)",
                   "step_timer": ("CUDA events (max over ranks)" if len(my_devs) == 1
                                  else "host clock around run+sync over all devices")},
        "e2e": e2e, "distance_matrix_e2e": dm_leg, "roofline": roofline, "cpu_baseline": cpu,
        "clocks": clk, "gpu_launches": int(launches), "wall_seconds_timed": wall,
        "cold_start": {"context_init_seconds": round(t_ctx, 3), "first_plan_create_seconds": round(cold_plan_s, 3),
                       "note": "first CUDA call + first plan of the process (pool, module load, first "
                               "allocations); the e2e calls above are warm"},
    }
    if world > 1:
        torch.distributed.destroy_process_group()
    return line


def pinned_empty(count: int, prec: int):
    import torch as _t
    dt = _t.float64 if prec == 8 else _t.float32
    return _t.empty((count,), dtype=dt, pin_memory=True).numpy()


def measured_int8_peak() -> dict:
    """Dense int8 tensor-core peak measured live on this device: cuBLASLt's
    int8 GEMM (torch._int_mm) at a large square-ish shape, best of 5."""
    import torch
    M, K, N = 8192, 65536, 8192
    a = torch.ones((M, K), dtype=torch.int8, device="cuda")
    b = torch.ones((K, N), dtype=torch.int8, device="cuda").t().contiguous().t()
    torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    torch.cuda.empty_cache()
    return {"tops": 2 * M * K * N / best / 1e9, "shape": f"{M}x{K}x{N}"}


def roofline_record(args, cfg, metric, prec, device, world, stop_all, E, n, str_ms, emb_ms, dev_ms, fp64_ops,
                    uexec, uexec_all, kernel, tens):
    """The dominant kernel's roofline (rank 0's share of the work)."""
    stripe_s = sum(str_ms) / 1e3
    cfg_name = args.config
    t_ops = sum(o for o, _ in tens)
    t_ms = sum(m for _, m in tens)
    if metric == 1 and t_ops > 0 and t_ms > 0:
        # split kernel (10), heavy rows on the int8 tensor cores: the GEMMs'
        # ops (2 per MAC over the M x W x K rectangles issued) / their
        # CUDA-event time, against the dense int8 peak measured live
        pk = measured_int8_peak()
        achieved = t_ops / (t_ms / 1e3) / 1e12
        bf16 = None
        try:
            bf16 = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("bf16_tflops")
        except (OSError, ValueError):
            pass
        tr = ncu_traffic(cfg_name, "heavy_gemm")
        return {
            "bound": "tensor", "achieved": round(achieved, 1), "peak": round(pk["tops"], 1),
            "unit": "TFLOP/s", "unit_note": "int8 tensor-core ops (MAC = 2), exact integer accumulation",
            "frac": round(achieved / pk["tops"], 4),
            "traffic": (round(tr["dram_bytes"] / tr["launches"]) if tr else None),
            "traffic_unit": "DRAM bytes per heavy GEMM launch (dram__bytes_read.sum + dram__bytes_write.sum)",
            "traffic_source": (f"{tr['source']} ({tr['launches']} launches of the {tr['stripes']}-stripe run)"
                               if tr else None),
            "kernel": "heavy-row int8 digit-plane GEMMs (cuBLASLt IMMA, tcgen05) of the split path",
            "largest_kernel_note": ("at C3 the light column kernel (sp_light_column_kernel, ~48% of the "
                                    "step in the ncu launch list) takes longer than the GEMMs (~29%); it is "
                                    "bound by the L1 data pipe (shared-memory atomics: 90% of cycles, "
                                    "profiles/r02_ncu_light_column_c3_v3.txt), which has no HBM or tensor "
                                    "roofline; the frac above is the GEMMs'"),
            "peak_source": (f"cuBLASLt int8 GEMM {pk['shape']} measured live on this device (best of 5)"
                            + (f"; MEASURED_PEAKS bf16 {bf16} TF/s x2 = {2 * bf16:.0f} for reference" if bf16 else "")),
            "tensor_ops_per_step": int(t_ops / args.steps),
            "gemm_ms_per_step": round(t_ms / args.steps, 3),
            "heavy_phase_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "prep_light_ms_per_step": round(sum(emb_ms) / args.steps, 3),
            "algorithmic_speedup_vs_dense_fp64_roofline": round(
                (E * stop_all * n * args.steps / (sum(dev_ms) / 1e3)) / (measured_fp_peak(device, "fp64") / 4), 2),
        }
    if metric == 1 and fp64_ops > 0:
        # split kernel (10): the heavy walk issues 2 DFMA (4 flops) per u bit
        # per live slot, counted by the kernel (stats.fp64_ops = DFMA lane-ops);
        # it accumulates exact limbs with DFMA in every output precision
        peak_fma = measured_fp_peak(device, "fp64")
        peak_tf = peak_fma * 2 / 1e12
        achieved_tf = fp64_ops * 2 / stripe_s / 1e12 if stripe_s else 0.0
        tr = ncu_traffic(cfg_name, "stripe_split_kernel")
        traffic = None
        if tr:  # per launch of the bench's step: scale the capture's stripes to this launch
            traffic = round(tr["dram_bytes"] / tr["stripes"] * (stop_all / max(world, 1)))
        return {
            "bound": "fp64", "achieved": round(achieved_tf, 3), "peak": round(peak_tf, 3),
            "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4) if peak_tf else None,
            "traffic": traffic, "traffic_unit": "DRAM bytes per launch",
            "traffic_source": (f"{tr['source']} ({tr['stripes']} stripes, scaled per stripe)" if tr else None),
            "kernel": "stripe_split_kernel (heavy-row walk, kernel 10)",
            "peak_source": "measured DFMA loop (tools/fp_peaks.cu) on this device, x2 flops/FMA",
            "work": "fp64_ops = DFMA lane-ops counted by the kernel (2 per u bit per live slot)",
            "dfma_per_step": int(fp64_ops / args.steps),
            "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "prep_ms_per_step": round(sum(emb_ms) / args.steps, 3),
            "algorithmic_speedup_vs_dense_fp64_roofline": round(
                (E * stop_all * n * args.steps / (sum(dev_ms) / 1e3)) / (peak_fma / 4), 2),
        }
    if metric != 1 and t_ms > 0 and fp64_ops > 0:
        # weighted split (13): the dense heavy-row kernel's FP64-pipe (fp32:
        # FP32-pipe) instructions, counted per (heavy row, slot) from its SASS
        # (WN/WU: DADD + DFMA; generalized alpha = 0.5: 14), over its CUDA-event
        # time, against the measured FMA-instruction peak of that pipe
        pipe = "fp64" if prec == 8 else "fp32"
        peak_fma = measured_fp_peak(device, pipe)
        rate = fp64_ops / (t_ms / 1e3)
        tr = ncu_traffic(cfg_name, "wx_dense_kernel")
        return {
            "bound": pipe, "achieved": round(rate * 2 / 1e12, 3), "peak": round(peak_fma * 2 / 1e12, 3),
            "unit": "TFLOP/s", "frac": round(rate / peak_fma, 4) if peak_fma else None,
            "unit_note": ("FMA-equivalent: pipe instructions x 2 (WN/WU: each (heavy row, slot) is a DADD + a "
                          "DFMA, |u - v| an operand modifier), so frac = the pipe's issue fraction"),
            "traffic": round(tr["dram_bytes"] / tr["stripes"] * (stop_all / max(world, 1))) if tr else None,
            "traffic_unit": "DRAM bytes per launch",
            "traffic_source": (f"{tr['source']} ({tr['stripes']} stripes, scaled per stripe)" if tr else None),
            "kernel": "wx_dense_kernel (weighted split, kernel 13: heavy rows dense)",
            "peak_source": "measured DFMA/FFMA loop (tools/fp_peaks.cu) on this device, x2 flops/FMA",
            "pipe_ops_per_step": int(fp64_ops / args.steps),
            "dense_ms_per_step": round(t_ms / args.steps, 3),
            "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "prep_ms_per_step": round(sum(emb_ms) / args.steps, 3),
        }
    if metric != 1 and fp64_ops > 0:
        # u-walk (12): the kernel counts the FP64-pipe instructions x live
        # lanes it issues (its accumulators are fp64 in both precisions)
        peak_fma = measured_fp_peak(device, "fp64")
        peak_tf = peak_fma * 2 / 1e12
        achieved_tf = fp64_ops * 2 / stripe_s / 1e12 if stripe_s else 0.0
        tr = ncu_traffic(cfg_name, "stripe_wuwalk_kernel")
        return {
            "bound": "fp64", "achieved": round(achieved_tf, 3),
            "peak": round(peak_tf, 3), "unit": "TFLOP/s",
            "frac": round(achieved_tf / peak_tf, 4) if peak_tf else None,
            "traffic": round(tr["dram_bytes"] / tr["stripes"] * stop_all) if tr else None,
            "traffic_unit": "DRAM bytes per launch",
            "traffic_source": (f"{tr['source']} ({tr['stripes']} stripes, scaled per stripe)" if tr else None),
            "kernel": "stripe_wuwalk_kernel (u-walk, kernel 12)",
            "peak_source": "measured DFMA/FFMA loop (tools/fp_peaks.cu) on this device, x2 flops/FMA",
            "work": ("fp64_ops = FP64-pipe instructions x live lanes counted by the kernel (1 DFMA per u row "
                     "and slot, 8 per shared row), reported as 2 flops each against the DFMA peak"),
            "fma_per_step": int(fp64_ops / args.steps),
            "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
            "prep_ms_per_step": round(sum(emb_ms) / args.steps, 3),
        }
    peak_fma = measured_fp_peak(device, "fp64" if prec == 8 else "fp32")
    peak_tf = peak_fma * 2 / 1e12
    fl = FLOPS_PER_UPDATE[metric]
    achieved_tf = (uexec / max(world, 1) if world > 1 else uexec) * fl / stripe_s / 1e12 if stripe_s else 0.0
    return {
        "bound": "fp64" if prec == 8 else "fp32",
        "achieved": round(achieved_tf, 3), "peak": round(peak_tf, 3), "unit": "TFLOP/s",
        "frac": round(achieved_tf / peak_tf, 4) if peak_tf else None, "traffic": None,
        "kernel": {1: "stripe_dense_kernel", 2: "stripe_sparse_kernel", 11: "stripe_wsparse_kernel"}.get(kernel,
                                                                                                       "auto"),
        "peak_source": "measured DFMA/FFMA loop (tools/fp_peaks.cu) on this device",
        "flops_per_update": fl, "updates_exec_per_step": int(uexec_all / args.steps),
        "stripe_ms_per_step": round(stripe_s * 1e3 / args.steps, 3),
        "embed_ms_per_step": round(sum(emb_ms) / args.steps, 3),
    }


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
        sample = (f"reference compute_unifrac hot loop, timed per step: Embedder::next_batch + cast_batch + "
                  f"accumulate_stripes over {threads} std::threads, one 64-row batch x stripes [0,{stripes}) x "
                  f"{n} samples; setup (instance + Embedder ctor) {rec['setup_s']:.1f}s untimed")
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
                         "sample": sample, "host": host_description()},
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
    ap.add_argument("--no-dm", action="store_true", help="skip the compute_distance_matrix leg")
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
