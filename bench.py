#!/usr/bin/env python
"""Benchmark of the B200 multi-RHS Laplacian solve path (BASELINE.json metric:
"multi-RHS Laplacian solves/s to ref tol; V-cycle HBM GB/s vs B200 peak").

A step is one pass of the hot path over one batch: the fused JL closeness
estimate of the configuration (seeded Q generated on device, right-hand
sides formed and centred, k solves to tau, distance-sum reduction for the
query nodes).  ``value`` = right-hand sides solved per second over the whole
job, inputs (graph, hierarchy) resident in HBM.  ``e2e`` = the same metric
through the reference-facing API ``solve_many`` with host supplies (the same
centred JL right-hand sides): host->device copy of the supplies and
device->host copy of the solutions inside the timed region.

Default workload is C2 (BASELINE.json configs[1]); ``--config c1..c5``
selects another.  Multi-GPU (torchrun): every rank owns a disjoint range of
k sketch rows (weak scaling), one all-reduce of the per-query partial sums.

``--impl reference`` times the reference algorithm's CPU implementation
(the oracle port of pkg/src/cfcent, oracle/lamg_oracle.py -- the reference
itself is pure Python and cannot be shipped to the GPU box) on the host
cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-RHS Laplacian solves/s to ref tol; V-cycle HBM GB/s vs B200 peak"
L2_REF_GBS = 6300 * 1.965  # full-chip L2 (LTS) throughput reference, GB/s


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region:
    NVML polled every 5 ms from a thread (so even a 50 ms region gets samples),
    falling back to `nvidia-smi -lms 200` when NVML is unavailable.  The GPU is
    addressed by the visible device's PCI bus id."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, int]] = []
        self.smax = 0.0
        self._stop = threading.Event()
        self._nv = None

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self._h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._nv = nv
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self._nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))))
            except Exception:
                pass
            self._stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self._nv is not None and self.samples:
            nv = self._nv
            reasons = set()
            for _, r in self.samples:
                for name, attr in self.REASONS:
                    if r & getattr(nv, attr, 0):
                        reasons.add(name)
            return {"sm_mhz": float(np.median([c for c, _ in self.samples])),
                    "sm_max_mhz": self.smax, "reasons": sorted(reasons),
                    "samples": len(self.samples), "source": "nvml 5 ms"}
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi 200 ms"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def row_range(k: int, world: int, rank: int):
    return (k * rank) // world, (k * (rank + 1)) // world


# ---------------------------------------------------------------------------
# reference arm (CPU)
# ---------------------------------------------------------------------------

def cpu_reference(cfgname: str, columns: int, budget_s: float, threads: int):
    """Time the reference algorithm (oracle port) on the host: solves of the
    configuration's centred JL right-hand sides, 64-column blocks over
    ``threads`` workers exactly like solver.py:771-811."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import lamg_oracle as O
    from paper_1607_02955_b200 import configs

    sys.setrecursionlimit(20000)
    bc = configs.make(cfgname)
    g = bc.graph
    og = (np.asarray(g.indptr), np.asarray(g.indices), np.asarray(g.weights))
    t0 = time.perf_counter()
    h = O.build_hierarchy(O.laplacian(og), O.OracleConfig(tau=bc.tau))
    setup_s = time.perf_counter() - t0
    _, rhs = O.jl_rhs(og, bc.jl_k, bc.jl_seed)
    cols = min(columns, rhs.shape[0])
    sample = rhs[:cols]
    blocks = [(lo, min(lo + 64, cols)) for lo in range(0, cols, 64)]
    nthreads = max(1, min(threads, len(blocks)))

    def run(b):
        O.solve_columns(h, sample[b[0]:b[1]].T)

    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        if nthreads > 1:
            with ThreadPoolExecutor(nthreads) as ex:
                list(ex.map(run, blocks))
        else:
            for b in blocks:
                run(b)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    per = float(np.mean(times))
    return {"value": cols / per, "unit": "solves/s", "cores": nthreads, "kind": "port",
            "workload": f"{bc.name.upper()}: {bc.description}", "n": g.n, "m": g.m,
            "sample": f"{cols} of {bc.jl_k} {cfgname.upper()} JL right-hand sides "
                      f"(tau {bc.tau:g}), {len(blocks)} x 64-column blocks, "
                      f"{len(times)} timed repetition(s); oracle port of pkg/src/cfcent",
            "setup_s": setup_s, "steps_timed": len(times), "s_per_step": per}


# Bounded CPU samples per configuration (columns of the JL batch).  The
# reference algorithm's own setup on the R-MAT graphs runs for hours (C4: 831
# levels / 1,108 s in SURVEY.md A.2 with its stalled coarsening), so C4/C5
# have no CPU sample.
CPU_COLUMNS = {"c1": 64, "c2": 64, "c3": 4}
REF_COLUMNS = {"c1": 64, "c2": 128, "c3": 8}
CPU_UNAVAILABLE = ("reference setup on this R-MAT graph stalls into hundreds of levels "
                   "(SURVEY.md A.2: 831 levels / 1,108 s on C4); no bounded CPU sample")


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if args.config not in REF_COLUMNS:
        print(json.dumps({"impl": "reference", "metric": METRIC, "unit": "solves/s",
                          "unavailable": CPU_UNAVAILABLE}), flush=True)
        return
    threads = len(os.sched_getaffinity(0))
    r = cpu_reference(args.config, min(args.ref_columns, REF_COLUMNS[args.config]),
                      args.ref_budget, threads)
    line = {"metric": METRIC, "value": r["value"], "unit": "solves/s", "n_gpus": args.gpus,
            "steps": r["steps_timed"], "warmup": 0, "ms_per_step": r["s_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d) recipes)", "impl": "reference",
            "config": {"workload": r["workload"], "n": r["n"], "m": r["m"],
                       "rhs_per_step": args.ref_columns},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "solves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "setup_s": r["setup_s"]}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm (GPU)
# ---------------------------------------------------------------------------

def run_gpu_arm(args):
    import torch

    import paper_1607_02955_b200 as P
    from paper_1607_02955_b200 import configs
    from paper_1607_02955_b200.resistance import jl_rhs_rows, sketch_closeness_sums
    from paper_1607_02955_b200.solver import set_device

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t0 = time.perf_counter()
    bc = configs.make(args.config)
    gen_s = time.perf_counter() - t0
    g = bc.graph
    cfg = P.SolverConfig(tau=bc.tau)
    t0 = time.perf_counter()
    h = P.setup(P.laplacian(g), cfg)
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev = h.device()
    upload_s = time.perf_counter() - t0
    k = bc.jl_k
    r0, r1 = row_range(k * world, world, rank)  # weak scaling: k rows per rank
    K_total = k * world
    eps = math.sqrt(math.log(g.n) / (K_total - 0.5))
    stream = torch.cuda.ExternalStream(h.stream_ptr())

    def step():
        _, sums, res = sketch_closeness_sums(g, h, eps, bc.jl_seed, bc.query, cfg, rows=(r0, r1))
        return sums, res

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        step()
    st0 = h.stats.vcycles
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            sums, res = step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    vcyc = (h.stats.vcycles - st0) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        s = torch.tensor(sums, device="cuda", dtype=torch.float64)
        dist.all_reduce(s)
        sums = s.cpu().numpy()
    n = g.n
    scores = (n - 1) / sums
    solves = (r1 - r0) * world
    value = solves / (ms / 1e3)

    # --- per-kernel profile of one step (eager launches bracketed by events)
    dev_h = h
    dev_h.profile(True)
    step()
    rep = dev_h.profile_report()
    dev_h.profile(False)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"profile_{args.config}_rank{rank}.txt"), "w") as f:
        f.write("kind level launches total_ms alg_bytes alg_GB/s gather_bytes gather_GB/s\n")
        for kind, lv, la, kms, by, gb in sorted(rep, key=lambda r: -r[3]):
            f.write(f"{kind} {lv} {la} {kms:.4f} {by:.0f} {by / max(kms, 1e-9) / 1e6:.1f} "
                    f"{gb:.0f} {gb / max(kms, 1e-9) / 1e6:.1f}\n")
    kinds = {}
    inst = {}
    launches = 0
    ginst = {}
    for kind, lv, la, kms, by, gb in rep:
        a = kinds.setdefault(kind, [0, 0.0, 0.0])
        a[0] += la
        a[1] += kms
        a[2] += by
        inst[f"{kind}@L{lv}"] = (la, kms, by)
        ginst[f"{kind}@L{lv}"] = gb
        if kind != "memset":
            launches += la
    prof_ms = sum(v[1] for v in kinds.values())
    # dominant kernel instance: (kind, level) with the largest total time
    dom_name, (dom_la, dom_ms, dom_by) = max(inst.items(), key=lambda kv: kv[1][1])
    peak, peak_src = _peaks()
    dom_bytes_per_launch = dom_by / dom_la
    dom_ms_per_launch = dom_ms / dom_la
    achieved = dom_bytes_per_launch / (dom_ms_per_launch * 1e-3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get(dom_name)
    total_bytes = sum(v[2] for v in kinds.values())

    # --- e2e through the public API with host buffers (same right-hand sides)
    rhs = jl_rhs_rows(g, h, K_total, bc.jl_seed, row0=r0, rows=r1 - r0)
    rhs -= rhs.mean(axis=1, keepdims=True)
    # supplies and result buffer in page-locked host memory (allocated once,
    # outside the timed region); the copies themselves are timed every step
    rhs_pin = torch.empty(rhs.shape, dtype=torch.float64, pin_memory=True).numpy()
    rhs_pin[...] = rhs
    rhs = rhs_pin
    out_pin = torch.empty(rhs.shape, dtype=torch.float64, pin_memory=True).numpy()
    P.solve_many(h, rhs, cfg, out=out_pin)  # warm
    barrier()
    torch.cuda.synchronize()
    e2 = []
    for _ in range(max(1, min(args.steps, 5))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        P.solve_many(h, rhs, cfg, out=out_pin)
        b.record(stream)
        torch.cuda.synchronize()
        e2.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = solves / (e2e_ms / 1e3)
    h2d = rhs.nbytes
    d2h = rhs.nbytes + 8 * rhs.shape[0]

    # sampling estimator (configs that name one): pivots + query solved in one batch
    sampling = None
    if bc.sampling_pivots and world == 1:
        P.cf_closeness_sampling(g, h, bc.sampling_query, bc.sampling_pivots, bc.sampling_seed, cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tab = P.cf_closeness_sampling(g, h, bc.sampling_query, bc.sampling_pivots,
                                      bc.sampling_seed, cfg)
        b.record(stream)
        torch.cuda.synchronize()
        sms = a.elapsed_time(b)
        nsolve = len(set(P.pivot_set(g.n, bc.sampling_pivots, bc.sampling_seed).tolist())
                     | set(bc.sampling_query))
        sampling = {"pivots": bc.sampling_pivots, "rhs": nsolve, "seconds_per_estimate": sms / 1e3,
                    "solves_per_s": nsolve / (sms / 1e3),
                    "score_first_query": float(tab.vector(bc.sampling_query[:1])[0])}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config in CPU_COLUMNS:
            cpu = cpu_reference(args.config, min(args.cpu_columns, CPU_COLUMNS[args.config]),
                                args.cpu_budget, 1)
            cpu = {k_: cpu[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
        else:
            cpu = {"value": None, "unit": "solves/s", "cores": 0, "kind": "port",
                   "sample": "none", "unavailable": CPU_UNAVAILABLE}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md §8(d) recipes)",
            "config": {"workload": f"{bc.name.upper()}: {bc.description}", "n": n, "m": g.m,
                       "rhs_per_step": solves, "levels": len(h.levels),
                       "parallelism": f"sketch rows sharded over {world} GPU(s)",
                       "l2": "working set (per-level b,x blocks) larger than the 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom_name,
                         "peak_source": peak_src,
                         "bytes_per_launch": dom_bytes_per_launch,
                         "ms_per_launch": dom_ms_per_launch,
                         "gather_bytes_per_launch": ginst[dom_name] / dom_la,
                         "gather_gbs": ginst[dom_name] / dom_la / (dom_ms_per_launch * 1e-3) / 1e9,
                         "l2_ref_gbs": L2_REF_GBS,
                         "l2_ref_source": "B300_MICROARCH.md LTS cap ~6300 B/clk x 1.965 GHz "
                                          "(B300-measured; B200 assumed similar)",
                         # measured DRAM bytes (ncu, per launch) over the live launch time
                         "dram_gbs": (traffic / (dom_ms_per_launch * 1e-3) / 1e9
                                      if traffic else None),
                         "dram_frac": (traffic / (dom_ms_per_launch * 1e-3) / 1e9 / peak
                                       if traffic else None)},
            "step_hbm_gbs": total_bytes / (prof_ms * 1e-3) / 1e9 if prof_ms > 0 else None,
            "cpu_baseline": cpu,
            "sampling": sampling,
            "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "solve_many (pinned host supplies and out=)"},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "vcycles_per_rhs": vcyc / max(1, r1 - r0),
            "vcycles_per_s": vcyc / (ms / 1e3) * world,
            "seconds_per_estimate": ms / 1e3,
            "setup_s": setup_s, "upload_s": upload_s, "graph_gen_s": gen_s,
            "max_residual": float(np.max(res)) if len(res) else 0.0,
            "score_first_query": float(scores[0]),
            "kernel_share": {kk: round(v[1] / prof_ms, 4) for kk, v in
                             sorted(kinds.items(), key=lambda kv: -kv[1][1])},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--cpu-columns", type=int, default=64)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-columns", type=int, default=128)
    ap.add_argument("--ref-budget", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
