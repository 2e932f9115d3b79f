#!/usr/bin/env python
"""Benchmark of the DoGIP hot path (BASELINE.json metric: "DoGIP apply GDoF/s
and CG s/iter at 1/2/4/8 B200; fraction of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Workload: config C4 of BASELINE.json (3D unit cube, 128^3 cubes x 6 Kuhn tets =
12,582,912 tets, P3 scalar elliptic, isotropic log-normal per-cell coefficient,
zero Dirichlet, f = 1), split into z-slabs over the ranks (strong scaling).
One STEP = one conjugate-gradient iteration, i.e. one pass over every row of
the hot path: the DoGIP apply q = A p (gather, B-hat, A_T, B-hat^T, scatter
-- Algorithm 1) with the slab interface exchange, the two
dot products (all-reduced) and the three vector updates.  The weights are
computed once before timing (setup, reported as weights_ms).

value = apply throughput = global DoFs / apply time (GDoF/s, whole job, max
over ranks), measured with CUDA events around every apply inside the K timed
CG iterations; ms_per_step = device time of one CG iteration (max over ranks).
Inputs (21 GB of weights per GPU at N=1) are far larger than the 126 MB L2,
so no L2 flush is needed between iterations.

--impl reference: the CPU oracle (oracle/, plain NumPy) timed on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DoGIP apply GDoF/s and CG s/iter (fraction of HBM roofline)"
# DFMA throughput measured on this pool's B200 (scripts/fp64_pipes.cu, profiles/r01_fp64_pipes.json)
FP64_PEAK_TFLOPS = 35.9
UNIT = "GDoF/s"


def _measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic_from_profiles(cfg_name: str, n_gpus: int):
    """dram bytes per apply launch from a committed `ncu --set full` summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    v = j.get(f"{cfg_name}@{n_gpus}") or j.get(cfg_name)
    return None if v is None else float(v["dram_bytes_per_launch"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------- oracle arm
def oracle_sample_apply(cfg, n_cells: int, seed_offset: int = 0):
    """The oracle's element route (oracle/assemble.py: y = sum_T P_T^T K_T P_T u)
    on the d! n_cells elements of n_cells consecutive cells of the workload.
    Returns (elements processed, seconds)."""
    from oracle.assemble import ElementData
    from oracle.mesh import Mesh, cell_elements
    d, N, p = cfg.d, cfg.N, cfg.p
    ncell_tot = N ** d
    c0 = (seed_offset * n_cells) % max(1, ncell_tot - n_cells)
    cells = np.arange(c0, c0 + n_cells)
    elems = cell_elements(d, N, cells)
    M = N + 1
    vids = np.unique(elems)
    vlat = np.stack([(vids // M ** a) % M for a in range(d)], axis=1)
    verts = cfg.vertices()
    X = vlat / N if verts is None else verts[vids]
    remap = np.full(vids.max() + 1, -1, dtype=np.int64)
    remap[vids] = np.arange(vids.size)
    sub = Mesh(d, N, vlat, X, remap[elems], np.repeat(cells, 2 if d == 2 else 6))
    coef = _ORACLE_CACHE.setdefault(cfg.name, cfg.coefficient())
    u = _ORACLE_CACHE.setdefault(cfg.name + "u", cfg.u())
    t0 = time.perf_counter()
    ed = ElementData(sub, p)
    form = cfg.forms[0]
    y = np.zeros(ed.ndof)
    for sl in ed.chunks():
        K = ed.element_matrices(form, coef, sl)
        lT = ed.lT[sl]
        yl = np.einsum("eij,ej->ei", K, u[lT])
        np.add.at(y, lT.ravel(), yl.ravel())
    return sub.n_elem, time.perf_counter() - t0


_ORACLE_CACHE: dict = {}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, target_s: float = 12.0) -> dict:
    """Oracle throughput in the metric's unit on a bounded element sample."""
    oracle_sample_apply(cfg, 8)                                     # warm caches / imports
    ne, t = oracle_sample_apply(cfg, 256)
    per_elem = t / ne
    n_cells = int(max(256, min(cfg.N ** cfg.d, target_s / per_elem / (2 if cfg.d == 2 else 6))))
    ne, t = oracle_sample_apply(cfg, n_cells, 1)
    frac = ne / cfg.n_elem
    gdofs = cfg.ndof * frac / t / 1e9
    return {"value": gdofs, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"oracle element route (NumPy, single-threaded einsum) over {ne} of {cfg.n_elem} "
                      f"elements ({n_cells} cells) of {cfg.name}; GDoF/s = ndof * sampled fraction / time",
            "seconds": t}


def run_reference(args, cfg) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _ = oracle_sample_apply(cfg, 8)
    ne, t = oracle_sample_apply(cfg, 256)
    per_elem = t / ne
    per_step_target = max(1.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    n_cells = int(max(64, per_step_target / per_elem / (2 if cfg.d == 2 else 6)))
    for w in range(args.warmup):
        oracle_sample_apply(cfg, n_cells, w)
    times, nes = [], []
    for k in range(args.steps):
        ne, t = oracle_sample_apply(cfg, n_cells, args.warmup + k)
        times.append(t)
        nes.append(ne)
    tot = sum(times)
    frac = sum(nes) / cfg.n_elem
    value = cfg.ndof * frac / tot / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": _config_dict(cfg, args.gpus),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"each step: oracle element-route apply over {nes[0]} elements "
                                      f"({n_cells} cells) of {cfg.name}"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def _config_dict(cfg, n_gpus):
    form = "EL" if cfg.forms[0] == 1 else "WP"
    return {"workload": cfg.name, "description": cfg.description, "d": cfg.d, "N": cfg.N, "p": cfg.p,
            "form": form, "n_elem": cfg.n_elem, "ndof": cfg.ndof,
            "parallelism": f"z-slabs x{n_gpus}" if n_gpus > 1 else "single GPU",
            "l2": "inputs larger than L2 (weights stream > 126 MB per GPU); no flush",
            "step": "one CG iteration = DoGIP apply (+ slab exchange) + 2 all-reduced dots + 3 vector updates"}


# ----------------------------------------------------------------- product arm
def run_product(args, cfg) -> None:
    import torch
    import torch.distributed as dist

    from paper_1710_09913_b200.api import Mesh, Operator, kernel_launches, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nccl_id = None
    dist_on = world > 1 or args.dist     # --dist: the multi-rank path with a 1-rank NCCL group
    if dist_on:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    form = cfg.forms[0]
    dirichlet = form == 1
    coef = cfg.coefficient()
    mesh = Mesh(cfg.d, cfg.N, cfg.p, cfg.vertices(), rank=rank, nranks=world, nccl_id=nccl_id, device=local)
    storage = 1 if (args.storage == "iso" and form == 1) else 5 if (args.storage == "sym" and form == 0) else 0
    op = Operator(mesh, form, coef, storage=storage)
    info, oinfo = mesh.info, op.info
    stream = torch.cuda.current_stream()
    b = op.load_vector(1.0, dirichlet=dirichlet)
    x = torch.zeros_like(b)

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: W CG iterations (first call initialises r = b - A x, p = r)
    op.cg(b, x, maxit=-max(1, args.warmup), dirichlet=dirichlet)
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = op.cg(b, x, maxit=-args.steps, dirichlet=dirichlet, resume=True)
    e1.record(stream)
    barrier()
    launches = kernel_launches() - l0
    clocks = sampler.stop()
    t_step = e0.elapsed_time(e1) * 1e-3 / args.steps
    t_apply = res["apply_seconds"] / args.steps
    tt = torch.tensor([t_step, t_apply], dtype=torch.float64, device="cuda")
    if dist_on:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step_max, t_apply_max = tt.tolist()

    # algorithmic bytes of one apply on this rank: streamed weights of
    # real elements + u read once + y written once
    n_w = oinfo["W_T"] + oinfo["n_c"] if storage == 1 else oinfo["W_T"] * oinfo["n_c"]
    alg_bytes = 8 * n_w * info["n_elem_local"] + 16 * info["ndof_local"]
    flops_apply = oinfo["flops_per_elem"] * info["n_elem_local"]
    peak, peak_src = _measured_peaks()
    achieved = alg_bytes / t_apply / 1e9

    # e2e: host buffers through the public API (dogip_apply_host), copies inside
    u_host = torch.from_numpy(cfg.u()[info["dof_offset"]:info["dof_offset"] + info["ndof_local"]].copy()).pin_memory()
    y_host = torch.empty_like(u_host).pin_memory()
    ke = max(1, min(args.steps, 5))
    op.apply_host_ptr(u_host.data_ptr(), y_host.data_ptr(), dirichlet=dirichlet)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(ke):
        op.apply_host_ptr(u_host.data_ptr(), y_host.data_ptr(), dirichlet=dirichlet)
    f1.record(stream)
    barrier()
    t_e2e = torch.tensor([f0.elapsed_time(f1) * 1e-3 / ke], dtype=torch.float64, device="cuda")
    if dist_on:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    # e2e at the solver level: CG through the public API (dogip_cg) one iteration per call,
    # each call reading the residual back to the host (a convergence monitor); b copied
    # from pinned host memory before the first step, x copied back after the last
    b_host = torch.empty(info["ndof_local"], dtype=torch.float64).pin_memory()
    x_host = torch.empty_like(b_host).pin_memory()
    b_host.copy_(b.cpu())
    kc = max(2, args.steps)
    op.cg(b, x, maxit=1, rtol=0.0, dirichlet=dirichlet)    # builds / caches the single-rank graph
    barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    b.copy_(b_host, non_blocking=True)
    x.zero_()
    rels = []
    for k in range(kc):
        rr = op.cg(b, x, maxit=1, rtol=0.0, dirichlet=dirichlet, resume=k > 0)
        rels.append(rr["rel_res"])                 # host read of the step's result
    x_host.copy_(x, non_blocking=True)
    g1.record(stream)
    barrier()
    t_cg = torch.tensor([g0.elapsed_time(g1) * 1e-3 / kc], dtype=torch.float64, device="cuda")
    if dist_on:
        dist.all_reduce(t_cg, op=dist.ReduceOp.MAX)
    t_cg_e2e = t_cg.item()

    # secondary (not the headline): the isotropic compressed storage of the corollary
    # P:411-428 on the same workload -- FP64-bound instead of HBM-bound
    iso = None
    if form == 1 and storage == 0 and coef.isotropic and not args.no_variants:
        op.close()                      # free the full weights first (21 GB at N=1)
        torch.cuda.empty_cache()
        op2 = Operator(mesh, form, coef, storage=1)
        y2 = torch.empty_like(b)
        for _ in range(3):
            op2.apply(b, y2, dirichlet=dirichlet)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            op2.apply(b, y2, dirichlet=dirichlet)
        g1.record(stream)
        barrier()
        ti = torch.tensor([g0.elapsed_time(g1) * 1e-3 / args.steps], dtype=torch.float64, device="cuda")
        if dist_on:
            dist.all_reduce(ti, op=dist.ReduceOp.MAX)
        oi2 = op2.info
        t_iso = ti.item()
        iso = {"storage": "iso (a_{T,j} and G_T = R^-1 R^-T, P:411-428)", "apply_ms": t_iso * 1e3,
               "value": info["ndof_global"] / t_iso / 1e9, "unit": UNIT,
               "bound": "fp64", "fp64_tflops": oi2["flops_per_elem"] * info["n_elem_local"] / t_iso / 1e12,
               "fp64_frac_of_measured_dfma": oi2["flops_per_elem"] * info["n_elem_local"] / t_iso / 1e12 / FP64_PEAK_TFLOPS,
               "weights_ms": oi2["weights_ms"],
               "alg_bytes_per_launch": 8 * (oi2["W_T"] + oi2["n_c"]) * info["n_elem_local"] + 16 * info["ndof_local"]}
        op2.close()
    nbytes_vec = 8 * info["ndof_local"]
    tot_vec = torch.tensor([nbytes_vec], dtype=torch.float64, device="cuda")
    if dist_on:
        dist.all_reduce(tot_vec)

    if rank == 0:
        value = info["ndof_global"] / t_apply_max / 1e9
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": t_step_max * 1e3, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded GRF coefficient, u ~ U[-1,1]; no dataset in the paper)",
               "config": dict(_config_dict(cfg, world), storage=args.storage),
               "cg_s_per_iter": t_step_max, "apply_ms": t_apply_max * 1e3,
               "weights_ms": oinfo["weights_ms"], "cg_rel_res_after": res["rel_res"],
               "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": _traffic_from_profiles(cfg.name, world),
                            "kernel": "DoGIP apply (memset y + apply_kernel + Dirichlet fix-up), rank 0",
                            "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                            "frac_of_8TBs": achieved / 8000.0,
                            "fp64_tflops": flops_apply / t_apply / 1e12,
                            "fp64_frac_of_measured_dfma": flops_apply / t_apply / 1e12 / FP64_PEAK_TFLOPS},
               "e2e": {"value": info["ndof_global"] / t_e2e.item() / 1e9, "unit": UNIT,
                       "h2d_bytes_per_step": int(tot_vec.item()), "d2h_bytes_per_step": int(tot_vec.item()),
                       "api": "dogip_apply_host (pinned host u -> device, apply, device -> host y; "
                              "pipelined over 16 chunks of cube layers on copy-in / compute / copy-out "
                              "streams when single-rank)"},
               "e2e_cg": {"value": info["ndof_global"] / t_cg_e2e / 1e9, "unit": UNIT,
                          "s_per_iter": t_cg_e2e, "iters": kc,
                          "h2d_bytes_per_step": int(tot_vec.item()) // kc, "d2h_bytes_per_step": 8 + int(tot_vec.item()) // kc,
                          "api": "dogip_cg one iteration per call with the residual read back each step; "
                                 "b in from / x out to pinned host memory once per run (bytes amortised per step)"},
               "gpu_launches": int(launches),
               "clocks": clocks}
        if iso:
            out["variants"] = {"iso": iso}
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(out), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the secondary ISO-storage measurement")
    ap.add_argument("--dist", action="store_true",
                    help="initialise torch.distributed (NCCL) and the library communicator even at world "
                         "size 1: runs the multi-rank code path (exchange, all-reduces, max over ranks) on "
                         "one GPU with a 1-rank group, nothing waits on another rank")
    ap.add_argument("--storage", default="full", choices=["full", "iso", "sym"],
                    help="weight storage: full (P:281 / P:443), iso = EL isotropic compression of "
                         "the corollary P:411-428 (a_{T,j} R^-1 R^-T), sym = WP symmetry-adapted "
                         "(DOGIP_STORE_SYM, e.g. --config C5 --storage sym)")
    args = ap.parse_args()
    from synth.configs import get_config
    cfg = get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_product(args, cfg)


if __name__ == "__main__":
    main()
