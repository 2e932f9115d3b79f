#!/usr/bin/env python
"""Per-config measurements on one GPU (DESIGN.md tables): apply time, algorithmic
GB/s and fraction of the measured HBM copy bandwidth, CG s/iter, and the full CG
solves BASELINE.json asks for (C1 EL Dirichlet 1e-10, C3 EL Dirichlet 1e-10,
C5 WP mass 1e-12), each followed by a GPU-side true-residual check.

    python scripts/config_sweep.py [--configs C1,C2p1,...] [--solve] [--iters 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_09913_b200.api import Mesh, Operator  # noqa: E402
from synth.configs import get_config  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def time_apply(op, u, y, n, dirichlet):
    s = torch.cuda.current_stream()
    for _ in range(3):
        op.apply(u, y, dirichlet=dirichlet)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        op.apply(u, y, dirichlet=dirichlet)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / n


_FLUSH = None


def time_apply_flushed(op, u, y, n, dirichlet):
    """Median per-apply time with the L2 (126 MB) flushed before every call by writing a
    256 MB buffer -- the HBM number for inputs that would otherwise stay L2-resident."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(n):
        _FLUSH.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        op.apply(u, y, dirichlet=dirichlet)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def graph_latency(op, u, y, dirichlet, reps=200):
    """Device latency of one apply replayed from a CUDA graph."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        op.apply(u, y, dirichlet=dirichlet, stream=s)       # configure before capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            op.apply(u, y, dirichlet=dirichlet, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2p1,C2p2,C2p3,C2p4,C3,C4,C5")
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--iso", action="store_true", help="also the isotropic compressed EL storage")
    ap.add_argument("--qp", action="store_true", help="also the quadrature-point matrix-free comparator")
    args = ap.parse_args()
    rows = []
    for name in args.configs.split(","):
        c = get_config(name)
        forms = c.forms
        t0 = time.time()
        coef = c.coefficient()
        mesh = Mesh(c.d, c.N, c.p, c.vertices())
        variants = [(f, 0) for f in forms]
        if args.iso and coef.isotropic and 1 in forms:
            variants.append((1, 1))
        if args.iso and 0 in forms and c.p <= 4:
            variants.append((0, 2))
        if args.iso and 0 in forms:
            variants += [(0, 5)]
        if args.qp:
            variants += [(f, 4) for f in forms]
        for form, storage in variants:
            op = Operator(mesh, form, coef, storage=storage)
            oi = op.info
            u = torch.from_numpy(c.u()).cuda()
            y = torch.empty_like(u)
            dirichlet = form == 1
            n = args.iters if c.ndof > 1e6 else 200
            t_apply = time_apply(op, u, y, n, dirichlet)
            t_flush = time_apply_flushed(op, u, y, 9, dirichlet) if c.ndof < 3e7 else None
            t_graph = graph_latency(op, u, y, dirichlet) if c.ndof < 1e5 else None
            nw = oi["W_T"] + oi["n_c"] if storage == 1 else oi["W_T"] * oi["n_c"]
            alg = 8 * nw * c.n_elem + 16 * c.ndof
            if storage == 2:                      # global W vector read once (Theorem 1)
                alg = 8 * (2 * c.p * c.N + 1) ** c.d + 16 * c.ndof
            if storage == 4:                      # comparator: no stored operator data
                alg = 16 * c.ndof
            b = op.load_vector(1.0, dirichlet=dirichlet)
            x = torch.zeros_like(b)
            op.cg(b, x, maxit=-3, dirichlet=dirichlet)
            r = op.cg(b, x, maxit=-n, dirichlet=dirichlet, resume=True)
            row = {"config": name, "form": (["WP", "EL", "EL-iso", "WP-glob"][form if storage == 0 else storage + 1]
                             if storage not in (4, 5) else (["WP-qp", "EL-qp"][form] if storage == 4 else "WP-sym")),
                   "d": c.d, "N": c.N, "p": c.p, "flops_per_elem": oi["flops_per_elem"],
                   "fp64_TFs": oi["flops_per_elem"] * c.n_elem / t_apply / 1e12,
                   "n_elem": c.n_elem, "ndof": c.ndof, "W_T": oi["W_T"], "n_c": oi["n_c"],
                   "weights_GB": oi["weight_bytes"] / 1e9, "weights_ms": oi["weights_ms"],
                   "apply_ms": t_apply * 1e3, "GDoF_s": c.ndof / t_apply / 1e9,
                   "alg_GB": alg / 1e9, "alg_GBs": alg / t_apply / 1e9, "frac_measured": alg / t_apply / 1e9 / PEAK,
                   "cg_ms_per_iter": r["seconds"] / n * 1e3, "cg_apply_ms": r["apply_seconds"] / n * 1e3}
            if t_flush is not None:       # L2 flushed before each apply (median of 9)
                row.update({"apply_ms_l2flushed": t_flush * 1e3, "frac_l2flushed": alg / t_flush / 1e9 / PEAK})
            if t_graph is not None:
                row["apply_graph_latency_us"] = t_graph * 1e6
            if args.solve and (name in ("C1", "C3", "C5")) and (name != "C1" or form == 1):
                tol = 1e-12 if name == "C5" else 1e-10
                x = torch.zeros_like(b)
                res = op.cg(b, x, rtol=tol, maxit=200000, dirichlet=dirichlet)
                yx = op.apply(x, dirichlet=dirichlet)
                true_res = (torch.linalg.vector_norm(b - yx) / torch.linalg.vector_norm(b)).item()
                row.update({"solve_tol": tol, "solve_iters": res["iters"], "solve_status": res["status"],
                            "solve_rel_res": res["rel_res"], "solve_true_rel_res": true_res,
                            "solve_s": res["seconds"]})
            row["wall_s"] = time.time() - t0
            print(json.dumps(row), flush=True)
            rows.append(row)
            op.close()
            del u, y, b, x
            torch.cuda.empty_cache()
        mesh.close()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
