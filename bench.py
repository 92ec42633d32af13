#!/usr/bin/env python
"""Benchmark of the Householder-product apply hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {hh,reference}]
                    [--workload C2|C1|C3|C4|C5h12|C5h64|C5h256|C5h1024|KNN|CONG|QR4095|SHF|U<n>H<h>] [--op N|T]

Default workload = BASELINE.json configs[1] (the metric's config): Y = H1...Hh X,
fp32, n=1024, h=10, N=262144 columns (1 GiB in, 1 GiB out; larger than the 126 MB
L2, so no flush is needed between steps).  One step = one hh_apply launch over the
whole batch.  metric = algorithmic GB/s (one read + one write of X per step),
whole job, max-over-ranks device time.  Rank 0 prints ONE JSON line.

Multi-GPU (torchrun): weak scaling, each rank applies Q to its own full-size batch;
no collective on the data path (columns are independent).
`--impl reference`: the fp64 C oracle (oracle/) on the host cores, timed per step on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gen import inputs as gi  # noqa: E402

METRIC = "H1…Hh·X GB/s and % of HBM roofline (n=1024,h=10,fp32); vectors/s"
FALLBACK_HBM = 6650.0


def workload_case(name: str, N_override=None):
    name = name.upper()
    if name == "C1":
        return gi.make_config(1, N=N_override)
    if name == "C2":
        return gi.make_config(2, N=N_override)
    if name == "C3":
        return gi.make_config(3, N=N_override)
    if name == "C4":
        return gi.make_config(4, N=N_override)
    if name.startswith("C5H"):
        return gi.make_config(5, h=int(name[3:]), N=N_override)
    if name == "KNN":   # NEXT-f3, Table-I-shaped (MNIST after PCA) synthetic stand-in
        return gi.make_knn_case()
    if name == "CONG":   # NEXT-f4: SHF congruences op(Q) M op(Q)^T, 64 matrices of n = 512, h = 18
        n, h, cnt = 512, 18, 64   # h = ceil(2 log2 n): the middle of Table I's h range
        g = gi.rng(600, n, h, cnt)
        c = gi.make_case("apply", n, h, 1, "f32", seed=60)
        c.U = gi.unit_reflectors(g, h, n, "f32")
        c.X = gi.gaussian_columns(g, cnt * n, n, "f32")     # (count * n, n) == count n x n matrices
        c.N, c.call, c.name, c.count = cnt * n, "congruence", "CONG", cnt
        return c
    if name == "SHF":   # NEXT-f4: C(u) and grad C for 256 candidates of one (A_k, B_k), n = 1024
        n, K = 1024, 256
        g = gi.rng(610, n, K)
        c = gi.make_case("apply", n, 1, 1, "f32", seed=61)
        A = g.standard_normal((n, n))
        B = g.standard_normal((n, n))
        c.X = ((A + A.T) / 2).astype(np.float32)          # A_k (symmetric)
        c.d = ((B + B.T) / 2).astype(np.float32)          # B_k (symmetric)
        c.U = gi.unit_reflectors(g, K, n, "f32")          # the candidates u (K, n)
        c.N, c.h, c.call, c.name, c.K = K, 0, "shf", "SHF", K
        return c
    if name.startswith("QR"):   # NEXT-f2: n=4096, h = n-1 partial-QR reflectors (C5's X)
        h = int(name[2:]) if len(name) > 2 else 4095
        c = gi.make_config(5, h=min(h, 1024), N=N_override)
        c.U = gi.qr_reflectors(gi.rng(5, h, 9), h, c.n, "f32")
        c.h, c.call, c.name = h, "apply_qr", f"QR{h}"
        return c
    if name.startswith("U") and "H" in name:   # context: an unaligned column stride, e.g. U1023H10
        n, h = (int(v) for v in name[1:].split("H"))   # 1 GiB of X; K1r / K1g / the padded detour
        return gi.make_case("apply", n, h, N_override or (1 << 28) // n, "f32", seed=70)
    raise SystemExit(f"unknown workload {name}")


def alg_cost(c, op_count=1):
    """Algorithmic bytes and flops of one step."""
    s = 4 if c.dtype == "f32" else 8
    if c.call == "knn":
        Mq = c.lam.shape[0]
        byts = (c.N + Mq) * c.n * s + Mq * c.k * 8           # points read once + results
        flops = 4 * c.h * c.n * (c.N + Mq) + 2 * c.n * c.N * Mq   # transform once + dots
        return byts, flops, Mq
    if c.call == "shf":   # A, B, the candidates read once; C and grad C written; 8 n^2 K flops
        byts = (2 * c.n * c.n + 2 * c.n * c.K + c.K) * s
        flops = 8 * c.n * c.n * c.K
        return byts, flops, c.K
    if c.call == "congruence":   # op(Q) M op(Q)^T: M read once, written once; 2 x 4hn per column
        byts = 2 * c.count * c.n * c.n * s
        flops = 2 * 4 * c.h * c.n * c.n * c.count
        return byts, flops, c.count
    if c.call == "mahalanobis":
        P = c.npairs
        byts = c.N * c.n * s + 2 * P * 4 + P * s          # points once + indices + dist
        flops = 4 * c.h * c.n * c.N + 3 * c.n * P          # transform-once reading (R11)
        units = P
    elif c.call == "sym":
        byts = 2 * c.N * c.n * s
        flops = (8 * c.h + 1) * c.n * c.N
        units = c.N
    elif c.call == "apply_qr":   # 4(n-k+1) per reflector, k = 1..h
        byts = 2 * c.N * c.n * s
        flops = sum(4 * (c.n - k) for k in range(c.h)) * c.N
        units = c.N
    else:
        byts = 2 * c.N * c.n * s
        flops = 4 * c.h * c.n * c.N
        units = c.N
    return byts, flops, units


def input_digest(c) -> str:
    """SHA-256 of the exact input bytes (U, X, lambda, d, ia, ib as present): the oracle and
    the GPU path provably saw the same inputs."""
    import hashlib
    hsh = hashlib.sha256()
    for nm in ("U", "X", "lam", "d", "ia", "ib"):
        a = getattr(c, nm, None)
        if a is not None:
            hsh.update(nm.encode())
            hsh.update(np.ascontiguousarray(a).tobytes())
    return hsh.hexdigest()


def same_run_copy_gbs(dev) -> float:
    """A 1 GiB device-to-device copy timed in this run (context for the roofline peak, which
    stays the driver-measured MEASURED_PEAKS.json figure)."""
    import torch
    a = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    b = torch.empty_like(a)
    b.copy_(a)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize(dev)
    gbs = 2 * a.numel() * 4 * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del a, b
    return gbs


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def rd():
            for line in self.proc.stdout:
                self.rows.append((time.time(), line.strip()))
        self.t = threading.Thread(target=rd, daemon=True)
        self.t.start()
        return self

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 <= t <= t1] or [r for (_, r) in self.rows]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    from paper_1811_07624_b200 import dist as hd
    return hd.env()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_oracle(c, op, target_s=10.0, max_cols=None):
    """Oracle (as it stands) on a bounded column / pair sample; returns (value GB/s,
    units/s, seconds, sample description, threads, k, out) -- `out` is the oracle's result
    for the first k units (all of them when the budget allows), reused for parity."""
    import oracle
    threads = oracle.num_threads()
    byts, flops, units = alg_cost(c)
    per_unit_bytes = byts / units
    res = {}

    def run(k):
        t0 = time.perf_counter()
        if c.call == "knn":
            res["out"] = oracle.knn(c.U, c.d, c.X, c.lam[:k], c.k)
        elif c.call == "shf":
            res["out"] = oracle.shf_cost(c.X, c.d, c.U[:k])
        elif c.call == "congruence":
            res["out"] = oracle.congruence(op, c.U, c.X[:k * c.n].reshape(k, c.n, c.n))
        elif c.call == "mahalanobis":
            res["out"] = oracle.mahalanobis(c.U, c.d, c.X, c.ia[:k], c.ib[:k])
        elif c.call == "sym":
            res["out"] = oracle.sym_apply(c.U, c.lam, c.X[:k])
        else:
            res["out"] = oracle.apply(op, c.U, c.X[:k])   # apply_qr: the plain apply (same U)
        return time.perf_counter() - t0

    total = units
    k = min(total, {"mahalanobis": 2048, "knn": 4, "congruence": 1, "shf": 64}.get(c.call, 256))
    dt = run(k)
    while dt < 0.5 and k < total:
        k = min(total, k * 4)
        dt = run(k)
    k2 = min(total, max(k, int(k * target_s / max(dt, 1e-6))))
    if max_cols:
        k2 = min(k2, max_cols)
    if k2 != k:
        dt = run(k2)
        k = k2
    what = {"mahalanobis": "pairs", "knn": "queries", "congruence": "matrices",
            "shf": "candidates"}.get(c.call, "columns")
    return (per_unit_bytes * k / dt / 1e9, k / dt, dt,
            f"{k} of {total} {what} of {c.name} (fp64 oracle, {threads} threads)", threads, k,
            res["out"])


def parity_of(c, k, ref, Y, dist_out, knn_out, dev):
    """Parity of the GPU result against the oracle's output for the first k units (the
    cpu_baseline run's own output): whole relative l2 error and the per-unit maximum, gated
    like tests/test_fullsize_gpu.py."""
    import torch
    g = 1e-12 if c.dtype == "f64" else 2e-5 * math.sqrt(max(c.h, 1))
    if c.call == "knn":
        ri, rd = ref
        gi_, gd_ = knn_out
        got = gd_[:k].double().cpu().numpy()
        e = float(np.linalg.norm(got - rd) / np.linalg.norm(rd))
        return {"rel_l2_dist": e, "index_agreement": float((gi_[:k].cpu().numpy() == ri).mean()),
                "gate": g, "sampled": int(k), "of": int(c.lam.shape[0]),
                "pass": bool(e <= g)}
    if c.call == "shf":   # reading R21: each candidate against the size of its terms
        cost, grad = knn_out
        c_ref, g_ref = ref
        A64, B64, U64 = (x.astype(np.float64) for x in (c.X, c.d, c.U[:k]))
        a, b = U64 @ A64, U64 @ B64
        al, be = np.sum(U64 * a, 1), np.sum(U64 * b, 1)
        na, nb = np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1)
        g = 1e-6 * math.sqrt(c.n)
        ec = np.abs(cost[:k].double().cpu().numpy() - c_ref) / (2 * na * nb + 2 * np.abs(al * be))
        sg = 2 * (np.linalg.norm(A64) * nb + np.linalg.norm(B64) * na) + 4 * (np.abs(al) * nb + np.abs(be) * na)
        eg = np.linalg.norm(grad[:k].double().cpu().numpy() - g_ref, axis=1) / sg
        return {"max_rel_cost": float(ec.max()), "max_rel_grad": float(eg.max()), "gate": g,
                "sampled": int(k), "of": int(c.K), "pass": bool(ec.max() <= g and eg.max() <= g)}
    if c.call == "congruence":
        got = Y[:k * c.n].double().cpu().numpy().reshape(ref.shape)
        e = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        return {"rel_fro": e, "gate": g, "sampled": int(k), "of": int(c.count), "pass": bool(e <= g)}
    if c.call == "mahalanobis":
        got = dist_out[:k].double().cpu().numpy()
        e = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        pos = ref > 0
        worst = float(np.max(np.abs(got[pos] - ref[pos]) / ref[pos]))
        return {"rel_fro": e, "max_unit_rel": worst, "gate": g, "sampled": int(k),
                "of": int(c.npairs), "pass": bool(e <= g and worst <= g)}
    sd = sr = worst = 0.0
    for j0 in range(0, k, 16384):
        gg = Y[j0:min(k, j0 + 16384)].double().cpu().numpy()
        rr = ref[j0:j0 + gg.shape[0]]
        dcol = np.sqrt(((gg - rr) ** 2).sum(1))
        rcol = np.sqrt((rr * rr).sum(1))
        sd += float((dcol ** 2).sum())
        sr += float((rcol ** 2).sum())
        worst = max(worst, float(np.max(dcol / np.where(rcol > 0, rcol, 1.0))))
    e = math.sqrt(sd / sr)
    return {"rel_fro": e, "max_unit_rel": worst, "gate": g, "sampled": int(k), "of": int(c.N),
            "finite": bool(torch.isfinite(Y).all().item()),
            "pass": bool(e <= g and worst <= g and torch.isfinite(Y).all().item())}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    c = workload_case(args.workload)
    op = 0 if args.op == "N" else 1
    import oracle
    steps, warm = args.steps, args.warmup
    budget = 150.0 / max(1, steps + warm)          # whole run within a few minutes
    _, _, units = alg_cost(c)
    byts, _, _ = alg_cost(c)
    # calibrate the sample size for ~budget seconds per step
    _, ups, _, _, threads, _, _ = time_oracle(c, op, target_s=min(2.0, budget))
    k = int(max(1, min(units, ups * budget)))
    sub = workload_case(args.workload, N_override=None)
    per_unit_bytes = byts / units
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        if c.call == "knn":
            oracle.knn(sub.U, sub.d, sub.X, sub.lam[:k], sub.k)
        elif c.call == "shf":
            oracle.shf_cost(sub.X, sub.d, sub.U[:k])
        elif c.call == "congruence":
            oracle.congruence(op, sub.U, sub.X[:k * sub.n].reshape(k, sub.n, sub.n))
        elif c.call == "mahalanobis":
            oracle.mahalanobis(sub.U, sub.d, sub.X, sub.ia[:k], sub.ib[:k])
        elif c.call == "sym":
            oracle.sym_apply(sub.U, sub.lam, sub.X[:k])
        else:
            oracle.apply(op, sub.U, sub.X[:k])
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    tot = sum(times)
    value = per_unit_bytes * k * steps / tot / 1e9
    what = {"mahalanobis": "pairs", "knn": "queries", "congruence": "matrices",
            "shf": "candidates"}.get(c.call, "columns")
    sample = f"{k} of {units} {what} of {c.name} per step (fp64 oracle, {threads} threads)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": ws, "steps": steps, "warmup": warm, "ms_per_step": 1e3 * tot / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen/inputs.py, seeded)",
        "config": config_of(c, args),
        "vectors_per_s": k * steps / tot,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(c, args):
    d = {"workload": f"{c.name}: {c.call} {'Q' if args.op == 'N' else 'Q^T'}·X"
         if c.call == "apply" else f"{c.name}: {c.call}",
         "n": c.n, "h": c.h, "N": c.N, "dtype": c.dtype,
         "l2": "inputs larger than L2 (no flush)" if c.N * c.n * (4 if c.dtype == "f32" else 8)
         > 256 << 20 else "L2-resident inputs (warm L2, labelled)"}
    if c.call == "mahalanobis":
        d["npairs"] = c.npairs
    if c.call == "congruence":
        d.update({"count": c.count, "op": args.op, "form": "op(Q) M op(Q)^T (eq:ak / eq:bk, P:297-304)"})
    if c.call == "shf":
        d.update({"K": c.K, "form": "C(u) and grad C(u) of one reflector (eq:theRk, eq:gradient, "
                                    "P:316-377), A, B symmetric"})
    if c.call == "knn":
        d.update({"M_ref": c.N, "M_query": int(c.lam.shape[0]), "k": c.k,
                  "stand_in_for": "Table I MNIST after PCA (P:670), iid N(0,1)"})
    if c.call == "apply":
        d["op"] = args.op
    return d


def run_hh(args):
    import torch
    import torch.distributed as dist

    import paper_1811_07624_b200 as hh

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    c = workload_case(args.workload)
    op = hh.HH_OP_N if args.op == "N" else hh.HH_OP_T
    byts, flops, units = alg_cost(c)

    U = torch.from_numpy(c.U).to(dev)
    X = torch.from_numpy(c.X).to(dev)
    Y = torch.empty_like(X)
    stream = torch.cuda.current_stream(dev)
    extra = {}
    if c.call == "knn":
        d = torch.from_numpy(c.d).to(dev)
        Pq = torch.from_numpy(c.lam).to(dev)
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_KNN, c.n, c.h, c.N, Pq.shape[0], X.dtype)
        wsp = torch.empty(wsb, dtype=torch.uint8, device=dev)
        knn_out = {}
        dist_out = None

        def step():
            knn_out["r"] = hh.hh_knn(U, d, X, Pq, c.k, workspace=wsp, stream=stream)
        launches = 6
    elif c.call == "sym":
        lam = torch.from_numpy(c.lam).to(dev)
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_SYM, c.n, c.h, c.N, 0, X.dtype)
        wsp = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        step = lambda: hh.hh_sym_apply(U, lam, X, Y, workspace=wsp, stream=stream)  # noqa: E731
        launches = 1
    elif c.call == "mahalanobis":
        d = torch.from_numpy(c.d).to(dev)
        ia = torch.from_numpy(c.ia).to(dev)
        ib = torch.from_numpy(c.ib).to(dev)
        dist_out = torch.empty(c.npairs, dtype=X.dtype, device=dev)
        knn_out = {}
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_MAHALANOBIS, c.n, c.h, c.N, c.npairs, X.dtype)
        wsp = torch.empty(wsb, dtype=torch.uint8, device=dev)
        step = lambda: hh.hh_mahalanobis(U, d, X, ia, ib, dist_out, workspace=wsp,  # noqa: E731
                                         stream=stream)
        launches = 2
    elif c.call == "shf":
        A = X
        B = torch.from_numpy(c.d).to(dev)
        cost = torch.empty(c.K, dtype=X.dtype, device=dev)
        gout = torch.empty_like(U)
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_SHF, c.n, 0, c.K, 0, X.dtype)
        wsp = torch.empty(wsb, dtype=torch.uint8, device=dev)
        knn_out = {"r": (cost, gout)}
        dist_out = None
        step = lambda: hh.hh_shf_cost(A, B, U, cost=cost, grad_out=gout, workspace=wsp,  # noqa: E731
                                      stream=stream)
        launches = 4
    elif c.call == "congruence":
        M = X.view(c.count, c.n, c.n)
        Mo = Y.view(c.count, c.n, c.n)
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_CONGRUENCE, c.n, c.h, c.count, 0, X.dtype)
        wsp = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        step = lambda: hh.hh_congruence(op, U, M, Mo, workspace=wsp, stream=stream)  # noqa: E731
        launches = 4
    elif c.call == "apply_qr":
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, c.n, c.h, c.N, 0, X.dtype)
        wsp = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        step = lambda: hh.hh_apply_qr(op, U, X, Y, workspace=wsp, stream=stream)  # noqa: E731
        launches = 1
        # the same U through the structure-blind path, for the 4(n-k+1) vs 4n comparison
        for _ in range(2):
            hh.hh_apply(op, U, X, Y, workspace=wsp, stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            hh.hh_apply(op, U, X, Y, workspace=wsp, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        extra["full_apply_ms"] = e0.elapsed_time(e1) / 3
    else:
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY, c.n, c.h, c.N, 0, X.dtype)
        wsp = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        step = lambda: hh.hh_apply(op, U, X, Y, workspace=wsp, stream=stream)  # noqa: E731
        launches = 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    info = hh.last_launch_info()
    wy_path = str(info.get("variant", "")).startswith("wy_")
    launches = int(info.get("launches") or launches)   # the library's own count per step

    sampler = ClockSampler(dev.index if dev.index is not None else 0).start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    t_wall1 = time.time()
    ms = ev0.elapsed_time(ev1)
    # per-step distribution (median, minimum) from a separate short run with an event
    # between steps, outside the timed region (events between kernels cost ~1 % here)
    ksplit = min(args.steps, 20)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(ksplit + 1)]
    evs[0].record(stream)
    for i in range(ksplit):
        step()
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    per_step = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(ksplit))
    if ws > 1:
        dist.barrier()
    # keep the GPU busy for >= 1 s of clock samples if the timed region was short
    t_obs0 = t_wall0
    if t_wall1 - t_wall0 < 1.0 and not args.ncu:
        t_obs0 = time.time()
        while time.time() - t_obs0 < 1.0:
            for _ in range(50):
                step()
            torch.cuda.synchronize(dev)
    t_obs1 = time.time()
    time.sleep(0.1)
    sampler.stop()
    clocks = sampler.summary(t_obs0, t_obs1)

    from paper_1811_07624_b200 import dist as hd
    ms_max = hd.max_over_ranks(ms, device=dev)          # max over ranks
    ms_step = ms_max / args.steps
    value = ws * byts / (ms_step * 1e-3) / 1e9

    # e2e through the public API with host buffers (hh_apply_host): H2D + compute + D2H
    e2e = None
    if c.call == "apply" and not args.no_e2e:
        Xh = torch.from_numpy(c.X).pin_memory()
        Yh = torch.empty_like(Xh).pin_memory()
        Uh = torch.from_numpy(c.U)
        wsb = hh.hh_workspace_bytes(hh.HH_CALL_APPLY_HOST, c.n, c.h, c.N, 0, X.dtype)
        wsp = torch.empty(wsb, dtype=torch.uint8, device=dev)
        hh.hh_apply_host(op, Uh, Xh, Yh, workspace=wsp)
        ke = max(1, min(args.steps, args.e2e_steps))
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(ke):
            hh.hh_apply_host(op, Uh, Xh, Yh, workspace=wsp)
        torch.cuda.synchronize(dev)
        se = hd.max_over_ranks(time.perf_counter() - t0, device=dev) / ke
        e2e = {"value": ws * byts / se / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(Xh.numel() * Xh.element_size() + Uh.numel() * 4),
               "d2h_bytes_per_step": int(Yh.numel() * Yh.element_size()),
               "ms_per_step": 1e3 * se, "steps": ke,
               "path": "hh_apply_host (pinned host X/Y, 3-slot H2D/compute/D2H ring)"}
        # the host path runs the same kernel per column: results must be bit-identical
        sel = torch.linspace(0, c.N - 1, 64).long()
        e2e["matches_device_path"] = bool(torch.equal(Yh[sel].to(dev), Y[sel.to(dev)]))

    out = None
    if rank == 0:
        hbm, hbm_src, _ = peaks()
        achieved = byts / (ms_step * 1e-3) / 1e9
        # ncu-measured DRAM bytes of one step of this workload (tools/traffic.py, committed
        # under profiles/r2/): bench.py cannot run ncu itself
        traffic, traffic_src = None, None
        tf = os.path.join(ROOT, "profiles", "r2", "traffic_r2.json")
        if os.path.exists(tf):
            try:
                tr = json.load(open(tf)).get(args.workload.upper().replace("H", "h") if
                                             args.workload.upper().startswith("C5") else
                                             args.workload.upper())
                if tr:
                    traffic = tr["dram_bytes_per_step"]
                    traffic_src = {"per_step_bytes": tr["dram_bytes_per_step"],
                                   "dominant_kernel": tr["dominant_kernel"],
                                   "dominant_bytes_per_launch": tr["dominant_bytes_per_launch"],
                                   "source": "profiles/r2/traffic_r2.json (" + tr["source"] + ")"}
            except (ValueError, OSError, KeyError):
                traffic = None
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_source": hbm_src,
                "frac_of_8TBps": achieved / 8000.0,
                "kernel": info.get("variant"), "launch": info, "traffic_detail": traffic_src}
        # the algorithmic roofline is max(bytes / HBM peak, flops / pipe peak);
        # the SIMT FP32 (FP64) pipe peak is #SM x 128 (64) FMA lanes x 2 x the maximum SM
        # clock (R13).  When the flops floor is the larger one (C4's transform-once
        # reading: 4.43 GFLOP vs 159 MB), the line reports the ALU bound.
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        fmax = float(peaks()[2].get("sm_max_mhz", 1965.0)) * 1e6 if peaks()[2] else 1.965e9
        alu_peak = sms * (128 if c.dtype == "f32" else 64) * 2 * fmax / 1e12   # TFLOP/s
        t_hbm_s, t_alu_s = byts / (hbm * 1e9), flops / (alu_peak * 1e12)
        if t_alu_s > t_hbm_s and not wy_path and c.call != "knn":
            roof = {"bound": "alu", "achieved": flops / (ms_step * 1e-3) / 1e12,
                    "peak": alu_peak, "unit": "TFLOP/s",
                    "frac": t_alu_s / (ms_step * 1e-3), "traffic": traffic,
                    "peak_source": f"derived: {sms} SMs x {128 if c.dtype == 'f32' else 64} "
                                   f"FMA lanes x 2 x {fmax / 1e6:.0f} MHz (DESIGN.md R13)",
                    "hbm_frac": achieved / hbm, "hbm_floor_ms": 1e3 * t_hbm_s,
                    "alu_floor_ms": 1e3 * t_alu_s,
                    "kernel": info.get("variant"), "launch": info}
        if str(info.get("variant", "")).startswith("knn_"):
            pk = peaks()[2]
            tpeak = float(pk.get("bf16_tflops", 1590.0)) if pk else 1590.0
            Mq = c.lam.shape[0]
            exe = 3 * 2 * ((c.n + 31) // 32 * 32) * c.N * Mq
            # the distances run as bf16x3 products (three bf16 products per fp32-accurate one):
            # the peak of that arithmetic is the bf16 peak / 3 (R18, as for K5)
            roof = {"bound": "tensor", "achieved": flops / (ms_step * 1e-3) / 1e12,
                    "peak": tpeak / 3, "unit": "TFLOP/s",
                    "frac": flops / (ms_step * 1e-3) / 1e12 / (tpeak / 3), "traffic": traffic,
                    "frac_of_bf16_burst_algorithmic": flops / (ms_step * 1e-3) / 1e12 / tpeak,
                    "peak_source": "measured bf16 burst (MEASURED_PEAKS.json bf16_tflops) / 3: the "
                                   "fp32-accurate bf16x3 rate (DESIGN.md R18)",
                    "executed_tflops": exe / (ms_step * 1e-3) / 1e12,
                    "executed_frac": exe / (ms_step * 1e-3) / 1e12 / tpeak,
                    "pairs_per_s": c.N * Mq / (ms_step * 1e-3),
                    "kernel": info.get("variant"), "launch": info,
                    "scope": "whole step (transform, pack, distance GEMM + top-k, merge)"}
        elif wy_path:
            # compact-WY block program: algorithmic 4hnN / (8h+1)nN flops and
            # 2 N n s bytes; executed: 3 bf16x3 products per GEMM and 3 passes of X per
            # block (project reads X, update reads X and writes Y).  The binding resource
            # is the larger executed fraction; `frac` is the algorithmic one.
            pk = peaks()[2]
            tpeak = float(pk.get("bf16_tflops", 1590.0)) if pk else 1590.0
            s_ = 4 if c.dtype == "f32" else 8
            npass = int(info["nchunks"])
            if c.call == "sym":
                m = (npass + 1) // 2
                b = ((c.h + m - 1) // m + 31) // 32 * 32
                kw = [b] * (npass - 1) + [2 * b]
            else:
                b = ((c.h + npass - 1) // npass + 31) // 32 * 32
                kw = [b] * npass
            exe = sum(3 * 2 * 2 * k_ * c.n * c.N for k_ in kw)
            exe_bytes = sum(3 * c.N * c.n * s_ + 2 * c.N * k_ * 4 for k_ in kw)
            if c.call == "apply_qr":
                # NEXT-f2: block k's project starts at K row (k b) rounded down to 32 and its
                # update at row chunk (k b) rounded down to 128 (op N); rows above are skipped
                exe, exe_bytes = 0, 0
                for kb in range(npass):
                    p0, u0 = (kb * b // 32) * 32, (kb * b // 128) * 128
                    exe += 3 * 2 * b * ((c.n - p0) + (c.n - u0)) * c.N
                    exe_bytes += ((c.n - p0) + 2 * (c.n - u0)) * c.N * s_ + 2 * c.N * b * 4
            t_s = ms_step * 1e-3
            ef_t, ef_h = exe / t_s / 1e12 / tpeak, exe_bytes / t_s / 1e9 / hbm
            # the binding floor of the METHOD on this hardware: its HBM bytes at the copy
            # rate vs its flops as bf16x3 products (3 per fp32-accurate product) at the
            # bf16 rate; `floor_frac` = that floor / measured time
            # tensor peak: the burst cuBLAS bf16 rate for a kernel timed alone, the sustained
            # (power-capped) one for a long run -- B200_PROFILING.md; this step is timed over
            # many back-to-back launches, and the run is long when the timed region exceeds
            # 20 ms or the SM clock sat below 90 % of its maximum (sw_power_cap)
            tsus = float(pk.get("bf16_tflops_sustained", tpeak)) if pk else tpeak
            long_run = ms_max >= 20.0 or (clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                                          clocks["sm_mhz"] < 0.9 * clocks["sm_max_mhz"])
            tpk = tsus if long_run else tpeak
            # the fp32-accurate contraction runs as bf16x3 (three bf16 products per fp32 product,
            # DESIGN.md R18): its peak on this pipe is the bf16 peak / 3
            t_hbm, t_ten = byts / (hbm * 1e9), 3 * flops / (tpk * 1e12)
            if t_ten >= t_hbm:
                roof = {"bound": "tensor", "achieved": flops / t_s / 1e12, "peak": tpk / 3,
                        "unit": "TFLOP/s", "frac": flops / t_s / 1e12 / (tpk / 3),
                        "peak_source": ("measured bf16 sustained" if long_run else "measured bf16 burst")
                        + " (MEASURED_PEAKS.json) / 3: the fp32-accurate bf16x3 rate (DESIGN.md R18)",
                        "frac_of_bf16_burst_algorithmic": flops / t_s / 1e12 / tpeak,
                        "bf16_peak_used": tpk}
            else:
                roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                        "frac": achieved / hbm, "peak_source": hbm_src}
            roof.update({"floor_ms": 1e3 * max(t_hbm, t_ten),
                         "floor_frac": max(t_hbm, t_ten) / t_s,
                         "traffic": traffic, "executed_tflops": exe / t_s / 1e12,
                         "executed_tensor_frac": ef_t, "executed_gbs": exe_bytes / t_s / 1e9,
                         "executed_hbm_frac": ef_h, "kernel": info.get("variant"),
                         "launch": info, "passes": npass,
                         "scope": "whole step (K4 prep + all K5 launches)"})
        cpu = None
        parity = None
        if not (args.no_cpu_baseline and args.no_parity):
            # the oracle as it stands on the host cores (cpu_baseline, rank 0 at N = 1), and
            # the parity of this run's output against that same oracle output
            v, ups, secs, sample, thr, k_or, ref = time_oracle(
                c, op, target_s=args.cpu_seconds if not args.no_cpu_baseline else 2.0)
            if not args.no_cpu_baseline and ws == 1:
                cpu = {"value": v, "unit": "GB/s", "cores": thr, "kind": "oracle",
                       "sample": sample, "seconds": secs, "vectors_per_s": ups, "cpu": cpu_model()}
            if not args.no_parity:
                parity = parity_of(c, k_or, ref, Y, dist_out if c.call == "mahalanobis" else None,
                                   knn_out.get("r") if c.call in ("knn", "shf") else None, dev)
        if not args.ncu and roof is not None:
            roof["same_run_copy_gbs"] = same_run_copy_gbs(dev)
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": c.dtype, "data": "synthetic (gen/inputs.py, seeded; BASELINE.json recipe)",
            "config": config_of(c, args),
            "vectors_per_s": ws * units / (ms_step * 1e-3),
            "gflops": ws * flops / (ms_step * 1e-3) / 1e9,
            "ms_per_step_median": per_step[len(per_step) // 2], "ms_per_step_min": per_step[0],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clocks, "parity": parity, **extra,
            "gpu": torch.cuda.get_device_name(dev),
            "inputs_sha256": input_digest(c),
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="hh", choices=["hh", "reference"])
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--op", default="N", choices=["N", "T"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling run: no parity / cpu baseline / e2e / clock-hold loop")
    args = ap.parse_args()
    if args.ncu:
        args.no_parity = args.no_cpu_baseline = args.no_e2e = True
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_hh(args)


if __name__ == "__main__":
    sys.exit(main())
