#!/usr/bin/env python
"""Benchmark: parameter queries solved per second to relative residual 1e-10.

Workload (BASELINE.json configs[1], "c2"): 2D 5-point thermal-block diffusion on
a 511x511 grid (N = 261,121), 3x3 subdomains (P = Q = 9), mu log-uniform in
[0.1, 10], f = 1, fp64, greedy basis n = 40 from 1024 seeded training mu
(built on the GPU by rbs_build_greedy, untimed), 256 queries per GPU batched
B = 32, RBCG to tol 1e-10 with symmetric red-black GS.

A step = one rbs_solve_batch of B queries to convergence (every row of the
hot path: reduced assembly + Cholesky, residual, projection, reduced solve,
prolongation, smoothing, CG recurrences, stop test).  Batches are independent:
--streams S (default 2) runs S of them at a time on S CUDA streams, each with
its own context, so one batch's latency-bound passes overlap another's.  N > 1: one process per
GPU (torchrun), queries sharded (rank r solves its own 256), no collective on
the data path: weak scaling.  Timing: CUDA events on the solve stream after a
barrier + synchronize, max over ranks.  The working set (W 84 MB + four 67 MB
state vectors) exceeds the 126 MB L2, so no explicit flush is needed.

--impl reference: the CPU oracle (oracle/, plain C fp64) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, query_set, train_set  # noqa: E402

METRIC = "parameter queries solved/sec to rel. residual 1e-10 (c2, RBCG, 1 GPU)"
UNIT = "queries/s"
HBM_FALLBACK_GBS = 6650.0     # /opt/skills/guides/B200_PROFILING.md fallback
# FP64 tensor (DMMA m8n8k4) peak measured on this pool's B200 with tools/fp64_peak.cu
# (148 SMs x 1 DMMA / 4 cycles at 1965 MHz; DFMA 36.7 TF/s); not in MEASURED_PEAKS.json
FP64_TENSOR_MEASURED_TFS = 37.2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-iters", type=int, default=30)
    p.add_argument("--streams", type=int, default=2, help="concurrent batch streams (1 = one batch at a time)")
    p.add_argument("--method", default="rbcg", choices=["rbcg", "rbi"],
                   help="RBCG (PAPER.md:260-279, default) or the stand-alone RB iteration (PAPER.md:155-169)")
    return p.parse_args()


def workload_desc(c, method="rbcg"):
    return (f"{c.name}: {c.dim}D {c.m}^{c.dim} (N={c.N}), {'x'.join(map(str, c.blocks))} blocks, "
            f"mu logU[{c.lo},{c.hi}]^{c.P}, f=1, greedy n={c.n} from {c.n_train} train mu, "
            f"{c.n_queries} queries/GPU, B={c.B}, {method.upper()} sym-RBGS nu=1, tol 1e-10")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU)
def _oracle_worker(args):
    path, idx, mu = args
    import oracle
    from synth import CONFIGS as CF
    c = CF["c2"]
    d = np.load(path)
    g = oracle.Grid(c.dim, c.m, c.blocks)
    t = time.perf_counter()
    out = g.rbcg(np.asfortranarray(d["W"]), d["ANq"], d["fn"], mu)
    return idx, time.perf_counter() - t, out["its"], out["status"]


def oracle_basis_file(c):
    """Oracle-built basis at full size (test input recipe): coarse
    greedy on 63^2, multilinear prolongation to the fine grid, oracle MGS and
    offline blocks.  Cached per process in /tmp (rebuilt if absent)."""
    import oracle
    path = os.path.join(tempfile.gettempdir(), f"rbs_oracle_basis_{c.name}_{c.n}.npz")
    if not os.path.exists(path):
        W, ANq, fn = oracle.interpolated_basis(c.dim, c.m, c.blocks, train_set(c), c.n, 63)
        np.savez(path, W=W, ANq=ANq, fn=fn)
    return path


def cpu_oracle_run(c, nq, offset=0):
    """solve nq queries with the oracle, one process per core; returns q/s, details."""
    import multiprocessing as mp
    path = oracle_basis_file(c)
    mus = query_set(c, offset + nq)[offset:]
    cores = min(nq, os.cpu_count() or 1)
    t = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, [(path, i, mus[i]) for i in range(nq)])
    wall = time.perf_counter() - t
    its = [r[2] for r in res]
    return nq / wall, cores, wall, its


def run_reference(a):
    c = CONFIGS[a.config]
    ncpu = os.cpu_count() or 1
    nq = min(ncpu, 8)
    oracle_basis_file(c)
    for w in range(a.warmup):
        cpu_oracle_run(c, nq, offset=w * nq)
    t0 = time.perf_counter()
    tot_q, its_all, cores = 0, [], 1
    for s in range(a.steps):
        _, cores, _, its = cpu_oracle_run(c, nq, offset=(a.warmup + s) * nq)
        tot_q += nq
        its_all += its
    el = time.perf_counter() - t0
    v = tot_q / el
    line = {"impl": "reference", "metric": METRIC.replace("(c2,", f"({c.name},"), "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * el / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(c), "basis": "oracle coarse-greedy (63^2) "
                       "interpolated, n=40", "oracle_its": [int(min(its_all)), int(max(its_all))]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{nq} queries per step, one oracle process per core, "
                                       f"RBCG to 1e-10 (host has {ncpu} cores)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
# Case 1 with RB dimension 1 and 5, Case 2 with 2 and 10 (AMB-17: the
# text's 10 over the caption's 20), 100 random parameters per case (96 = 6 batches of 16 here)
CASE_M, CASE_B, CASE_TRAIN, CASE_QUERIES = 127, 16, 64, 96
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r1_final_traffic.json")


def ncu_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    ncu --set full capture of the same kernel and configuration (profiles/), else None."""
    try:
        d = json.load(open(TRAFFIC_FILE))
        if d.get("config") == config and kernel in d:
            return d[kernel]["dram_bytes_per_launch"], f"{os.path.relpath(TRAFFIC_FILE, ROOT)}: {d[kernel]['kernel']}"
    except (OSError, ValueError, KeyError):
        pass
    return None, None
CASE_N = {1: 5, 2: 10}


def run_case(a, case):
    """NEXT(4) measurement: the paper's Case 1 / Case 2 (Table 1) as a
    7-point FD face operator on 127^3 interior nodes (h = 1/128, N = 2,048,383; AMB-23):
    GPU greedy basis from 64 seeded training mu with the affine right-hand side
    (untimed; n = 5 for Case 1, 10 for Case 2), 96 queries in batches of
    B = 16, RBCG to 1e-10.  A step = one batch:
    device assembly of f(mu) (rbs_affine_rhs) + rbs_solve_batch.  1 GPU only."""
    import torch
    import paper_1804_06363_b200 as rbs
    from synth import cases
    torch.cuda.set_device(0)
    P = cases.case_problem(case, CASE_M)
    s = rbs.Solver(3, CASE_M, faces=P["faces"])
    terms = torch.as_tensor(P["terms"]).to(s.device)
    t0 = time.perf_counter()
    tr = cases.case_params(case, CASE_TRAIN, 1000 + case)
    gr = s.build_greedy(np.stack([P["theta"](mu) for mu in tr]), CASE_N[case],
                        phi_train=np.stack([P["phi"](mu) for mu in tr]), terms=terms)
    torch.cuda.synchronize()
    offline_s = time.perf_counter() - t0
    q = cases.case_params(case, CASE_QUERIES, 2000 + case)
    th = np.stack([P["theta"](mu) for mu in q])
    phi = np.stack([P["phi"](mu) for mu in q])
    nb = CASE_QUERIES // CASE_B
    N = s.N
    X = torch.empty((CASE_B, N), dtype=torch.float64, device=s.device)
    stream = torch.cuda.current_stream()

    def step(k, **kw):
        b = k % nb
        sl = slice(b * CASE_B, (b + 1) * CASE_B)
        rhs = s.affine_rhs(phi[sl], terms)
        return s.solve_batch(th[sl], rhs=rhs, X=X, want_a_n=False, **kw)

    for w in range(max(a.warmup, 1)):
        step(w)
    clocks = Clocks(0)
    clocks.start()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches, its = 0, []
    for k in range(a.steps):
        out = step(k)
        launches += out["launches"] + 1
        its += [int(i) for i in out["its"]]
        assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    prof = step(0, profile=1, tol=0.0, max_iter=a.profile_iters)["profile"]
    hbm, hbm_src = peaks()
    n, B = gr["n"], CASE_B
    face_b = 8 * 2 * 3 * N          # Q = 2 face arrays, 3 new faces per node, read once per pass
    alg = {"k_cgp": 24 * B * N + face_b, "k_proj": 40 * B * N + 8 * N * n + face_b,
           "k_gs": 16 * B * N + face_b, "k_prolong": 8 * B * N + 8 * N * n}
    tot_ms = sum(v[0] for v in prof.values())
    kernels = {k: {"avg_us": 1e3 * v[0] / max(v[1], 1), "launches": v[1],
                   "share": v[0] / tot_ms if tot_ms else None} for k, v in prof.items() if v[1]}
    for k, kb in alg.items():
        if k in kernels:
            d = kernels[k]["avg_us"] * 1e-6
            kernels[k].update(alg_bytes=kb, GBps=kb / d / 1e9, hbm_frac=kb / d / 1e9 / hbm)
    top = max((k for k in alg if k in kernels), key=lambda k: kernels[k]["share"])
    kt = kernels[top]
    line = {"metric": f"parameter queries solved/sec to rel. residual 1e-10 (Case {case}, RBCG, 1 GPU)",
            "value": a.steps * B / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"case{case}: PAPER.md Table 1 Case {case}, 3D 7-point FD face operator "
                                   f"{CASE_M}^3 (N={N}), Q=2, R={P['terms'].shape[0]}, GPU greedy n={n} "
                                   f"from {CASE_TRAIN} train mu, {CASE_QUERIES} queries, B={B}, RBCG "
                                   "sym-RBGS nu=1 (flat kernels), tol 1e-10",
                       "B": B, "n": n, "its_min_med_max": [min(its), int(np.median(its)), max(its)],
                       "offline_greedy_s": round(offline_s, 2),
                       "l2": "inputs larger than L2 (4 x 262 MB state)"},
            "clocks": clk, "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": top, "achieved": kt["GBps"], "peak": hbm,
                         "unit": "GB/s", "frac": kt["GBps"] / hbm, "traffic": None,
                         "peak_source": hbm_src, "alg_bytes_per_launch": kt["alg_bytes"],
                         "avg_launch_us": kt["avg_us"], "share_of_iteration": kt["share"]},
            "kernels": kernels}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.config in ("case1", "case2"):
        if a.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "case workloads: GPU measurement only"}))
        elif int(os.environ.get("RANK", "0")) == 0:
            run_case(a, int(a.config[-1]))
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        if rank == 0:
            run_reference(a)
        return
    import torch
    import torch.distributed as dist
    import paper_1804_06363_b200 as rbs
    from paper_1804_06363_b200.dist import broadcast_basis, gather_counts

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[a.config]
    s = rbs.Solver(c.dim, c.m, c.blocks, device=local)
    stream = torch.cuda.current_stream()

    # ---- offline: greedy basis on the GPU (rank 0), broadcast over NCCL -----
    t0 = time.perf_counter()
    if rank == 0:
        gr = s.build_greedy(train_set(c), c.n, load=False)
        W = gr["W"].contiguous()
        ANq = torch.tensor(gr["ANq"], device=s.device)
        fn = torch.tensor(gr["fn"], device=s.device)
        snap = [int(x) for x in gr["snap_iters"]]
    else:
        W = torch.empty((c.N, c.n), dtype=torch.float64, device=s.device)
        ANq = torch.empty((c.P, c.n, c.n), dtype=torch.float64, device=s.device)
        fn = torch.empty((c.n,), dtype=torch.float64, device=s.device)
        snap = []
    if world > 1:
        broadcast_basis(W, ANq, fn, src=0)        # NCCL over NVLink, once, off the hot path
    s.load_basis(W, ANq.cpu().numpy(), fn.cpu().numpy())
    torch.cuda.synchronize()
    offline_s = time.perf_counter() - t0

    # ---- queries: rank r owns its own n_queries (weak scaling) ---------------
    nq = c.n_queries
    mus_all = query_set(c, nq * world)
    mus = mus_all[rank * nq:(rank + 1) * nq]
    nb = nq // c.B
    # S concurrent batch streams (DESIGN.md §7 "Concurrent batches"): batch k runs on stream
    # k mod S, each stream with its own context (same basis) and buffers; the batches are
    # independent, so this is a scheduling choice that lets one batch's latency-bound
    # passes overlap another's
    S = max(1, a.streams)
    ss = [s] + [rbs.Solver(c.dim, c.m, c.blocks, device=local).load_basis(W, ANq.cpu().numpy(), fn.cpu().numpy())
                for _ in range(S - 1)]
    sts = [torch.cuda.Stream(device=s.device) for _ in range(S)]
    Xs = [torch.empty((c.B, c.N), dtype=torch.float64, device=s.device) for _ in range(S)]

    mkw = (dict(method=rbs.RBS_RBI, max_iter=500000) if a.method == "rbi" else dict(method=rbs.RBS_RBCG))

    def step(t, k, **kw):
        b = k % nb
        return ss[t].solve_batch(mus[b * c.B:(b + 1) * c.B], X=Xs[t], stream=sts[t], want_a_n=False,
                                 **{**mkw, **kw})

    def run(nsteps, fn, nvtx=None):
        outs = [[] for _ in range(S)]

        def worker(t):
            torch.cuda.set_device(local)
            if nvtx:
                torch.cuda.nvtx.range_push(nvtx)
            for k in range(t, nsteps, S):
                outs[t].append(fn(t, k))
            if nvtx:
                torch.cuda.nvtx.range_pop()

        th = [threading.Thread(target=worker, args=(t,)) for t in range(S)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        return [o for ol in outs for o in ol]

    run(max(a.warmup, S), step)
    # ---- timed region (device events, max over ranks) ------------------------
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include "timed/" profiles only this
    ev0.record(stream)
    outs = run(a.steps, step, nvtx="timed")     # every worker thread marks its launches too
    torch.cuda.synchronize()
    ev1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches, its = 0, []
    for out in outs:
        launches += out["launches"]
        its += [int(i) for i in out["its"]]
        assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    if world > 1:
        t = torch.tensor([ms], device=s.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    value = a.steps * c.B * world / (ms / 1e3)
    if world > 1:   # per-query iteration counts of every rank, for the its statistics
        t_its = torch.tensor(its, dtype=torch.int32, device=s.device)
        all_its, _ = gather_counts(t_its, torch.zeros_like(t_its))
        its = [int(v) for v in all_its.cpu()]

    # ---- e2e: public API with host buffers (pinned X, host mu) --------------
    Xh = [torch.empty((c.B, c.N), dtype=torch.float64, pin_memory=True) for _ in range(S)]

    def step_host(t, k):
        b = k % nb
        return ss[t].solve_batch(mus[b * c.B:(b + 1) * c.B], X=Xh[t], x_location=rbs.RBS_MEM_HOST,
                                 stream=sts[t], want_a_n=True, **mkw)

    run(S, step_host)      # warm-up: host-output workspace and its iteration graph per context
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    run(a.steps, step_host)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t
    if world > 1:
        tt = torch.tensor([e2e_s], device=s.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = {"value": a.steps * c.B * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": c.B * c.P * 8,
           "d2h_bytes_per_step": c.B * c.N * 8 + c.B * (4 + 4 + 8 + 8 + 8 * c.n)}

    # ---- per-kernel device times (eager, events on the launching stream) -----
    prof = step(0, 0, profile=1, tol=0.0, max_iter=a.profile_iters)["profile"]
    hbm, hbm_src = peaks()
    # queries per pass: 2D batches above 32 run as 32-query sub-batches
    Bq, N, n = (min(c.B, 32) if c.dim == 2 else c.B), c.N, c.n
    # algorithmic bytes per launch (each vector once, W once per batch)
    alg = {"k_cgp": 24 * Bq * N,                    # y, p_old read; p_new written
           "k_proj": 40 * Bq * N + 8 * N * n,       # p, x, r read; x, r written; W
           "k_gs": 16 * Bq * N + 8 * N * n}         # 2D fused smoother: r read, y written; W
    if a.method == "rbi":   # RBI: K3' x_new = S(x_old + W e) (x_old, W read; x written), resid f - A x + W^T (x, W)
        alg = {"k_gs": 16 * Bq * N + 8 * N * n, "k_proj": 8 * Bq * N + 8 * N * n}
    elif c.dim == 3:   # separate prolongation pass; k_gs is one red-black half-sweep per launch
        alg["k_prolong"] = 8 * Bq * N + 8 * N * n   # W read, y0 written
        alg["k_gs"] = 16 * Bq * N                   # y read, r and y of one colour
    flops = {"k_proj": 2.0 * N * n * Bq, "k_gs": 2.0 * N * n * Bq}   # W^T r / W e on DMMA
    tot_ms = sum(v[0] for v in prof.values())
    kernels = {k: {"avg_us": 1e3 * v[0] / max(v[1], 1), "launches": v[1],
                   "share": v[0] / tot_ms if tot_ms else None} for k, v in prof.items() if v[1]}
    for k, kb in alg.items():
        if k in kernels:
            d = kernels[k]["avg_us"] * 1e-6
            kernels[k]["alg_bytes"] = kb
            kernels[k]["GBps"] = kb / d / 1e9
            kernels[k]["hbm_frac"] = kb / d / 1e9 / hbm
            if k in flops:
                kernels[k]["fp64_tensor_TFs"] = flops[k] / d / 1e12
    top = max((k for k in alg if k in kernels), key=lambda k: kernels[k]["share"])
    kt = kernels[top]
    iter_us = 1e3 * tot_ms / max(prof["k_proj"][1], 1)     # per pass-iteration of Bq queries
    iter_bytes = ((24 * Bq + 16 * n) if a.method == "rbi" else (80 * Bq + 16 * n)) * N   # minimum per batch-iteration
    traffic, traffic_src = ncu_traffic(a.config, top)
    roof = {"bound": "hbm", "kernel": top, "achieved": kt["GBps"], "peak": hbm, "unit": "GB/s",
            "frac": kt["GBps"] / hbm, "traffic": traffic, "traffic_source": traffic_src, "peak_source": hbm_src,
            "alg_bytes_per_launch": kt["alg_bytes"], "avg_launch_us": kt["avg_us"],
            "share_of_iteration": kt["share"],
            "iteration": {"us": iter_us, "alg_bytes": iter_bytes,
                          "GBps": iter_bytes / (iter_us * 1e-6) / 1e9,
                          "frac": iter_bytes / (iter_us * 1e-6) / 1e9 / hbm},
            "fp64_tensor_peak_tflops": FP64_TENSOR_MEASURED_TFS,
            "fp64_tensor_peak_source": "measured, tools/fp64_peak.cu (DMMA m8n8k4, all SMs)"}

    wbytes, sbytes = c.N * (((c.n + 7) // 8) * 8 + 4) * 8, 4 * c.N * c.B * 8
    l2 = (f"inputs larger than L2 (W {wbytes / 1e6:.0f} MB + 4 x {sbytes / 4e6:.0f} MB state > 126 MB)"
          if wbytes + sbytes > 126e6 else
          f"inputs fit in L2 (W {wbytes / 1e6:.1f} MB + state {sbytes / 1e6:.1f} MB): warm-L2 figure")
    metric = METRIC.replace("(c2,", f"({c.name},").replace("RBCG", a.method.upper())
    line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(c, a.method), "queries_per_gpu": nq, "B": c.B, "n": c.n,
                       "parallelism": f"query-shard x{world}" if world > 1 else "1 GPU",
                       "concurrent_batches": S,
                       "l2": l2,
                       "its_min_med_max": [min(its), int(np.median(its)), max(its)],
                       "offline_greedy_s": round(offline_s, 2), "snapshot_its": snap[:6]},
            "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "kernels": kernels}
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.method == "rbcg":
        try:
            nq_cpu = min(os.cpu_count() or 1, 8)
            v, cores, wall, oits = cpu_oracle_run(c, nq_cpu)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{nq_cpu} c2 queries, one oracle process per core, "
                                              f"RBCG to 1e-10, oracle-built interpolated basis "
                                              f"n=40 (its {min(oits)}-{max(oits)}), wall {wall:.1f}s"}
        except Exception as e:  # reported, never silently dropped
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle",
                                    "sample": f"failed: {e!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
