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
GPU (torchrun; `--gpus N` without WORLD_SIZE re-launches itself under
torch.distributed.run), no collective on the data path.  c1/c2: every rank its
own query set (weak scaling); c3/c4: one fixed query set (`--queries`) split into
contiguous shards (strong scaling); c5: one 511^3 system, z-slabs over the ranks
(rbs_dist_init, NCCL halos + 3 small allreduces per iteration; strong scaling).  Timing: CUDA events on the solve stream after a
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
    p.add_argument("--shard", default=None, choices=["weak", "strong"],
                   help="weak: every rank its own query set (c1/c2 default); strong: one fixed set split "
                        "over the ranks (c3/c4 default)")
    p.add_argument("--order", default="contrast", choices=["contrast", "given"],
                   help="query-to-batch schedule: group queries of similar coefficient contrast "
                        "(paper_1804_06363_b200.dist.batch_order) or keep the seeded order")
    p.add_argument("--precond", default="post", choices=["post", "sym"],
                   help="RBCG preconditioner: the paper's post-smoothed RBI (default) or the symmetric "
                        "two-level RBI (NEXT(3), RBS_PRECOND_SYM)")
    p.add_argument("--queries", type=int, default=0,
                   help="strong shards / c5: size of the fixed query set (0 = the config's)")
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
    path, idx, mu, cname = args
    import oracle
    from synth import CONFIGS as CF
    c = CF[cname]
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
    if not os.path.exists(path) and c.m <= 63:     # small grids: the oracle greedy itself
        res = oracle.Grid(c.dim, c.m, c.blocks).greedy(train_set(c), c.n)
        np.savez(path, W=res["W"], ANq=res["ANq"], fn=res["fn"])
    if not os.path.exists(path):
        W, ANq, fn = oracle.interpolated_basis(c.dim, c.m, c.blocks, train_set(c), c.n, 63)
        np.savez(path, W=W, ANq=ANq, fn=fn)
    return path


def host_info():
    """CPU model, logical cores and RAM of this host (the cpu_baseline's machine)."""
    model, ram = "unknown", None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "ram_gib": ram}


def cpu_oracle_run(c, nq, offset=0):
    """solve nq queries with the oracle, one process per core (all host cores); returns
    q/s, cores, wall, its, seconds per iteration per query."""
    import multiprocessing as mp
    path = oracle_basis_file(c)
    mus = query_set(c, offset + nq)[offset:]
    cores = min(nq, os.cpu_count() or 1)
    t = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, [(path, i, mus[i], c.name) for i in range(nq)])
    wall = time.perf_counter() - t
    its = [r[2] for r in res]
    s_per_it = statistics.median(r[1] / max(r[2], 1) for r in res)
    return nq / wall, cores, wall, its, s_per_it


def run_reference(a):
    c = CONFIGS[a.config]
    ncpu = os.cpu_count() or 1
    nq = ncpu                  # one query per host core per step (all cores)
    oracle_basis_file(c)
    for w in range(a.warmup):
        cpu_oracle_run(c, nq, offset=w * nq)
    t0 = time.perf_counter()
    tot_q, its_all, cores = 0, [], 1
    for s in range(a.steps):
        _, cores, _, its, _ = cpu_oracle_run(c, nq, offset=(a.warmup + s) * nq)
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
                                       f"RBCG to 1e-10 (host has {ncpu} cores)", "host": host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
# Case 1 with RB dimension 1 and 5, Case 2 with 2 and 10 (AMB-17: the
# text's 10 over the caption's 20), 100 random parameters per case (96 = 6 batches of 16 here)
CASE_M, CASE_B, CASE_TRAIN, CASE_QUERIES = 127, 16, 64, 96
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r2z_traffic.json")
# the exact instantiation each kernel class runs as at each config (what the committed
# ncu capture must name; a capture of another instantiation is not reported)
TIMED_KERNEL = {("c2", "k_gs"): "void k_smooth2<32, 3, 1, 32, 3, 10>(SmoothMarchArgs)",
                ("c2", "k_proj"): "void k_resid2<32, 0, 2>(ResidMarchArgs)",
                ("c2", "k_cgp"): "void k_cgp2<32>(CGP2Args)"}


def ncu_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    ncu --set full capture of the same configuration AND the same kernel instantiation
    (profiles/), else None."""
    try:
        d = json.load(open(TRAFFIC_FILE))
        want = TIMED_KERNEL.get((config, kernel))
        e = d.get("config") == config and d.get(kernel)
        if e and want and e["kernel"] == want:
            return e["dram_bytes_per_launch"], f"{os.path.relpath(TRAFFIC_FILE, ROOT)}: {e['kernel']}"
    except (OSError, ValueError, KeyError):
        pass
    return None, None
CASE_N = {1: 5, 2: 10}


def run_case(a, case):
    """NEXT(4) measurement: the paper's Case 1 / Case 2 (Table 1) as a
    7-point FD face operator on 127^3 interior nodes (h = 1/128, N = 2,048,383; AMB-23):
    GPU greedy basis from 64 seeded training mu with the affine right-hand side
    (untimed; n = 5 for Case 1, 10 for Case 2), 96 queries in batches of
    B = 16, RBCG to 1e-10.  The right-hand side is affine and online (rbs_set_rhs_terms +
    rbs_set_param_map: f(mu) formed in the solve, f_N(mu) = sum_r phi_r f_{N,r}; Case 2's
    bilinear phi in the derived parameters (mu_1, mu_2, mu_1 mu_2)).  A step = one
    rbs_solve_batch of B queries.  1 GPU only."""
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
                        phi_train=np.stack([P["phi"](mu) for mu in tr]), terms=terms, load=False)
    if case == 1:     # theta = (1, mu_1), phi = 1
        s.set_rhs_terms(terms).set_param_map(1, np.array([[1.0, 0.0], [0.0, 1.0]]), None)
    else:             # mu' = (mu_1, mu_2, mu_1 mu_2)
        s.set_rhs_terms(terms).set_param_map(
            3, np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0]]),
            np.array([[1.0, 0, 0, 0], [1.0, 0, -1.0, 0], [0, 0, 1.0, 0], [0, 1.0, 0, -1.0], [0, 0, 0, 1.0]]))
    s.load_basis(gr["W"], gr["ANq"], gr["fn"][0])
    torch.cuda.synchronize()
    offline_s = time.perf_counter() - t0
    q = cases.case_params(case, CASE_QUERIES, 2000 + case)
    qp = q if case == 1 else np.stack([[x, y, x * y] for x, y in q])
    nb = CASE_QUERIES // CASE_B
    N = s.N
    X = torch.empty((CASE_B, N), dtype=torch.float64, device=s.device)
    stream = torch.cuda.current_stream()

    def step(k, **kw):
        b = k % nb
        return s.solve_batch(qp[b * CASE_B:(b + 1) * CASE_B], X=X, want_a_n=False, **kw)

    for w in range(max(a.warmup, 1)):
        step(w)
    clocks = Clocks(0)
    clocks.start()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches, its, trr = 0, [], []
    for k in range(a.steps):
        out = step(k)
        launches += out["launches"]
        its += [int(i) for i in out["its"]]
        trr += [float(v) for v in out["true_relres"]]
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
           "k_gs": 16 * B * N + face_b, "k_prolong": (8 * B * N + 8 * N * n) // 2}   # colour skip
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
                                   "sym-RBGS nu=1, affine rhs online (rbs_set_rhs_terms), tol 1e-10",
                       "B": B, "n": n, "its_min_med_max": [min(its), int(np.median(its)), max(its)],
                       "true_relres_max": max(trr),
                       "offline_greedy_s": round(offline_s, 2),
                       "l2": "inputs larger than L2 (4 x 262 MB state)"},
            "clocks": clk, "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": top, "achieved": kt["GBps"], "peak": hbm,
                         "unit": "GB/s", "frac": kt["GBps"] / hbm, "traffic": None,
                         "peak_source": hbm_src, "alg_bytes_per_launch": kt["alg_bytes"],
                         "avg_launch_us": kt["avg_us"], "share_of_iteration": kt["share"]},
            "kernels": kernels}
    print(json.dumps(line), flush=True)


def spawn(a):
    """`--gpus N` (N > 1) outside torchrun: re-launch under torch.distributed.run, one
    process per GPU, rendezvous on 127.0.0.1."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def run_c5(a, world, rank, local):
    """BASELINE configs[4]: one 3D 511^3 system (N = 133,432,831), 2x2x2 blocks, mu logU
    [0.01, 100]^8, n = 40, B = 8 queries per solve, RBCG.  N = 1: the unpartitioned
    one-GPU reference solve; N > 1: z-slabs over the ranks (rbs_dist_init; NCCL halos and
    3 small allreduces per iteration).  Basis (offline, untimed): the
    multi-fidelity GPU builder of PAPER.md:310 -- GPU greedy on the 127^3 grid selects the
    parameters, the fine-grid snapshots at them solved 8 at a time (RBS_GREEDY_SAMPLES_BATCH).  A step =
    one batch of B queries to convergence on all ranks (the whole job: strong scaling)."""
    import torch
    import torch.distributed as dist
    import paper_1804_06363_b200 as rbs
    c = CONFIGS["c5"]
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    plane = c.m * c.m
    t0 = time.perf_counter()
    n = c.n
    if rank == 0:
        coarse = rbs.Solver(3, 127, c.blocks, device=local)
        grc = coarse.build_greedy(train_set(c), c.n, load=False)
        sel = train_set(c)[grc["selected"]]
        del coarse, grc
        torch.cuda.empty_cache()
        fine = rbs.Solver(3, c.m, c.blocks, device=local)
        gr = fine.build_greedy(sel, c.n, load=False, samples=True, batched=True)
        W, ANq, fn, n = gr["W"], np.asarray(gr["ANq"]), np.asarray(gr["fn"]), gr["n"]
        snap = [int(x) for x in gr["snap_iters"]]
        del fine, gr        # the builder's workspace and its references to W
        torch.cuda.empty_cache()
    if world > 1:
        meta = torch.tensor([n], device=dev)
        dist.broadcast(meta, 0)
        n = int(meta.item())
        At = torch.tensor(ANq, device=dev) if rank == 0 else torch.empty((c.P, n, n), dtype=torch.float64, device=dev)
        ft = torch.tensor(fn, device=dev) if rank == 0 else torch.empty((n,), dtype=torch.float64, device=dev)
        dist.broadcast(At, 0)
        dist.broadcast(ft, 0)
        ANq, fn = At.cpu().numpy(), ft.cpu().numpy()
        uid = [rbs.rbs_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, 0)
        s = rbs.Solver(3, c.m, c.blocks, device=local).dist_init(uid[0], world, rank, 3)
        lr = s.local
        spans = [None] * world
        dist.all_gather_object(spans, (lr["g0"], lr["g1"]))
        rows = torch.empty((lr["n_stored"], n), dtype=torch.float64, device=dev)
        if rank == 0:       # each rank gets the basis rows of its stored planes
            for r, (g0, g1) in enumerate(spans):
                blk = W[(g0 - 1) * plane:(g1 - 1) * plane].contiguous()
                if r == 0:
                    rows.copy_(blk)
                else:
                    dist.send(blk, r)
                del blk
            del W
        else:
            dist.recv(rows, 0)
        s.load_basis(rows, ANq, fn)
        del rows
        snap = snap if rank == 0 else []
    else:
        s = rbs.Solver(3, c.m, c.blocks, device=local).load_basis(W, ANq, fn)
        del W
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    offline_s = time.perf_counter() - t0
    nq = a.queries or c.n_queries
    mus_all = query_set(c, nq)
    nb = max(1, nq // c.B)
    nx = s.local["n_owned"] if world > 1 else c.N
    X = torch.empty((c.B, nx), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    pkw = dict(precond=rbs.RBS_PRECOND_SYM) if a.precond == "sym" else {}

    def step(k, **kw):
        b = k % nb
        return s.solve_batch(mus_all[b * c.B:(b + 1) * c.B], X=X, want_a_n=False, **{**pkw, **kw})

    for w in range(max(a.warmup, 1)):
        step(w)
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches, its, trr = 0, [], []
    for k in range(a.steps):
        out = step(k)
        launches += out["launches"]
        its += [int(i) for i in out["its"]]
        trr += [float(v) for v in out["true_relres"]]
        assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop()
    # e2e: host mu in, X (this rank's owned planes) out to pinned host memory, every step
    # (one solve workspace at a time: each is ~48 GB at 511^3)
    s._ws.clear()
    torch.cuda.empty_cache()
    Xh = torch.empty((c.B, nx), dtype=torch.float64, pin_memory=True)
    s.solve_batch(mus_all[:c.B], X=Xh, x_location=rbs.RBS_MEM_HOST, want_a_n=False, **pkw)
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for k in range(a.steps):
        b = k % nb
        s.solve_batch(mus_all[b * c.B:(b + 1) * c.B], X=Xh, x_location=rbs.RBS_MEM_HOST, want_a_n=False, **pkw)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - te
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    prof = None
    s._ws.clear()
    torch.cuda.empty_cache()
    if world == 1:
        prof = step(0, profile=1, tol=0.0, max_iter=min(a.profile_iters, 10))["profile"]
    hbm, hbm_src = peaks()
    line = {"metric": f"parameter queries solved/sec to rel. residual 1e-10 (c5, RBCG{'-sym' if a.precond == 'sym' else ''}, {world} GPU)",
            "value": a.steps * c.B / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(c), "B": c.B, "n": n,
                       "parallelism": f"mesh z-slabs x{world} (NCCL)" if world > 1 else "1 GPU (reference solve)",
                       "queries": nq, "its_min_med_max": [min(its), int(np.median(its)), max(its)],
                       "preconditioner": "symmetric two-level RBI (RBS_PRECOND_SYM)" if a.precond == "sym"
                       else "post-smoothed RBI (the paper's)",
                       "true_relres_max": max(trr), "offline_s": round(offline_s, 1),
                       "basis": "multi-fidelity GPU builder (127^3 greedy selects, 511^3 snapshots)",
                       "snapshot_its": snap[:6] if rank == 0 else [],
                       "l2": "inputs larger than L2 (W 47 GB + 4 x 8.5 GB state)"},
            "clocks": clk, "gpu_launches": launches,
            "e2e": {"value": a.steps * c.B / e2e_s, "unit": UNIT, "h2d_bytes_per_step": c.B * c.P * 8,
                    "d2h_bytes_per_step": c.B * nx * 8 * world}}
    if prof is not None:
        tot_ms = sum(v[0] for v in prof.values())
        line["kernels"] = {k: {"avg_us": 1e3 * v[0] / max(v[1], 1), "launches": v[1],
                               "share": v[0] / tot_ms if tot_ms else None} for k, v in prof.items() if v[1]}
        # one K1 (k_cgp class) per RBCG iteration; the symmetric preconditioner launches the
        # projection class twice per iteration (K2 and the residual-projection)
        iter_us = 1e3 * tot_ms / max(prof["k_cgp"][1], 1)
        # minimum bytes per batch-iteration: the fused schedule's 80 B + 16n / B per node-query
        # (DESIGN.md §7); the symmetric two-level preconditioner's passes (3D flat schedule: K1,
        # K2, y = 0, 3 pre + 3 post half-sweeps, residual-projection, prolongation) 200 B + 24n / B;
        # 3D z-plane marches: the first pre half-sweep from y = 0 as k_gsz<ZERO> (r of the
        # colour 4 B + both colours' stores 8 B instead of the fill 8 B + a half-sweep 12 B): 192 B
        iter_bytes = ((192 * c.B + 24 * n) if a.precond == "sym" else (80 * c.B + 16 * n)) * c.N
        line["roofline"] = {"bound": "hbm", "kernel": "iteration", "achieved": iter_bytes / (iter_us * 1e-6) / 1e9,
                            "peak": hbm, "unit": "GB/s", "frac": iter_bytes / (iter_us * 1e-6) / 1e9 / hbm,
                            "traffic": None, "peak_source": hbm_src, "alg_bytes_per_launch": iter_bytes,
                            "avg_launch_us": iter_us}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        spawn(a)           # does not return
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RBS_BENCH_SMOKE_1GPU=1: code-path smoke of the N > 1 query-shard bench on a one-GPU box
    # (every rank on cuda:0, gloo for the barrier / max-over-ranks plumbing).  The shards share
    # no data-path collective, so no kernel waits on another rank; the timing is not a scaling
    # number (the ranks share one GPU) and is never reported as one.
    smoke1 = os.environ.get("RBS_BENCH_SMOKE_1GPU") == "1"
    if smoke1:
        local = 0
    if a.config in ("case1", "case2"):
        if a.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "case workloads: GPU measurement only"}))
        elif rank == 0:
            run_case(a, int(a.config[-1]))
        return
    if a.impl == "reference":
        if rank == 0:
            run_reference(a)
        return
    if a.config == "c5":
        run_c5(a, world, rank, local)
        return
    import torch
    import torch.distributed as dist
    import paper_1804_06363_b200 as rbs
    from paper_1804_06363_b200.dist import batch_order, broadcast_basis, gather_counts, query_shard

    torch.cuda.set_device(local)
    if world > 1:
        if smoke1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[a.config]
    shard = a.shard or ("strong" if a.config in ("c3", "c4") else "weak")
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

    # ---- queries ------------------------------------------------------------
    # weak: rank r owns its own n_queries; strong: one fixed set, contiguous shards
    if shard == "weak":
        nq = c.n_queries
        mus_all = query_set(c, nq * world)
        mus = mus_all[rank * nq:(rank + 1) * nq]
        Bq = c.B
    else:
        nq_tot = a.queries or c.n_queries
        q0, q1 = query_shard(nq_tot, world, rank)
        mus = query_set(c, nq_tot)[q0:q1]
        nq = q1 - q0
        Bq = min(c.B, nq)
    if a.order == "contrast":     # batches of similar contrast (dist.batch_order): lanes finish together
        mus = mus[batch_order(mus, Bq)]
    batches = [mus[i:i + Bq] for i in range(0, nq, Bq)]
    nb = len(batches)
    # S concurrent batch streams (DESIGN.md §7 "Concurrent batches"): batch k runs on stream
    # k mod S, each stream with its own context (same basis) and buffers; the batches are
    # independent, so this is a scheduling choice that lets one batch's latency-bound
    # passes overlap another's
    S = max(1, a.streams)
    ss = [s] + [rbs.Solver(c.dim, c.m, c.blocks, device=local).load_basis(W, ANq.cpu().numpy(), fn.cpu().numpy())
                for _ in range(S - 1)]
    sts = [torch.cuda.Stream(device=s.device) for _ in range(S)]
    Xs = [torch.empty((Bq, c.N), dtype=torch.float64, device=s.device) for _ in range(S)]

    mkw = (dict(method=rbs.RBS_RBI, max_iter=500000) if a.method == "rbi" else dict(method=rbs.RBS_RBCG))
    if a.precond == "sym" and a.method == "rbcg":
        mkw["precond"] = rbs.RBS_PRECOND_SYM

    def step(t, k, **kw):
        mb = batches[k % nb]
        return ss[t].solve_batch(mb, X=Xs[t][:len(mb)], stream=sts[t], want_a_n=False, **{**mkw, **kw})

    def run(nsteps, fn_, nvtx=None):
        outs = [[] for _ in range(S)]

        def worker(t):
            torch.cuda.set_device(local)
            if nvtx:
                torch.cuda.nvtx.range_push(nvtx)
            for k in range(t, nsteps, S):
                outs[t].append(fn_(t, k))
            if nvtx:
                torch.cuda.nvtx.range_pop()

        th = [threading.Thread(target=worker, args=(t,)) for t in range(S)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        return [o for ol in outs for o in ol]

    # strong: a step = one pass over this rank's shard (the fixed set over all ranks)
    steps_per = nb if shard == "strong" else 1
    run(max(a.warmup * steps_per, S), step)
    # ---- timed region (device events, max over ranks) ------------------------
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include "timed/" profiles only this
    ev0.record(stream)
    outs = run(a.steps * steps_per, step, nvtx="timed")     # every worker thread marks its launches too
    torch.cuda.synchronize()
    ev1.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches, its, trr, nsolved = 0, [], [], 0
    # lane occupancy: useful node-query iterations / lane-iterations streamed (a batch runs until
    # its slowest query; frozen lanes still stream their rows -- the case for batch compaction)
    lane_used = sum(sum(int(i) for i in o["its"]) for o in outs)
    lane_streamed = sum(len(o["its"]) * max(int(i) for i in o["its"]) for o in outs)
    for out in outs:
        launches += out["launches"]
        its += [int(i) for i in out["its"]]
        trr += [float(v) for v in out["true_relres"]]
        nsolved += len(out["its"])
        assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    if world > 1:
        t = torch.tensor([ms], device=s.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tq = torch.tensor([nsolved], device=s.device)
        dist.all_reduce(tq)
        nsolved = int(tq.item())
        tr = torch.tensor([max(trr)], device=s.device)
        dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        trr = [float(tr.item())]
        dist.barrier()
    clk = clocks.stop()
    value = nsolved / (ms / 1e3)
    if world > 1:   # per-query iteration counts of every rank, for the its statistics
        L = torch.tensor([len(its)], device=s.device)
        Lmax = L.clone()
        dist.all_reduce(Lmax, op=dist.ReduceOp.MAX)
        t_its = torch.full((int(Lmax.item()),), -1, dtype=torch.int32, device=s.device)
        t_its[:len(its)] = torch.tensor(its, dtype=torch.int32, device=s.device)
        all_its, _ = gather_counts(t_its, torch.zeros_like(t_its))
        its = [int(v) for v in all_its.cpu() if v >= 0]

    # ---- e2e: public API with host buffers (pinned X, host mu) --------------
    Xh = [torch.empty((Bq, c.N), dtype=torch.float64, pin_memory=True) for _ in range(S)]

    def step_host(t, k):
        mb = batches[k % nb]
        return ss[t].solve_batch(mb, X=Xh[t][:len(mb)], x_location=rbs.RBS_MEM_HOST,
                                 stream=sts[t], want_a_n=True, **mkw)

    run(S, step_host)      # warm-up: host-output workspace and its iteration graph per context
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    eo = run(a.steps * steps_per, step_host)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t
    ne = sum(len(o["its"]) for o in eo)
    if world > 1:
        tt = torch.tensor([e2e_s], device=s.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
        tq = torch.tensor([ne], device=s.device)
        dist.all_reduce(tq)
        ne = int(tq.item())
    e2e = {"value": ne / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": Bq * c.P * 8,
           "d2h_bytes_per_step": Bq * c.N * 8 + Bq * (4 + 4 + 8 + 8 + 8 * c.n)}

    # ---- per-kernel device times (eager, events on the launching stream) -----
    prof = step(0, 0, profile=1, tol=0.0, max_iter=a.profile_iters)["profile"]
    hbm, hbm_src = peaks()
    # queries per pass: 2D batches above 32 run as 32-query sub-batches
    Bp_ = min(Bq, 32) if c.dim == 2 else Bq
    N, n = c.N, c.n
    # algorithmic bytes per launch (each vector once, W once per batch)
    alg = {"k_cgp": 24 * Bp_ * N,                    # y, p_old read; p_new written
           "k_proj": 40 * Bp_ * N + 8 * N * n,       # p, x, r read; x, r written; W
           "k_gs": 16 * Bp_ * N + 8 * N * n}         # 2D fused smoother: r read, y written; W
    if a.method == "rbi" and c.dim == 3:
        # 3D RBI: x_old + W e for the nodes outside the first half-sweep's colour (x_old, W
        # rows read, x written: half), one half-sweep per k_gs launch (x read, one colour of x
        # written; f constant), Step 2's residual-projection at its minimum (x, W read)
        alg = {"k_prolong": (16 * Bp_ * N + 8 * N * n) // 2, "k_gs": 12 * Bp_ * N,
               "k_proj": 8 * Bp_ * N + 8 * N * n}
    elif a.method == "rbi":   # RBI: K3' x_new = S(x_old + W e) (x_old, W read; x written), resid f - A x + W^T (x, W)
        alg = {"k_gs": 16 * Bp_ * N + 8 * N * n, "k_proj": 8 * Bp_ * N + 8 * N * n}
    elif c.dim == 3:   # separate prolongation pass; k_gs is one red-black half-sweep per launch
        # W read, y0 written -- for the nodes outside the first half-sweep's colour only (the
        # colour skip of k_prolong: those nodes are overwritten unread)
        alg["k_prolong"] = (8 * Bp_ * N + 8 * N * n) // 2
        alg["k_gs"] = 16 * Bp_ * N                   # y read, r and y of one colour
    flops = {"k_proj": 2.0 * N * n * Bp_, "k_gs": 2.0 * N * n * Bp_}   # W^T r / W e on DMMA
    if c.dim == 3:   # 3D: W e in its own pass (half the rows: colour skip); k_gs is a half-sweep
        flops = {"k_proj": 2.0 * N * n * Bp_, "k_prolong": 1.0 * N * n * Bp_}
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
    iter_us = 1e3 * tot_ms / max(prof["k_proj"][1], 1)     # per pass-iteration of Bp_ queries
    iter_bytes = ((24 * Bp_ + 16 * n) if a.method == "rbi" else
                  ((192 if c.dim == 3 else 200) * Bp_ + 24 * n) if a.precond == "sym" else
                  (80 * Bp_ + 16 * n)) * N   # per batch-iteration (3D sym: k_gsz<ZERO> pre-sweep)
    traffic, traffic_src = ncu_traffic(a.config, top)
    roof = {"bound": "hbm", "kernel": top, "timed_instantiation": TIMED_KERNEL.get((a.config, top)),
            "achieved": kt["GBps"], "peak": hbm, "unit": "GB/s",
            "frac": kt["GBps"] / hbm, "traffic": traffic, "traffic_source": traffic_src, "peak_source": hbm_src,
            "alg_bytes_per_launch": kt["alg_bytes"], "avg_launch_us": kt["avg_us"],
            "share_of_iteration": kt["share"],
            "iteration": {"us": iter_us, "alg_bytes": iter_bytes,
                          "GBps": iter_bytes / (iter_us * 1e-6) / 1e9,
                          "frac": iter_bytes / (iter_us * 1e-6) / 1e9 / hbm},
            "solve_level": None,
            "fp64_tensor_peak_tflops": FP64_TENSOR_MEASURED_TFS,
            "fp64_tensor_peak_source": "measured, tools/fp64_peak.cu (DMMA m8n8k4, all SMs)"}
    # solve level: the whole timed region against the per-iteration minimum bytes
    # (queries x iterations x (80 + 16 n / B) B per node), concurrency included
    it_q = sum(its) / max(len(its), 1)
    per_q = (iter_bytes / Bp_) * it_q
    roof["solve_level"] = {"GBps": value * per_q / 1e9, "frac": value * per_q / 1e9 / hbm / max(world, 1),
                           "mean_its": it_q}

    wbytes, sbytes = c.N * (((c.n + 7) // 8) * 8 + 4) * 8, 4 * c.N * Bq * 8
    l2 = (f"inputs larger than L2 (W {wbytes / 1e6:.0f} MB + 4 x {sbytes / 4e6:.0f} MB state > 126 MB)"
          if wbytes + sbytes > 126e6 else
          f"inputs fit in L2 (W {wbytes / 1e6:.1f} MB + state {sbytes / 1e6:.1f} MB): warm-L2 figure")
    metric = METRIC.replace("(c2,", f"({c.name},").replace(
        "RBCG", a.method.upper() + ("-sym" if a.precond == "sym" and a.method == "rbcg" else ""))
    if world > 1:
        metric = metric.replace("1 GPU)", f"{world} GPUs)")
    line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": shard, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(c, a.method), "B": Bq, "n": c.n,
                       "queries_per_gpu": nq,
                       "queries_total": (a.queries or c.n_queries) if shard == "strong" else nq * world,
                       "step": "one pass over the rank's query shard" if shard == "strong" else "one batch of B queries",
                       "parallelism": f"query-shard x{world} ({shard})" if world > 1 else "1 GPU",
                       "concurrent_batches": S, "batch_order": a.order,
                       "l2": l2,
                       "its_min_med_max": [min(its), int(np.median(its)), max(its)],
                       "lane_occupancy": round(lane_used / max(lane_streamed, 1), 4),
                       "true_relres_max": max(trr),
                       "offline_greedy_s": round(offline_s, 2), "snapshot_its": snap[:6]},
            "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "kernels": kernels}
    if rank == 0 and world == 1 and not a.no_cpu_baseline and a.method == "rbcg" and c.name in ("c1", "c2"):
        try:
            nq_cpu = min(os.cpu_count() or 1, 32)
            v, cores, wall, oits, spi = cpu_oracle_run(c, nq_cpu)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{nq_cpu} {c.name} queries, one oracle process per host core, "
                                              f"RBCG to 1e-10, oracle-built interpolated basis n={c.n} "
                                              f"(its {min(oits)}-{max(oits)}; the GPU arm's basis comes from its own "
                                              f"builder: the oracle takes no input from the CUDA path), "
                                              f"wall {wall:.1f}s",
                                    "s_per_iteration_per_query": spi,
                                    "gpu_s_per_iteration_per_query": (ms / 1e3) / max(sum(its), 1),
                                    "host": host_info()}
        except Exception as e:  # reported, never silently dropped
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle",
                                    "sample": f"failed: {e!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
