"""Benchmark of the deferred-compression LoRaSp hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

A step = one pass of the whole hot path on one synthetic system: hs_factor (Algorithm 1:
POTRF, deferred-compression TRSM, CPQR to eps, Schur updates, top Cholesky) followed by
hs_pcg (CSR SpMV + the Algorithm-2 apply) to the config's tolerance.

Default workload: BASELINE.json configs[3] (C4: Q1 first-order-Stokes-type operator, 512 x 512
x 20 hexahedra, 2 DOF/node, 10,485,760 DOF, eps 1e-2, PCG to 1e-8; "1 GPU and 8 GPUs"), the
largest BASELINE config and the one north_star's FP64 target is defined on.  It fits one B200
because the factor records of completed levels spill to pinned host memory while a later
level's block store needs the HBM (level 2: a 131 GB store) and are mapped back at the same
addresses before the apply (RecSpace).  Default K = 2 steps for C4 (a step is
~40 s), 5 otherwise.  --config C3 / C2 / C4/2 / ... run the other configs (a "/k" suffix = the
config's operator on a 1/k horizontal grid).

Inputs (CSR values, b) are resident in HBM when the timed region starts and the analysis
(pattern only) is done once before it.  value = DOF/s = N * K / (device time of the K steps);
e2e repeats the step through the same C API with HOST buffers (values and b uploaded, x
downloaded inside the timed region).  N > 1 (torchrun, one process per GPU): the factor is
partitioned by the 8 fixed subdomains over the GPUs with NCCL exchanges (SURVEY §8(e),
DESIGN.md §7; strong scaling: one system per step), and so is the solve (owner-computes
Algorithm 2 and PCG with a halo SpMV and all-reduced dots, every rank keeping only its own
elimination records); --replicas runs N independent systems instead (weak).  A watchdog aborts a run whose exchanges never complete
(exit 3, an error JSON line).  --impl reference times the CPU oracle (oracle/) on all host
cores on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factor+PCG DOF/s at 1/2/4/8 B200; FP64 TFLOP/s frac of peak; PCG iters"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default: 2 for C4, 5 otherwise")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--cpu-budget", type=float, default=8.0,
                    help="seconds of oracle work per host core for the CPU baseline")
    ap.add_argument("--eps", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent single-GPU factorizations instead of the subdomain-distributed one")
    ap.add_argument("--watchdog", type=float, default=900.0,
                    help="N>1: abort (exit 3) if the run has not finished after this many seconds")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 2 if args.config == "C4" else 5
    return args


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    fp = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    f64 = json.load(open(fp)) if os.path.exists(fp) else {}
    return mp, f64


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.path = f"/tmp/hs_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        load = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _problem(name):
    from problems.generators import gen_config, gen_config_scaled
    if "/" in name:
        base, k = name.split("/")
        return gen_config_scaled(base, int(k))
    return gen_config(name)


def _sample_name(config):
    """The bounded CPU sample of a workload: its family member on a 1/4 horizontal grid (1/16
    of the DOFs for the 2-D-extruded configs; 1/64 for C2) -- same generator, leaf, eps, tol.
    The C4/C5 operators keep high ranks (r/m ~ 0.6-0.8): their oracle samples are the 1/32
    (C4: 10,240 DOF, ~13 s per oracle factor + PCG on one core) and 1/64 grids."""
    base = config.split("/")[0]
    k = int(config.split("/")[1]) if "/" in config else 1
    if base == "C4":
        return f"C4/{max(32, k)}"
    if base == "C5":
        return f"C5/{max(64, k)}"
    return f"{base}/{4 * k}" if base in ("C2", "C3") else base


def _oracle_worker(args):
    """One host core: the oracle as it stands (one BLAS thread) on independent samples until
    its time budget is spent; returns (DOFs factored+solved, seconds, PCG iterations)."""
    name, budget, t_start = args
    import time as _t
    from threadpoolctl import threadpool_limits
    from oracle.analyze import analyze_problem
    from oracle.factor import factor
    from oracle.solve import apply, pcg
    p = _problem(name)
    an = analyze_problem(p)
    A = p.to_scipy()
    while _t.time() < t_start:
        _t.sleep(0.001)
    t0 = _t.perf_counter()
    dofs, its = 0, 0
    with threadpool_limits(1):
        while True:
            f = factor(an, p.rowptr, p.colind, p.vals, eps=p.eps)
            x, rep = pcg(A, p.b, lambda r: apply(f, r), tol=p.tol)
            dofs += p.n
            its = rep.iters
            if _t.perf_counter() - t0 >= budget:
                break
    return dofs, _t.perf_counter() - t0, its


def cpu_pool_run(config, budget):
    """The oracle on every host core (multiprocessing pool, one worker per core, spawn), each
    on independent copies of the bounded sample; value = all DOFs / the slowest worker's time."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    name = _sample_name(config)
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        t_start = time.time() + 5.0 + 0.05 * cores   # every worker has imported and built its sample
        res = pool.map(_oracle_worker, [(name, budget, t_start)] * cores, chunksize=1)
    dofs = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    n1 = _problem(name).n
    return {"value": dofs / wall, "unit": "DOF/s", "cores": cores, "kind": "oracle", "cpu_model": model,
            "sample": f"{name} ({n1} DOF per system, the {config} operator family at reduced horizontal size; same "
                      f"generator, leaf, eps, tol, analyze reading): {cores} processes, one per host core, one BLAS "
                      f"thread each, factor + PCG ({res[0][2]} iterations) of independent systems for >= {budget:.0f} s; "
                      f"{dofs // n1} systems in {wall:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    budget = max(2.0, args.cpu_budget / 2)
    for _ in range(args.warmup):
        cpu_pool_run(args.config, 1.0)
    tot, vals = 0.0, []
    cb = None
    for _ in range(args.steps):
        cb = cpu_pool_run(args.config, budget)
        vals.append(cb["value"])
    value = float(np.mean(vals))
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} (oracle on the host cores, bounded sample: {cb['sample']})"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def khat_level0_flops(H, a, f, p):
    """Level-0 factor flops with the SUPPORT-RESTRICTED column counts of SURVEY §8(d) (k̂_n, k̂_w:
    only the structurally nonzero columns of a block count), next to the dense live counts the
    kernels compute.  Symbolic, host-side: the column support of block (s, q) starts as the CSR
    coupling of the two leaves, grows by the fill of every eliminated t with s, q in n(t)
    (supp(t, q)), and is dense (r_q columns) once q is eliminated (its coarse DOFs)."""
    perm = H.hs_analysis_export(a, H.HS_EXP_PERM)
    loff = H.hs_analysis_export(a, H.HS_EXP_LEAF_OFF)
    nleaf = loff.size - 1
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(perm.size)
    leaf = np.searchsorted(loff, iperm, side="right") - 1          # leaf of every original DOF
    rows = np.repeat(np.arange(p.n), np.diff(p.rowptr))
    lp, lq = leaf[rows], leaf[p.colind]
    sel = lp != lq
    loc = iperm[p.colind[sel]] - loff[lq[sel]]
    supp = {}
    for x, y, c in zip(lp[sel].tolist(), lq[sel].tolist(), loc.tolist()):
        supp.setdefault((x, y), set()).add(c)
    hp, hi = H.hs_analysis_export(a, H.HS_EXP_H_PTR, 0), H.hs_analysis_export(a, H.HS_EXP_H_IDX, 0)
    wp, wi = H.hs_analysis_export(a, H.HS_EXP_W_PTR, 0), H.hs_analysis_export(a, H.HS_EXP_W_IDX, 0)
    bp, bi = H.hs_analysis_export(a, H.HS_EXP_BATCH_PTR, 0), H.hs_analysis_export(a, H.HS_EXP_BATCH_IDX, 0)
    rk = H.hs_factor_export(f, H.HS_FEXP_RANKS, 0)
    done = np.zeros(nleaf, dtype=bool)
    fl_hat = fl_dense = 0.0
    for b in range(bp.size - 1):
        batch = bi[bp[b]:bp[b + 1]].tolist()
        fills = []
        for s_ in batch:
            m = int(loff[s_ + 1] - loff[s_])
            if m == 0:
                continue
            ns, ws = hi[hp[s_]:hp[s_ + 1]].tolist(), wi[wp[s_]:wp[s_ + 1]].tolist()
            def cnt(q, hat):
                if done[q]:
                    return int(rk[q])
                return len(supp.get((s_, q), ())) if hat else int(loff[q + 1] - loff[q])
            r = int(rk[s_])
            for hat in (True, False):
                kn = sum(cnt(q, hat) for q in ns)
                kw = sum(cnt(q, hat) for q in ws)
                K = m - r
                fq = sum(4.0 * (m - j) * (kw - j) + 4.0 * (m - j) * kn for j in range(r))
                v = m ** 3 / 3.0 + m * m * (kn + kw) + fq + K * kn * (kn + 1)
                if hat:
                    fl_hat += v
                else:
                    fl_dense += v
            if r < m:   # fill of the fine DOFs' elimination on n(s) x n(s)
                fills.append([(q, frozenset(supp.get((s_, q), ()))) for q in ns if not done[q]])
        for s_ in batch:
            done[s_] = True
        for nb in fills:
            for x, _ in nb:
                for y, sy in nb:
                    if x != y and sy:
                        supp.setdefault((x, y), set()).update(sy)
    return fl_hat, fl_dense


def run_ours(args, rank, world, local):
    import torch
    from paper_1811_11248_b200 import hsolve as H
    torch.cuda.set_device(local)
    dist_factor = world > 1 and not args.replicas
    if world > 1:
        import threading
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

        def _watchdog():   # an NCCL exchange that never completes must not hang the job
            time.sleep(args.watchdog)
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": "DOF/s", "n_gpus": world,
                                  "error": f"watchdog: no result after {args.watchdog:.0f} s"}), flush=True)
            os._exit(3)
        threading.Thread(target=_watchdog, daemon=True).start()
    p = _problem(args.config)
    if args.eps is not None:
        p.eps = args.eps
    if dist_factor:
        # the factor is partitioned by the 8 fixed subdomains over the ranks
        # (NCCL exchanges inside hs_factor_create), and the solve with it (dsolve.cu)
        uid = [H.hs_nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        h = H.hs_create(local, world, rank, uid[0])
    else:
        h = H.hs_create(local)
    stream = torch.cuda.current_stream()
    H.hs_set_stream(h, stream.cuda_stream)
    t0 = time.perf_counter()
    a = H.hs_analyze(h, p.n, p.rowptr, p.colind, p.coords, p.column_id, leaf_size=p.leaf_size,
                     leaf_columns=p.leaf_columns)
    t_analyze = time.perf_counter() - t0
    vals = torch.tensor(p.vals, dtype=torch.float64, device="cuda")
    b = torch.tensor(p.b, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    solver = True   # the distributed solve is collective: every rank runs hs_pcg (owner-computes)

    def step():
        f = H.hs_factor_create(h, a, vals, eps=p.eps)
        rep = None
        if solver:
            xx, rep = H.hs_pcg(f, b, tol=p.tol, x=x)
        return f, rep

    # the timed steps carry no per-batch CUDA events (each record costs stream time per
    # batch); the phase breakdown and the roofline kernel's live timing come from the
    # profiled steps below (same workload, every phase bracketed with CUDA events)
    os.environ["HS_PHASE_EVENTS"] = "none"
    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks(local)
    l0 = H.hs_launch_count()
    tot_ms = 0.0
    stats, reps = [], []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f, rep = step()
        e1.record(stream)
        e1.synchronize()
        tot_ms += e0.elapsed_time(e1)
        stats.append(H.hs_factor_get_stats(f))
        reps.append(rep)
        del f
    barrier()
    launches = H.hs_launch_count() - l0
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    units = p.n if dist_factor else world * p.n   # distributed: one system split over the GPUs
    value = units * args.steps / (tot_ms * 1e-3)
    # ---- e2e through the C API with host buffers -------------------------------------------
    e2e = None
    hv = np.ascontiguousarray(p.vals)
    if not args.no_e2e:
        hb = np.ascontiguousarray(p.b)
        hx = np.empty_like(hb)
        e2e_ms = 0.0   # (the warm-up steps ran the same kernels; the host-buffer path adds copies)
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f = H.hs_factor_create(h, a, hv, eps=p.eps)
            if solver:
                H.hs_pcg(f, hb, tol=p.tol, x=hx)
            e1.record(stream)
            e1.synchronize()
            e2e_ms += e0.elapsed_time(e1)
            del f
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": units * args.steps / (e2e_ms * 1e-3), "unit": "DOF/s",
               "h2d_bytes_per_step": int(p.vals.nbytes + p.b.nbytes), "d2h_bytes_per_step": int(hx.nbytes)}
    # profiled steps: the same factor, every phase bracketed with CUDA events on the
    # library stream (HS_PHASE_EVENTS=all); the roofline's achieved rate is measured here
    # (one profiled factor for the large configs: a C4 factor is ~40 s); the last one also
    # gives the exports the apply roofline and the k-hat flop count need (a second factor
    # cannot coexist with it at C4's size)
    os.environ["HS_PHASE_EVENTS"] = "all"
    pstats, prof_ms = [], 0.0
    n_prof = 1 if p.n > 4_000_000 else args.steps
    vec, fl0_hat, fl0_dense = 0, None, None
    for i in range(n_prof):
        flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fp = H.hs_factor_create(h, a, hv, eps=p.eps)
        e1.record(stream)
        e1.synchronize()
        prof_ms += e0.elapsed_time(e1)
        pstats.append(H.hs_factor_get_stats(fp))
        if i == n_prof - 1 and rank == 0:
            for lv in range(pstats[-1]["n_levels"]):
                vec += int(H.hs_factor_export(fp, H.HS_FEXP_LIVE0, lv).sum() + H.hs_factor_export(fp, H.HS_FEXP_KN, lv).sum())
            if p.n <= 4_000_000:   # (a host-side Python pass over every CSR entry: minutes at C4)
                fl0_hat, fl0_dense = khat_level0_flops(H, a, fp, p)
        del fp
    os.environ.pop("HS_PHASE_EVENTS")
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0
    # ---- roofline of the dominant kernel class -----------------------------------------------
    mp, f64 = peaks()
    names = ["gather", "potrf", "trsm", "cpqr", "schur", "writeback", "top"]
    t_ph = np.sum([s["t_phase_s"][:7] for s in pstats], axis=0)
    fl_ph = np.sum([s["flops_phase"][:7] for s in pstats], axis=0)
    t_pcg = sum(r["t_pcg_s"] for r in reps)
    t_apply = sum(r["t_apply_s"] for r in reps)
    dom = int(np.argmax(t_ph))
    alu_peak = f64.get("dfma_tflops")
    dmma_peak = f64.get("dmma_tflops") or f64.get("dgemm_tflops")
    if names[dom] in ("potrf", "trsm", "cpqr", "schur", "top"):
        achieved = fl_ph[dom] / t_ph[dom] / 1e12
        peak = alu_peak if alu_peak else None
        roof = {"bound": "alu", "kernel": names[dom],
                "kernels": {"cpqr": "k_cpqr3 (+ k_elim_small: the fused elimination of small-cluster levels)",
                            "potrf": "k_chol (+ G^-1)", "trsm": "k_scale_mma (DMMA)", "schur": "k_schur3 (DMMA)",
                            "top": "dense_potrf"}.get(names[dom], names[dom]),
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if peak else None, "traffic": None,
                "peak_source": "profiles/fp64_peaks.json dfma_tflops (FFMA.F64 chain, measured on this pool's B200)"
                if peak else "FP64 peak not measured yet"}
    else:
        # byte-bound copy kernels: algorithmic bytes are not accounted per phase yet
        roof = {"bound": "hbm", "kernel": names[dom], "achieved": None, "peak": mp.get("hbm_gbs"), "unit": "GB/s",
                "frac": None, "traffic": None}
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (tools/profile_round.sh -> profiles/*_traffic.json; one representative launch)
    # (one per workload: the file's "workload" key, C3 when absent)
    tp = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if "_traffic" in f and f.endswith(".json"))
    for f in reversed(tp):
        tr = json.load(open(os.path.join(ROOT, "profiles", f)))
        if tr.get("workload", "C3") == args.config and tr.get("class") == roof["kernel"]:
            roof["traffic"] = tr["dram_bytes_per_launch"]
            roof["traffic_source"] = f"profiles/{f}: {tr['note']}"
            break
    S = stats[-1]
    factor_flops = float(np.mean([s["flops"] for s in stats]))
    t_fac = float(np.mean([s["t_factor_s"] for s in stats]))
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_pool_run(args.config, args.cpu_budget)
    # ---- HBM-bound kernels: the apply (Algorithm 2) and the CSR SpMV of PCG ------------------
    # algorithmic bytes (§8(d)): apply = T_s (m^2) and C_s (K kn) read by each of the forward
    # and backward sweeps + the top factor twice + vector gathers/scatters (8 bytes each way of
    # every live and neighbour entry per sweep); SpMV = 8 nnz + 4 nnz + 8 (N+1) + 8 N (x) + 8 N (y)
    hbm = mp.get("hbm_gbs")
    apply_bytes = 2.0 * S["factor_bytes"] + 2 * 2 * 8.0 * vec
    # the library counts every level with the column widths its kernels compute: at a
    # support-restricted level 0 those are B_s's supported columns (>= k-hat), dense above
    lib_l0 = float(np.mean([s["flops_level"][0] for s in stats]))
    flops_khat = factor_flops - lib_l0 + fl0_hat if fl0_hat is not None else None
    flops_dense = factor_flops - lib_l0 + fl0_dense if fl0_dense is not None else None
    n_apply = sum(r["iters"] for r in reps)   # z = M^{-1} r once before the loop, then every non-final iteration
    n_spmv = sum(r["iters"] for r in reps)
    t_spmv = sum(r["t_spmv_s"] for r in reps)
    spmv_bytes = 12.0 * p.nnz + 8.0 * (p.n + 1) + 16.0 * p.n

    def bw(bytes_, t, n):
        if not n or not t:
            return None
        ach = bytes_ / (t / n) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm if hbm else None,
                "traffic": None, "bytes_per_launch": bytes_, "us_per_launch": 1e6 * t / n, "launches": n}
    roof["apply"] = bw(apply_bytes, t_apply, n_apply)
    roof["spmv"] = bw(spmv_bytes, t_spmv, n_spmv)
    for key in ("apply", "spmv"):
        tf = os.path.join(ROOT, "profiles", f"r02_traffic_{key}.json")
        if roof[key] and os.path.exists(tf) and args.config == "C3":
            tr = json.load(open(tf))
            roof[key]["traffic"] = tr.get("dram_bytes_per_launch")
            roof[key]["traffic_source"] = f"profiles/r02_traffic_{key}.json: {tr.get('note', '')}"
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if dist_factor else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {p.name}, N={p.n}, nnz={p.nnz}, eps={p.eps}, pcg_tol={p.tol}, "
                               f"leaf={p.leaf_size or p.leaf_columns}",
                   "l2": "256 MB buffer written between timed steps (and the factor working set > L2)",
                   "analyze": "reading R-coarse (coarse_fill=0: structural coarse neighbours, DESIGN.md §2)",
                   "flops": "the column counts the kernels compute (level 0: B_s's supported columns, >= k-hat; levels >= 1: dense live k_n, k_w)",
                   "parallelism": (f"subdomains over {world} GPUs (factor and solve)" if dist_factor
                                   else "replicas" if world > 1 else "single"),
                   "pcg_iters": [r["iters"] for r in reps], "relres_true": reps[-1]["relres_true"],
                   "t_analyze_s": t_analyze, "t_factor_s": t_fac, "t_pcg_s": t_pcg / args.steps,
                   "t_apply_s_per_step": t_apply / args.steps,
                   "factor_tflops": factor_flops / t_fac / 1e12,
                   "factor_gflop": factor_flops / 1e9, "factor_gb": S["factor_bytes"] / 1e9,
                   "factor_gflop_khat": flops_khat / 1e9 if flops_khat else None,
                   "factor_tflops_khat": flops_khat / t_fac / 1e12 if flops_khat else None,
                   "factor_gflop_dense": flops_dense / 1e9 if flops_dense else None,
                   "flops_note": "factor_gflop counts the columns the kernels compute; *_khat counts level 0 with "
                                 "the support-restricted k̂_n, k̂_w of SURVEY §8(d), *_dense with the dense live "
                                 "widths (levels >= 1 are dense in all three)",
                   "phase_s_per_step": {nm: float(t_ph[i] / n_prof) for i, nm in enumerate(names)},
                   "phase_events": f"phases and roofline from {n_prof} profiled factor step(s) (every phase "
                                   f"bracketed with CUDA events, {prof_ms / n_prof:.1f} ms/factor); the timed "
                                   f"steps run without per-batch events",
                   "host_planning_s_per_step": float(np.mean([s["t_phase_s"][7] for s in stats])),
                   "batches": S["n_batches"], "levels": S["n_levels"], "n_top": S["n_top"],
                   "max_m": S["max_m"], "max_rank": S["max_rank"]},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
