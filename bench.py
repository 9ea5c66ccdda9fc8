"""Headline benchmark: elastodynamic U H-matvec at N_c = 32,768 (BASELINE.json
config 3, "100 timed H-matvecs with seeded complex Gaussian input vectors").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hmx|reference] [--config U32k]

A step is one H-matvec y = A_H x_j over the assembled H-matrix (x_j a fresh
seeded complex Gaussian vector per step, already in HBM).  ``value`` is the
algorithmic H-matvec traffic of all ranks divided by the device time of the K
steps (max over ranks): GB/s.  The packed H streams (10.5 GB at U32k) are far
larger than the 126 MB L2, so no L2 flush is needed between steps.

Multi-GPU (N > 1; ``--gpus N`` outside torchrun re-launches itself as N
ranks): the row-sharded H of SURVEY 8(e) -- rank p assembles the leaves of
its owned row range, a step is the local matvec plus one all-gather of the
owned y segments; value = full-H bytes x K / max-over-ranks device time,
scaling "strong".  ``--replicas`` runs independent full copies instead.

``--impl reference`` times the reference's CPU implementation of the same
path (the oracle restatement, oracle/hmatrix.py, all host threads) on the
same workload -- every U32k leaf assembled in a process pool, then full
oracle H-matvecs -- and prints the same JSON line shape.
"""

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0
SEED = 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hmx", choices=["hmx", "reference"])
    ap.add_argument("--config", default="U32k")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the T65k time-to-solve run")
    ap.add_argument("--no-reserve", action="store_true",
                    help="do not reserve the context's device arena up front (hmx_ctx_reserve): every assembly then "
                         "allocates its workspaces with cudaMalloc inside its timed region")
    ap.add_argument("--no-estimate", action="store_true", help="skip the delta_{H,F} estimator timing")
    ap.add_argument("--solve-config", default="T65k")
    ap.add_argument("--no-direct", action="store_true", help="skip the H-LU direct-solve section")
    ap.add_argument("--direct-config", default="H4k,U8k@2562",
                    help="H-LU direct-solve workloads (TAG or TAG@points; U8k@2562 = 7,686 dofs, the paper's Table 5 size)")
    ap.add_argument("--extra-configs", default="U32k45,U131k,U8k,H4k",
                    help="other BASELINE configs measured briefly (assembly + 20 matvecs); '' to skip")
    ap.add_argument("--shard", action="store_true",
                    help="row-sharded H (SURVEY 8(e)) even at N = 1 (the default for N > 1): each rank "
                         "assembles the leaves of its owned row range, one all-gather of y per matvec, "
                         "strong scaling")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent full replicas instead of the row-sharded H (weak scaling)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": FALLBACK_HBM_GBS}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_problem(tag, stripe=None):
    """The oracle's inputs for workload ``tag``: every leaf (stripe None, the same
    configuration as the device run) or, for a quick bounded sample, the leaves whose row
    cluster lies in the first 1/stripe of the tree-ordered rows (keeps the leaf mix)."""
    from oracle import geometry as OG
    from paper_1706_09384_b200.configs import WORKLOADS
    from tests._problems import oracle_params, spec_for

    w = WORKLOADS[tag]
    pts, nrm = OG.sphere_cloud(w.n_points)
    ct = OG.cluster_tree(pts, w.n_leaf)
    lv = OG.block_leaves(ct, ct, w.eta)
    tab = OG.leaf_table(ct, ct, lv)
    params = oracle_params(spec_for(w))
    if stripe is None:
        return w, ct, nrm, tab, params, f"all {len(tab)} leaves of {tag} (same configuration as the device run)"
    cut = w.n_points // stripe
    sel = np.flatnonzero(tab[:, 2] <= cut)
    return w, ct, nrm, tab[sel], params, f"rows [0, {cut}) of {tag} (1/{stripe} block-row stripe, {len(sel)} leaves)"


def run_cpu(tag, steps, warmup, budget_s=None, stripe=None):
    """The oracle (oracle/hmatrix.py) on the host cores: leaf-parallel assembly in a fork pool
    (SPEC.md:456), then ``steps`` threaded H-matvecs (permutation to tree order, every leaf,
    permutation back), each timed; returns throughput (bytes of all steps / their total time)
    and the median step."""
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    from oracle import hmatrix as OH

    w, ct, nrm, tab, params, desc = cpu_problem(tag, stripe)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oh = OH.assemble(w.kind, params, ct.points_tree, None if w.kind != "T" else nrm[ct.perm], ct.perm, tab, w.eps,
                     self_shift=float(w.n_points), workers=cores)
    t_setup = time.perf_counter() - t0
    d = w.d
    m = (tab[:, 2] - tab[:, 1]).astype(np.float64)
    n = (tab[:, 4] - tab[:, 3]).astype(np.float64)
    cost = np.where(tab[:, 0] == 0, d * d * m * n, oh.rank_after * d * (m + n))
    bytes_ = 16.0 * float(cost.sum()) + 32.0 * d * w.n_points
    # balanced leaf chunks (LPT on the leaf bytes), one per thread
    order = np.argsort(-cost, kind="stable")
    chunks = [[] for _ in range(cores)]
    load = np.zeros(cores)
    for b in order:
        i = int(np.argmin(load))
        chunks[i].append(int(b))
        load[i] += cost[b]
    rng = np.random.default_rng(SEED)
    nd = d * w.n_points
    xs = [rng.standard_normal(nd) + 1j * rng.standard_normal(nd) for _ in range(4)]

    def step(x, pool):
        return OH.from_tree(oh, OH.matvec_tree_threads(oh, OH.to_tree(oh, x), pool, chunks))

    times = []
    with ThreadPoolExecutor(cores) as pool, threadpool_limits(1):
        for j in range(warmup):
            step(xs[j % 4], pool)
        t_all = time.perf_counter()
        for j in range(steps):
            t0 = time.perf_counter()
            step(xs[j % 4], pool)
            times.append(time.perf_counter() - t0)
            if budget_s is not None and time.perf_counter() - t_all > budget_s:
                break
    dt = float(sum(times))
    done = len(times)
    pairs = int(np.sum(np.where(tab[:, 0] == 0, m * n, oh.steps * (m + n))))
    return {"value": bytes_ * done / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "same_config": stripe is None,
            "sample": f"{desc}; oracle factors (numpy ACA + QR/SVD recompression); {done} threaded "
                      f"oracle H-matvecs of {bytes_ / 1e9:.3f} GB each", "ms_per_step": dt / done * 1e3,
            "ms_per_step_median": float(np.median(times)) * 1e3, "steps": done, "setup_s": t_setup,
            "max_rank_after": int(oh.rank_after.max()),
            "assembly": {"pooled_s": t_setup, "workers": cores, "pairs": pairs,
                         "green_entries_per_s": d * d * pairs / t_setup,
                         "sample": f"{desc}, leaf-parallel process pool (SPEC.md:456)"}}


def cpu_end_to_end(tag="H4k"):
    """The reference's own CPU-runnable configuration (BASELINE config 1) end to end on the host:
    oracle assembly in a process pool, one H-matvec, GMRES(50, 1e-4) -- SURVEY 8(d)'s CPU
    assembly / matvec / GMRES baseline at full size."""
    from threadpoolctl import threadpool_limits

    from oracle import hmatrix as OH
    from oracle import solve as OS
    from tests._problems import Problem

    cores = os.cpu_count() or 1
    pb = Problem(tag)
    t0 = time.perf_counter()
    oh = pb.oracle_h(workers=cores)
    t_asm = time.perf_counter() - t0
    b = pb.rhs(SEED)
    with threadpool_limits(cores):
        t0 = time.perf_counter()
        for _ in range(5):
            OH.matvec(oh, b)
        t_mv = (time.perf_counter() - t0) / 5
        t0 = time.perf_counter()
        _, it, _, conv = OS.gmres(lambda v: OH.matvec(oh, v), b, 1e-4, 50, 1000)
        t_gm = time.perf_counter() - t0
    return {"workload": tag, "cores": cores, "kind": "port", "assembly_pooled_s": t_asm, "matvec_ms": 1e3 * t_mv,
            "gmres_s": t_gm, "gmres_iterations": it, "converged": bool(conv),
            "time_to_solve_s": t_asm + t_gm}


def reference_arm(args):
    """BASELINE config 3 on the host: the oracle assembles every U32k leaf, then times
    ``--steps`` full oracle H-matvecs (bounded at ~3 minutes of steps)."""
    ws, rank, local = dist_setup(args)
    if rank != 0:
        return
    r = run_cpu(args.config, args.steps, args.warmup, budget_s=180.0)
    line = {
        "impl": "reference", "metric": f"{args.config} H-matvec algorithmic HBM throughput (elasto U)",
        "value": r["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (Fibonacci sphere, seeded complex Gaussian x)",
        "config": {"workload": f"{args.config} H-matvec", "sample": r["sample"], "same_config": r["same_config"]},
        "cpu_baseline": {"value": r["value"], "unit": "GB/s", "cores": r["cores"], "kind": "port",
                         "cpu_model": r["cpu_model"], "sample": r["sample"],
                         "ms_per_step_median": r["ms_per_step_median"], "assembly": r["assembly"]},
        "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
def time_to_solve(tag, device):
    """BASELINE config 5: assembly + GMRES(restart 50, tol 1e-4) on the
    elastodynamic T kernel, seeded complex Gaussian RHS; device-timed phases
    plus the host tree build."""
    import torch

    import paper_1706_09384_b200 as hmx
    from paper_1706_09384_b200.configs import WORKLOADS

    w = WORKLOADS[tag]
    t0 = time.perf_counter()
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    t_tree = time.perf_counter() - t0
    torch.cuda.synchronize()
    free_before = torch.cuda.mem_get_info(device)[0]
    t0 = time.perf_counter()
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=device)
    t_asm = time.perf_counter() - t0
    st = H.stats()
    n = w.d * w.n_points
    rng = np.random.default_rng(SEED)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    t0 = time.perf_counter()
    res = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-4, restart=50))
    t_gm = time.perf_counter() - t0
    r = b - hmx.matvec(H, res.x)
    out = {"workload": tag, "n_points": w.n_points, "ks": w.ks, "iterations": res.iters,
           "converged": res.converged, "true_rel_residual": float(np.linalg.norm(r) / np.linalg.norm(b)),
           "assembly_ms": st["t_total_ms"], "assembly_wall_s": t_asm, "gmres_s": t_gm, "tree_build_s": t_tree,
           "time_to_solve_s": st["t_total_ms"] * 1e-3 + t_gm,
           "time_to_solve_with_tree_s": st["t_total_ms"] * 1e-3 + t_gm + t_tree,
           "max_rank_before": rep.max_rank_before, "max_rank_after": rep.max_rank_after,
           "matvec_bytes": st["matvec_bytes"], "aca_passes": st["aca_passes"],
           "free_gb_before_assembly": free_before / 1e9, "n_fallback": st["n_fallback"]}
    # warm: the same job again in the same process (workspaces from the context cache)
    del H
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=device)
    st = H.stats()
    t0 = time.perf_counter()
    res = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-4, restart=50))
    t_gm = time.perf_counter() - t0
    out["warm"] = {"assembly_ms": st["t_total_ms"], "gmres_s": t_gm, "iterations": res.iters,
                   "time_to_solve_s": st["t_total_ms"] * 1e-3 + t_gm}
    out["note"] = ("time_to_solve_s: first assembly of this workload in the process (its workspaces come from the "
                   "context's reserved arena, or with --no-reserve from cudaMalloc after the other sections "
                   "released theirs); warm: the same job repeated")
    del H
    return out


def direct_solve(tag, device, eps_lu=1e-4, cpu=True):
    """H-LU of the assembled H with eps_LU and one
    triangular solve on the device (a second factorisation is timed: the first call warms
    cuSOLVER / the allocator), GMRES on the same H for comparison, and the oracle's H-LU of the same
    leaf factors on one host core as the section's CPU baseline."""
    import torch

    import paper_1706_09384_b200 as hmx
    from paper_1706_09384_b200 import hierarchical_lu as HL
    from paper_1706_09384_b200.configs import WORKLOADS

    base, _, npts = tag.partition("@")
    w = WORKLOADS[base] if not npts else WORKLOADS[base].with_points(int(npts))
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=device)
    n = w.d * w.n_points
    rng = np.random.default_rng(SEED)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    HL.hlu(H, eps_lu)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = HL.hlu(H, eps_lu)
    t_lu = time.perf_counter() - t0
    t0 = time.perf_counter()
    x = HL.triangular_solve(f, b)
    t_sv = time.perf_counter() - t0
    y = hmx.matvec(H, b)
    cons = float(np.linalg.norm(HL.lu_matvec(f, b) - y) / np.linalg.norm(y))
    res = float(np.linalg.norm(hmx.matvec(H, x) - b) / np.linalg.norm(b))
    t0 = time.perf_counter()
    g = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-4, restart=50))
    t_gm = time.perf_counter() - t0
    out = {"workload": f"{tag} H-LU (eps_LU {eps_lu:g}) + triangular solve", "dofs": n,
           "hlu_s": t_lu, "solve_ms": 1e3 * t_sv, "consistency_LU_vs_AH": cons, "residual": res,
           "rel_diff_vs_gmres": float(np.linalg.norm(g.x - x) / np.linalg.norm(x)),
           "gmres_s": t_gm, "gmres_iterations": g.iters,
           "factor_storage_MB": f.storage() * 16 / 1e6, "h_storage_MB": rep.n_stored * 16 / 1e6,
           "truncations": f.stats["n_truncations"], "truncate_calls": f.stats["n_truncate_calls"],
           "truncate_s": f.stats["truncate_s"], "dense_leaf_lu": f.stats["n_getrf"],
           "max_rank": f.stats["max_rank"]}
    if cpu:
        from threadpoolctl import threadpool_limits

        from oracle import hlu as OL

        payload = [H.block(i) for i in range(len(H.table))]
        payload = [p if isinstance(p, np.ndarray) else (p.u, p.v) for p in payload]
        with threadpool_limits(1):
            root = OL.from_payload(bt, w.d, payload)
            t0 = time.perf_counter()
            OL.hlu(root, eps_lu)
            t_cpu = time.perf_counter() - t0
        out["cpu_baseline"] = {"hlu_s": t_cpu, "cores": 1, "kind": "port",
                               "sample": "oracle/hlu.py (numpy / LAPACK QR + SVD truncations) on the same leaf factors, "
                                         "one thread"}
    del f, H
    torch.cuda.empty_cache()
    return out


def config_summary(tag, device, dfma_tflops, steps=20):
    """Brief measurement of another BASELINE config: steady-state assembly
    (second call) and the device H-matvec (mean of ``steps`` calls)."""
    import torch

    import paper_1706_09384_b200 as hmx
    from paper_1706_09384_b200.configs import WORKLOADS
    from paper_1706_09384_b200.flops import PAIR_FLOPS, survey_flops

    w = WORKLOADS[tag]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=device)
    # steady state: the fastest of three repeated assemblies (a single sample of a 3-35 ms job is at the
    # mercy of one host hiccup between its launches)
    st, asm_ms = None, []
    for _ in range(3):
        del H
        H, rep = hmx.assemble(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=device)
        s_i = H.stats()
        asm_ms.append(s_i["t_total_ms"])
        if st is None or s_i["t_total_ms"] < st["t_total_ms"]:
            st = s_i
    n = w.d * w.n_points
    x = torch.randn(n, dtype=torch.complex128, device=f"cuda:{device}")
    y = torch.empty_like(x)
    for _ in range(3):
        hmx.matvec(H, x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        hmx.matvec(H, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    mv_ms = e0.elapsed_time(e1) / steps
    bi = H.block_info()
    t = st["t_total_ms"] * 1e-3
    sv, _ = survey_flops(H.table, bi["steps"], bi["rank_before"], bi["rank_after"], w.d, w.kind,
                         st["pairs_evaluated"])
    ex = st["flops_assembly"] + PAIR_FLOPS[w.kind] * st["pairs_evaluated"]
    out = {"n_points": w.n_points, "kind": w.kind, "n_leaf": w.n_leaf, "assembly_ms": st["t_total_ms"],
           "assembly_ms_samples": asm_ms,
           "green_entries_per_s": w.d * w.d * st["pairs_evaluated"] / t,
           "fp64_frac_survey_model": sv / t / 1e12 / dfma_tflops, "fp64_frac_executed": ex / t / 1e12 / dfma_tflops,
           "matvec_ms": mv_ms, "matvec_GBps": st["matvec_bytes"] / (mv_ms * 1e-3) / 1e9,
           "matvec_bytes": st["matvec_bytes"], "l2_resident": st["matvec_bytes"] < 100e6,
           "max_rank_after": rep.max_rank_after, "tau": rep.tau}
    if "gmres" in w.runs:
        rng = np.random.default_rng(SEED)
        b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        t0 = time.perf_counter()
        g = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-4, restart=50))
        out["gmres_s"] = time.perf_counter() - t0
        out["gmres_iterations"] = g.iters
        out["time_to_solve_s"] = t + out["gmres_s"]
    del H
    return out


def hmx_arm(args):
    import torch

    import paper_1706_09384_b200 as hmx
    from paper_1706_09384_b200 import _lib
    from paper_1706_09384_b200.configs import WORKLOADS
    from paper_1706_09384_b200.dist import replica_throughput
    from tests._problems import spec_for

    ws, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = WORKLOADS[args.config]
    t0 = time.perf_counter()
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    t_tree = time.perf_counter() - t0
    spec = spec_for(w)
    # untimed set-up, like loading a model: one reserved device region serves every assembly's
    # workspaces and streams from here on (no cudaMalloc / cudaFree inside the timed regions, whose
    # cost varies 10x between the boxes of the pool)
    reserve_s = None
    if not args.no_reserve:
        try:
            reserve_s = _lib.reserve(local, 0.0)
        except Exception as exc:  # e.g. a co-tenant holds the memory: per-assembly allocation instead
            print(f"[bench] hmx_ctx_reserve failed ({exc!r}); continuing with per-assembly cudaMalloc", file=sys.stderr)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H, rep = hmx.assemble(spec, cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=local)
    t_asm_wall = time.perf_counter() - t0
    st = H.stats()
    # steady state: a second assembly of the same problem (workspaces come from the
    # context's allocator cache instead of fresh cudaMalloc first touches)
    del H
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H, rep = hmx.assemble(spec, cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), device=local)
    t_asm_wall_warm = time.perf_counter() - t0
    st_warm = H.stats()
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)  # launch stream of every timed matvec (the CUDA events' stream)
    n = w.d * w.n_points
    K, W = args.steps, args.warmup
    rng = np.random.default_rng(SEED + rank)
    X = torch.from_numpy(np.stack([rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(K + W)]))
    Xd = X.to(f"cuda:{local}")
    Y = torch.empty(n, dtype=torch.complex128, device=f"cuda:{local}")
    L = _lib.lib()
    hp = H.handle

    def mv_dev(j):
        _lib.check(L.hmx_matvec_on(hp, C.c_void_p(Xd[j].data_ptr()), C.c_void_p(Y.data_ptr()), 1, sp), "matvec")

    for j in range(W):
        mv_dev(K + j)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    peaks, peak_kind = measured_peaks()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        _lib.check(L.hmx_profile_begin(hp), "profile")
        e0.record()
        for j in range(K):
            mv_dev(j)
        e1.record()
        torch.cuda.synchronize()
    ncalls = C.c_int64()
    ph = np.zeros(4)
    _lib.check(L.hmx_profile_end(hp, C.byref(ncalls), _lib.ptr(ph)), "profile")
    ms = e0.elapsed_time(e1)
    clocks = clk.summary()
    mv_bytes = st["matvec_bytes"]
    value, ms_max = replica_throughput(ms, mv_bytes, K, f"cuda:{local}")

    # ---- e2e through the C-ABI with pinned host buffers (H2D + kernels + D2H per step)
    Xh = X.pin_memory()
    Yh = torch.empty(n, dtype=torch.complex128).pin_memory()
    for j in range(W):
        _lib.check(L.hmx_matvec_on(hp, C.c_void_p(Xh[K + j].data_ptr()), C.c_void_p(Yh.data_ptr()), 0, sp), "matvec")
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for j in range(K):
        _lib.check(L.hmx_matvec_on(hp, C.c_void_p(Xh[j].data_ptr()), C.c_void_p(Yh.data_ptr()), 0, sp), "matvec")
    f1.record()
    torch.cuda.synchronize()
    e2e_serial, e2e_serial_ms = replica_throughput(f0.elapsed_time(f1), mv_bytes, K, f"cuda:{local}")
    # the same K host-buffer calls from two host threads on two streams (an assembled H is safe for
    # concurrent matvec: per-stream workspaces): one call's PCIe copies overlap the other
    # call's kernels.  Every step still copies its x in and its y out inside the timed region.
    import threading

    streams = [torch.cuda.Stream(device=local), torch.cuda.Stream(device=local)]
    Yh2 = [Yh, torch.empty(n, dtype=torch.complex128).pin_memory()]
    for t in range(2):
        for j in range(W):
            _lib.check(L.hmx_matvec_on(hp, C.c_void_p(Xh[K + j].data_ptr()), C.c_void_p(Yh2[t].data_ptr()), 0,
                                       int(streams[t].cuda_stream)), "matvec")
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    g0 = torch.cuda.Event(enable_timing=True)
    g0.record(streams[0])
    streams[1].wait_event(g0)
    errs = []

    def worker(t):
        try:
            for j in range(t, K, 2):
                _lib.check(L.hmx_matvec_on(hp, C.c_void_p(Xh[j].data_ptr()), C.c_void_p(Yh2[t].data_ptr()), 0,
                                           int(streams[t].cuda_stream)), "matvec")
        except Exception as exc:  # reported below
            errs.append(exc)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    g1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for t in range(2):
        g1[t].record(streams[t])
    torch.cuda.synchronize()
    e2e_value, e2e_ms = replica_throughput(max(g0.elapsed_time(e) for e in g1), mv_bytes, K, f"cuda:{local}")

    # ---- roofline of the dominant kernel (phase 2: row-stream GEMV)
    nc = max(int(ncalls.value), 1)
    p1_ms, p2_ms = ph[1] / nc, ph[2] / nc
    fused = p2_ms == 0.0  # phases 1 + 2 in one launch (mv_fused)
    if fused:
        dom_kernel, dom_bytes, dom_ms = "mv_fused", st["phase1_bytes"] + st["phase2_bytes"], p1_ms
    else:
        dom_kernel, dom_bytes, dom_ms = "mv_phase2", st["phase2_bytes"], p2_ms
    dom_gbs = dom_bytes / (dom_ms * 1e-3) / 1e9
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(args.config, {}).get(dom_kernel)
        except Exception:
            traffic = None
    # ---- assembly roofline (FP64)
    dfma = C.c_double()
    _lib.check(L.hmx_bench_dfma(_lib.context(local), C.byref(dfma)), "dfma")
    read_bw = C.c_double()  # read-only streaming rate: the matvec kernels read ~all their bytes
    _lib.check(L.hmx_bench_read_bw(_lib.context(local), C.byref(read_bw)), "read_bw")
    from paper_1706_09384_b200.flops import PAIR_FLOPS

    pair_flops = PAIR_FLOPS[w.kind] * st["pairs_evaluated"]
    asm_flops = st["flops_assembly"] + pair_flops
    t_asm = st["t_total_ms"] * 1e-3
    t_asm_warm = st_warm["t_total_ms"] * 1e-3
    from paper_1706_09384_b200.flops import survey_flops

    bi = H.block_info()
    sv_flops, sv_parts = survey_flops(H.table, bi["steps"], bi["rank_before"], bi["rank_after"], w.d, w.kind,
                                      st["pairs_evaluated"])
    entries = w.d * w.d * st["pairs_evaluated"]
    line = {
        "metric": f"{args.config} H-matvec algorithmic HBM throughput (elasto U)",
        "value": value, "unit": "GB/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (Fibonacci sphere, seeded complex Gaussian x, seed 0)",
        "config": {"workload": f"{args.config} H-matvec", "kernel": "elasto U", "n_points": w.n_points,
                   "n_leaf": w.n_leaf, "eta": w.eta, "eps_aca": w.eps, "ks": w.ks,
                   "parallelism": f"replicas x{ws}",
                   "l2": "inputs larger than L2 (H streams %.1f GB vs 126 MB L2), no flush" % (mv_bytes / 1e9),
                   "allocator": ("cudaMalloc per assembly (caching allocator)" if reserve_s is None else
                                 "context arena reserved before the first assembly (hmx_ctx_reserve, 88%% of the free "
                                 "device memory, %.3f s, untimed): the assemblies of every section call no "
                                 "cudaMalloc / cudaFree; --no-reserve restores per-assembly allocation" % reserve_s)},
        "gpu_launches": 4 * K,
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
                "ms_per_step": e2e_ms / K,
                "mode": "hmx_matvec_on with pinned host x / y, two host threads on two streams (copies of one "
                        "call overlap the other's kernels)",
                "serial_value": e2e_serial, "serial_ms_per_step": e2e_serial_ms / K},
        "roofline": {"bound": "hbm", "kernel": dom_kernel, "achieved": dom_gbs, "peak": hbm_peak,
                     "unit": "GB/s", "frac": dom_gbs / hbm_peak, "traffic": traffic,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                     else "fallback 6.65 TB/s (B200_PROFILING.md)",
                     "bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
                     "whole_matvec_frac": (mv_bytes / (ms_max / K * 1e-3) / 1e9) / hbm_peak,
                     "read_only_ceiling_gbs": read_bw.value,
                     "frac_of_read_only_ceiling": dom_gbs / read_bw.value,
                     "vs_8TBps": (mv_bytes / (ms_max / K * 1e-3) / 1e9) / 8000.0},
        "matvec_phases": ({"gather_ms": ph[0] / nc, "fused_vhx_row_gemv_ms": p1_ms, "fused_GBps": dom_gbs,
                           "finalize_ms": ph[3] / nc, "bytes": mv_bytes} if fused else
                          {"gather_ms": ph[0] / nc, "vhx_ms": p1_ms,
                           "vhx_GBps": st["phase1_bytes"] / (p1_ms * 1e-3) / 1e9, "row_gemv_ms": p2_ms,
                           "row_gemv_GBps": dom_gbs, "finalize_ms": ph[3] / nc, "bytes": mv_bytes}),
        "assembly": {"ms": st["t_total_ms"], "wall_s": t_asm_wall, "ms_warm": st_warm["t_total_ms"],
                     "wall_s_warm": t_asm_wall_warm,
                     "note": "ms = first assembly in the process (empty allocator cache, cold host vectors, "
                             "clocks ramping); ms_warm = a second assembly of the same problem (steady state)",
                     "tree_build_s": t_tree,
                     "aca_ms": st["t_aca_ms"], "recompress_ms": st["t_recompress_ms"],
                     "dense_ms": st["t_dense_ms"], "form_ms": st["t_form_ms"],
                     "green_entries_per_s": entries / t_asm,
                     "green_entries_per_s_warm": entries / t_asm_warm, "pairs": st["pairs_evaluated"],
                     "fp64_peak_tflops": dfma.value,
                     "fp64_peak_source": "measured DFMA microkernel (hmx_bench_dfma)",
                     # executed flops: what this implementation computes (Gram-based recompression)
                     "fp64_flops": asm_flops, "fp64_tflops": asm_flops / t_asm / 1e12,
                     "fp64_frac": asm_flops / t_asm / 1e12 / dfma.value,
                     "fp64_frac_warm": asm_flops / t_asm_warm / 1e12 / dfma.value,
                     "fp64_tflops_warm": asm_flops / t_asm_warm / 1e12,
                     # against the nominal 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (the probe varies 27-33 TF/s per box)
                     "fp64_nominal_tflops": 37.2, "fp64_frac_warm_nominal": asm_flops / t_asm_warm / 1e12 / 37.2,
                     # SURVEY.md 8(d) work model: flops of the reference algorithm (two panel QRs + SVD)
                     "survey_model": {"fp64_flops": sv_flops, "parts": sv_parts,
                                      "fp64_tflops_warm": sv_flops / t_asm_warm / 1e12,
                                      "fp64_frac_warm": sv_flops / t_asm_warm / 1e12 / dfma.value,
                                      "fp64_frac": sv_flops / t_asm / 1e12 / dfma.value},
                     "max_rank_before": rep.max_rank_before, "max_rank_after": rep.max_rank_after,
                     "tau": rep.tau, "aca_passes": st["aca_passes"]},
        "clocks": clocks,
    }
    if not args.no_estimate:
        # delta_{H,F} estimator: every leaf regenerated on the device
        from paper_1706_09384_b200.hmatrix import block_errors

        ra = H.block_info()["rank_after"].astype(np.float64)
        tb = np.asarray(bt.leaf_table)
        mn = ((tb[:, 2] - tb[:, 1]) * (tb[:, 4] - tb[:, 3])).astype(np.float64)
        est_flops = float(np.sum(mn * (8.0 * w.d * w.d * ra + PAIR_FLOPS[w.kind])))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        err2, norm2 = block_errors(H, spec, cloud)
        t_est = time.perf_counter() - t0
        adm = tb[:, 0] == 1
        ratio = np.sqrt(err2[adm] / norm2[adm]) / w.eps
        line["estimator"] = {"wall_s": t_est, "pairs": float(mn.sum()), "fp64_flops": est_flops,
                             "fp64_tflops": est_flops / t_est / 1e12,
                             "fp64_frac": est_flops / t_est / 1e12 / dfma.value,
                             "delta_h_frob_rel": float(np.sqrt(err2.sum() / norm2.sum())),
                             "worst_leaf_eps": float(ratio.max()), "leaves_above_eps": int((ratio > 1).sum()),
                             "leaves_above_3eps": int((ratio > 3).sum())}
    if args.extra_configs:
        del H
        if reserve_s is None:
            L.hmx_ctx_release_cache(_lib.context(local))
        line["other_configs"] = {}
        for tag in [t for t in args.extra_configs.split(",") if t]:
            line["other_configs"][tag] = config_summary(tag, local, dfma.value)
            if reserve_s is None:
                L.hmx_ctx_release_cache(_lib.context(local))
        H = None
    if not args.no_solve:
        # its own job: the U32k H-matrix and the cached workspaces are handed back first
        del H
        import gc

        gc.collect()
        if reserve_s is None:
            L.hmx_ctx_release_cache(_lib.context(local))
        del Xd, Y
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        line["time_to_solve"] = time_to_solve(args.solve_config, local)
    if not args.no_direct:
        import gc

        H = None
        gc.collect()
        L.hmx_ctx_release_cache(_lib.context(local))  # the reserved region goes back: the H-LU engine has its own pool
        try:
            line["direct_solve"] = {t: direct_solve(t, local, cpu=(rank == 0 and ws == 1))
                                    for t in args.direct_config.split(",") if t}
        except Exception as exc:  # reported, never fatal for the headline line
            line["direct_solve"] = {"failed": repr(exc)}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            r = run_cpu(args.config, steps=5, warmup=1)
            line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                      "same_config", "ms_per_step", "ms_per_step_median",
                                                      "max_rank_after", "assembly")}
            line["cpu_baseline"]["end_to_end_H4k"] = cpu_end_to_end("H4k")
        except Exception as exc:  # the baseline is reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {exc!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------------------------
def shard_arm(args):
    """Row-sharded U32k H-matvec (strong scaling; the N > 1 default).  Rank p
    assembles the leaves of its owned row range (no collective); a step is the
    sharded matvec: local matvec + one NCCL all-gather of the owned y segments
    (d N complex128 in total).  value = full-H algorithmic bytes x K / device
    time (max over ranks)."""
    import torch

    import paper_1706_09384_b200 as hmx
    from paper_1706_09384_b200 import shard
    from paper_1706_09384_b200.configs import WORKLOADS
    from paper_1706_09384_b200.dist import max_over_ranks

    ws, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = WORKLOADS[args.config]
    cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
    ct = hmx.build_cluster_tree(cloud, w.n_leaf)
    bt = hmx.build_block_tree(ct, ct, w.eta)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh = shard.assemble_sharded(w.spec(), cloud, ct, bt, hmx.ACAConfig(eps_aca=w.eps), rank, ws, device=local)
    torch.cuda.synchronize()
    t_asm = max_over_ranks(time.perf_counter() - t0, f"cuda:{local}")
    st = sh.local.stats() if sh.local is not None else {"matvec_bytes": 0.0, "phase2_bytes": 0.0}
    # full-H algorithmic bytes: the stripes' leaf bytes sum to the full H's, x / y counted once
    n = w.d * w.n_points
    leaf_b = torch.tensor([float(st["matvec_bytes"]) - 32.0 * n if sh.local is not None else 0.0],
                          dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        tdist.all_reduce(leaf_b)
    mv_bytes = float(leaf_b.item()) + 32.0 * n
    K, W = args.steps, args.warmup
    rng = np.random.default_rng(SEED)
    X = torch.from_numpy(np.stack([rng.standard_normal(n) + 1j * rng.standard_normal(n) for _ in range(K + W)]))
    Xd = X.to(f"cuda:{local}")
    for j in range(W):
        sh.matvec(Xd[K + j])
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_1706_09384_b200 import _lib

    L = _lib.lib()
    if sh.local is not None:
        _lib.check(L.hmx_profile_begin(sh.local.handle), "profile")
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for j in range(K):
            sh.matvec(Xd[j])
        e1.record()
        torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), f"cuda:{local}")
    # roofline of the dominant kernel (this rank's row GEMV), the slowest rank's rate
    ph = np.zeros(4)
    ncalls = C.c_int64()
    if sh.local is not None:
        _lib.check(L.hmx_profile_end(sh.local.handle, C.byref(ncalls), _lib.ptr(ph)), "profile")
    p2_ms = ph[2] / max(int(ncalls.value), 1)
    p2_gbs = st["phase2_bytes"] / (p2_ms * 1e-3) / 1e9 if p2_ms > 0 else 0.0
    p2_gbs = -max_over_ranks(-p2_gbs, f"cuda:{local}")  # min over ranks
    peaks, peak_kind = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    # e2e: pinned host x -> device, sharded matvec, y -> pinned host, every step
    Xh = X.pin_memory()
    Yh = torch.empty(n, dtype=torch.complex128).pin_memory()
    if ws > 1:
        tdist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    f0.record()
    for j in range(K):
        y = sh.matvec(Xh[j].to(f"cuda:{local}", non_blocking=True))
        Yh.copy_(y, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), f"cuda:{local}")
    line = {
        "metric": f"{args.config} H-matvec algorithmic HBM throughput (elasto U), row-sharded",
        "value": mv_bytes * K / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (Fibonacci sphere, seeded complex Gaussian x, seed 0)",
        "config": {"workload": f"{args.config} H-matvec", "kernel": "elasto U", "n_points": w.n_points,
                   "n_leaf": w.n_leaf, "eta": w.eta, "eps_aca": w.eps, "ks": w.ks,
                   "parallelism": f"row-range shards x{ws} (one all-gather of y per matvec)",
                   "l2": "inputs larger than L2, no flush"},
        "gpu_launches": 4 * K,
        "e2e": {"value": mv_bytes * K / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 16 * n, "ms_per_step": e2e_ms / K},
        "roofline": {"bound": "hbm", "kernel": "mv_phase2", "achieved": p2_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": p2_gbs / hbm_peak, "traffic": None,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                     else "fallback 6.65 TB/s (B200_PROFILING.md)",
                     "note": "per-rank row-GEMV rate, slowest rank"},
        "assembly": {"wall_s_max_over_ranks": t_asm, "leaves_this_rank": int(len(sh.part_idx)),
                     "row_bounds": [int(v) for v in sh.bounds]},
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def relaunch_under_torchrun(args):
    """``python bench.py --gpus N`` (N > 1) outside torchrun: re-run this command as N ranks, one per
    GPU, through torch.distributed.run on 127.0.0.1 (the NCCL INIT lines go to stderr)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl != "reference" and a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(a))
    if a.impl == "reference":
        reference_arm(a)
    elif a.shard or (world > 1 and not a.replicas):
        shard_arm(a)
    else:
        hmx_arm(a)
