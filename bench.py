"""Benchmark: HODLR-multifrontal factorization + preconditioned GMRES solve.

One step = ``mf_factorize`` (numeric, accelerated mode) + ``gmres`` (restart
30, tol 1e-10) of BASELINE.json's configs[1] (C2): 3D 7-point Poisson 48^3,
N = 110,592, HODLR leaf 64, eps 1e-5, RHS N(0,1) seed 0. The free BDLR
parameters are fixed as SURVEY.md 6.5 / BASELINE.md 3b recommend so that the
REFERENCE converges: d = 1, n_c = 1024 (the reference default n_c = 256 stalls
at 4,000 iterations). The symbolic analysis (ND + etree, host) is done once
outside the timed region and reported separately.

Arms:
  default             this framework (libmfh.so, sm_100a)
  --impl reference    the reference algorithm on the host cores (the CPU
                      oracle restatement; the Python reference cannot travel
                      to the GPU box), timed on the full workload (1 core)

Multi-GPU (torchrun, N > 1): the factorization is sharded by nested-dissection
subtree: each rank factors the subtrees and top fronts it owns;
cut-child updates travel point to point to the parent's owner in compressed
form (NCCL send/recv), preconditioner contributions and solution pieces cross
ranks through NCCL all-reduces on the library stream, and GMRES is distributed
(rank-local Krylov vectors, halo SpMV, CGS2 with all-reduced dot products).
Strong scaling: one system per job, value is the max-over-ranks step time.
"""

from __future__ import annotations

import os

# The reference algorithm's many tiny BLAS calls are 5-15x slower with more
# than one BLAS thread; the CPU legs run single-threaded. Must be
# set before numpy loads OpenBLAS.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse
import json
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, nd_leaf, params, restart, tol, rhs)
    "c2": dict(desc="3D Poisson 7-pt 48^3 (BASELINE configs[1])", gen=("poisson7", (48, 48, 48)), leaf=64,
               params=dict(n_c=1024, eps=1e-5, d=1, n_leaf=64), restart=30, tol=1e-10, rhs="normal"),
    "c1": dict(desc="2D Q1 128^2 (BASELINE configs[0])", gen=("q1_2d", (128,)), leaf=64,
               params=dict(n_c=256, eps=1e-6, d=1, n_leaf=32), restart=30, tol=1e-10, rhs="uniform"),
    "c2_nc256": dict(desc="3D Poisson 48^3, reference defaults d=1 n_c=256", gen=("poisson7", (48, 48, 48)),
                     leaf=64, params=dict(n_c=256, eps=1e-5, d=1, n_leaf=64), restart=30, tol=1e-10,
                     rhs="normal"),
    "t8": dict(desc="3D Poisson 8^3 (tests of the bench arms)", gen=("poisson7", (8, 8, 8)), leaf=16,
               params=dict(n_c=64, eps=1e-5, d=1, n_leaf=16), restart=30, tol=1e-10, rhs="normal"),
    "p32": dict(desc="3D Poisson 32^3 (C2 params)", gen=("poisson7", (32, 32, 32)), leaf=64,
                params=dict(n_c=256, eps=1e-5, d=1, n_leaf=64), restart=30, tol=1e-10, rhs="normal"),
    # larger BASELINE configs (parity at these sizes is through the size-independent
    # properties in tests/; the oracle does not finish them in bench time). C3's
    # (n_c, d) were chosen on the GPU so that GMRES converges (n_c 1024/2048 with
    # d 1 stall like C2 at the reference defaults; n_c 4096, d 2: 17 iterations)
    "c3": dict(desc="3D Q1 hex 64^3, log-normal kappa seed 0 (BASELINE configs[2])", gen=("hex_q1", (64,)),
               leaf=64, params=dict(n_c=4096, eps=1e-4, d=2, n_leaf=64), restart=50, tol=1e-10, rhs="uniform"),
    "c4": dict(desc="2D P1 Delaunay 1000^2 jittered lattice seed 0 (BASELINE configs[3])",
               gen=("p1_delaunay", (1000,)), leaf=64, params=dict(n_c=1024, eps=1e-5, d=1, n_leaf=64), restart=30,
               tol=1e-10, rhs="normal"),
    # C5: one factorization and 8 GMRES solves per step (8 RHS N(0,1), seeds 0..7);
    # (n_c, d) = (12288, 2): 23 iterations per solve, the fastest step of the
    # GPU sweep in BASELINE.md (n_c 2048..16384, d 1..3)
    "c5": dict(desc="3D Poisson 7-pt 128^3 (BASELINE configs[4]), 8 RHS", gen=("poisson7", (128, 128, 128)),
               leaf=64, params=dict(n_c=12288, eps=1e-4, d=2, n_leaf=64), restart=50, tol=1e-10, rhs="normal",
               nrhs=8),
}
METRIC = "factor+GMRES solve time (s) at N; HODLR front GFLOP/s & % of FP64/HBM roofline"


def make_problem(cfg):
    from paper_1410_2697_b200 import problems as PR
    kind, args = cfg["gen"]
    A, _ = {"poisson7": PR.gen_poisson7, "q1_2d": PR.gen_q1_2d, "hex_q1": PR.gen_hex_q1,
            "p1_delaunay": PR.gen_p1_delaunay}[kind](*args)
    b = PR.seeded_rhs(A.n_rows, 0, cfg["rhs"])
    return A, b


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def fp64_peak_tflops():
    """cuBLAS DGEMM throughput measured live (4096^3, best of 5, CUDA events):
    the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 figure)."""
    import torch
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    best = float("inf")
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * n ** 3 / best / 1e12


def phase_rooflines(tim, hbm, fp64, apply_ms, apply_bytes, spmv_ms, nnz, n):
    """Per-phase achieved throughput against the binding roofline, with the
    algorithmic counts of the REFERENCE's algorithm on this factor's structure
    (counted by the engine: mfh_timing_t):
      sample        16 B per sampled entry (write + source read), HBM; plus the
                    2 r flops per entry and low-rank child term W V^T it meets
      pivot_lu      8 B per trailing-entry visit (nominal: the cores live in
                    shared memory, see traffic); latency model = the longest
                    core's steps summed over structured heights, us per step
    The FP64 phases (skeleton, hodlr_factor, eliminate, hodlr_front,
    dense_front) report the flops this engine EXECUTED (GEMMs 2mnk, register
    inverses 2n^3; mfh_timing_t.exec_flops_*) as achieved / frac, and the
    reference algorithm's count beside it (ref_amount, ref_tflops): the
    explicit-inverse form does more work than the reference's HODLR solves in
    a14 and less in a16 (where the reference re-solves with an identity).
      skeleton      ref: r^2 (m + n) flops per low-rank block (the two TRSMs)
      hodlr_factor  ref a14: sum_leaves (2/3) n^3 + sum_nodes [2 r1 S(L) + 2 r2 S(R)
                    + 2 r1 r2 n + (2/3)(r1 + r2)^3]  (hodlr.py:298-357)
      eliminate     ref a16: 2 r_pf S_pp + 2 r_fp n_p r_pf + 2 nf r_fp r_pf
      hodlr_front   a14 + a16 over both phases' time: BASELINE's "HODLR front GFLOP/s"
      dense_front   ref a5: (2/3) n_p^3 + 2 n_p^2 nf + 2 n_p nf^2
      materialize   executed flops of writing child updates out as dense blocks (no reference
                    count: the reference samples them entry by entry)
      apply         8 sum(2 S_pp + S_pf + S_fp) + 32 N (the engine's own read
                    bytes beside it)
      spmv          12 nnz + 4 (N + 1) + 16 N
    FP64 peak: cuBLAS DGEMM measured live; HBM: MEASURED_PEAKS.json."""
    out = {}

    def put(name, amount, ms, unit, peak, **extra):
        if ms <= 0:
            return
        ach = amount / (ms * 1e-3) / (1e9 if unit == "GB/s" else 1e12)
        out[name] = {"achieved": ach, "unit": unit, "peak": peak, "frac": ach / peak, "ms": ms,
                     "amount": amount, **extra}

    put("sample", 16.0 * tim["sample_entries"], tim["sample_ms"], "GB/s", hbm,
        lr_tflops=tim["sample_lr_flops"] / (tim["sample_ms"] * 1e-3) / 1e12 if tim["sample_ms"] > 0 else None)
    steps = tim["pivot_lu_crit_steps"]
    put("pivot_lu", 8.0 * tim["pivot_lu_visits"], tim["pivot_lu_ms"], "GB/s", hbm,
        latency={"critical_steps": steps, "us_per_step": tim["pivot_lu_ms"] * 1e3 / steps if steps else None,
                 "note": "sequential complete-pivot steps (argmax -> barrier -> pivot broadcast) bound this "
                         "phase; the cores stay in shared memory (profiles/r2_traffic_c2.json)"})
    def fp(name, exec_fl, ref_fl, ms):
        if ms <= 0:
            return
        put(name, exec_fl, ms, "TFLOP/s", fp64, ref_amount=ref_fl, ref_tflops=ref_fl / (ms * 1e-3) / 1e12)

    ex = {k: tim.get("exec_flops_" + k, 0.0) for k in ("skeleton", "hodlr", "elim", "dense")}
    fp("skeleton", ex["skeleton"], tim["skeleton_flops"], tim["skeleton_ms"])
    fp("hodlr_factor", ex["hodlr"], tim["hodlr_flops"], tim["hodlr_factor_ms"])
    fp("eliminate", ex["elim"], tim["elim_flops"], tim["eliminate_ms"])
    fp("hodlr_front", ex["hodlr"] + ex["elim"], tim["hodlr_flops"] + tim["elim_flops"],
       tim["hodlr_factor_ms"] + tim["eliminate_ms"])
    if "hodlr_front" in out:
        out["hodlr_front"]["gflops"] = out["hodlr_front"]["achieved"] * 1e3
        out["hodlr_front"]["ref_gflops"] = out["hodlr_front"]["ref_tflops"] * 1e3
    fp("dense_front", ex["dense"], tim["dense_flops"], tim["dense_front_ms"])
    # child updates written out as dense blocks for their parents' sampling (part of a7's work
    # in this engine; the reference samples the HODLR / low-rank form entry by entry instead)
    if tim.get("materialize_ms", 0.0) > 0:
        put("materialize", tim.get("exec_flops_materialize", 0.0), tim["materialize_ms"], "TFLOP/s", fp64,
            note="extend-add: child updates materialized before the parent's height samples them")
    put("apply", tim["apply_ref_bytes"], apply_ms, "GB/s", hbm, engine_bytes=apply_bytes,
        engine_gbs=apply_bytes / (apply_ms * 1e-3) / 1e9 if apply_ms > 0 else None)
    put("spmv", 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n, spmv_ms, "GB/s", hbm)
    fac = [out[k] for k in ("sample", "pivot_lu", "skeleton", "hodlr_factor", "eliminate", "dense_front",
                            "materialize") if k in out]
    tot = sum(v["ms"] for v in fac)
    out["factor_weighted_frac"] = sum(v["frac"] * v["ms"] for v in fac) / tot if tot else None
    out["factor_covered_ms"] = tot
    out["fp64_peak_kind"] = "cuBLAS DGEMM 4096^3 measured live"
    return out


def traffic_record(config):
    """DRAM traffic per kernel class from the committed ncu capture of this
    config's step (profiles/r2_traffic_<config>.json, scripts/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"r2_traffic_{config}.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process
    through NVML (spawning nvidia-smi every 200 ms perturbs the sync-heavy GMRES
    loop by tens of milliseconds). NVML is initialised and the thread started
    before warm-up (first NVML queries are slow and contend with the driver);
    only samples taken while `active` is set (the timed region) are reported.
    MFH_BENCH_NO_CLOCKS=1 disables sampling (diagnostics only)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index=0, period=0.2):
        self.index = index
        self.period = period
        self.samples = []
        self.active = False
        self._stop = threading.Event()
        self._wake = threading.Event()
        self._t = None

    def activate(self, on=True):
        """Enter / leave the timed region; entering wakes the thread so even a
        region shorter than the period gets a sample."""
        self.active = on
        if on:
            self._wake.set()

    def start(self):
        if os.environ.get("MFH_BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            return self

        def run():
            while not self._stop.is_set():
                if self.active:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        if self.active:
                            self.samples.append((sm, mx, rs))
                    except Exception:
                        pass
                self._wake.wait(self.period)
                self._wake.clear()

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        self._wake.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for _, _, rs in self.samples for bit, name in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": float(max(s[1] for s in self.samples)), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MFH_BENCH_EMULATE"):
        # diagnostics on a one-GPU box: every rank on cuda:0, gloo host exchanges
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo" if os.environ.get("MFH_BENCH_EMULATE") else "nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    """Max of a host scalar over ranks (NCCL on the GPU box, gloo in the CPU tests)."""
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle (reference algorithm restated)
# ---------------------------------------------------------------------------

class OracleWorkload:
    """The reference algorithm (CPU oracle restatement) on the bench workload.

    The symbolic analysis is done once (outside the timed step, like the GPU
    arm); one step = the full numeric factorization + the preconditioned GMRES
    solve, single-threaded (OPENBLAS_NUM_THREADS=1: the reference's many tiny
    BLAS calls run 5-15x slower with more BLAS threads).

    Configurations the reference cannot finish in bench time (C3-C5: hours;
    its ordering alone takes 444 s at C5) run a BOUNDED sample instead: the
    post-order prefix of the numeric factorization that fits in
    ``BOUNDED_S`` seconds, on the bit-identical native ordering, scaled to the
    whole factorization by the front_size^2 * max(n_pivot, 1) work proxy
    (the subtree partition's cost model). GMRES is not part of that sample,
    so the value is a lower bound of the reference's factor + solve time.
    """

    BOUNDED = ("c3", "c4", "c5")
    BOUNDED_S = 30.0

    def __init__(self, cfg):
        from oracle import mfh_oracle as O
        self.O = O
        self.cfg = cfg
        self.A, self.b = make_problem(cfg)
        self.bounded = cfg.get("name") in self.BOUNDED
        t0 = time.perf_counter()
        if self.bounded:
            self.et = self._native_tree()
        else:
            ip, ix = O.adjacency(self.A._csc)
            self.et = O.build_elimination_tree(O.nested_dissection(ip, ix, self.A.n_rows, cfg["leaf"]), self.A._csc)
        self.t_symbolic = time.perf_counter() - t0

    def _native_tree(self):
        """The oracle's ETree from the native ND + etree (bit-identical to the
        reference's ordering, tests/test_symbolic.py)."""
        import paper_1410_2697_b200 as P
        t = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(self.A), self.cfg["leaf"]), self.A)
        nn = len(t.nodes)
        return self.O.ETree([t.nodes[v].pivot_ids for v in range(nn)], [t.nodes[v].frontal_ids for v in range(nn)],
                            [list(t.nodes[v].children) for v in range(nn)],
                            [-1 if t.nodes[v].parent is None else t.nodes[v].parent for v in range(nn)],
                            list(t.post_order), np.asarray(t.permutation), t.root)

    def step(self):
        O, cfg, A, b = self.O, self.cfg, self.A, self.b
        if self.bounded:
            t0 = time.perf_counter()
            done = O.factorize_prefix(A._csc, self.et, "accelerated", self.BOUNDED_S, **cfg["params"])
            t = time.perf_counter() - t0
            own = {v: float(len(self.et.pivots[v]) + len(self.et.frontal[v])) ** 2 * max(len(self.et.pivots[v]), 1)
                   for v in self.et.post_order}
            frac = sum(own[v] for v in done) / sum(own.values())
            return dict(t=t / max(frac, 1e-12), t_factor=t / max(frac, 1e-12), t_gmres=0.0, its=None, conv=None,
                        res=None, bounded=True, t_sample=t, frac=frac, fronts=len(done), nfronts=len(own))
        t0 = time.perf_counter()
        F = O.factorize(A._csc, self.et, "accelerated", **cfg["params"])
        t1 = time.perf_counter()
        x, res, its, conv = O.gmres(lambda v: A._csc @ v, b, lambda v: O.solve(F, v), tol=cfg["tol"],
                                    restart=cfg["restart"])
        t2 = time.perf_counter()
        return dict(t=t2 - t0, t_factor=t1 - t0, t_gmres=t2 - t1, its=its, conv=conv, res=res[-1])


def sample_text(r, w):
    if r.get("bounded"):
        return (f"bounded sample on 1 host core (OPENBLAS_NUM_THREADS=1): the post-order prefix of the oracle "
                f"factorization that fits in {w.BOUNDED_S:.0f} s ({r['fronts']} of {r['nfronts']} fronts, "
                f"{100 * r['frac']:.2f}% of the front_size^2*max(n_pivot,1) work proxy) took {r['t_sample']:.1f} s; "
                f"value = that time scaled to the whole factorization; GMRES not sampled (value is a lower bound "
                f"of factor + solve); native bit-identical ordering, symbolic analysis excluded")
    return (f"full workload on 1 host core (OPENBLAS_NUM_THREADS=1): oracle factorization "
            f"{r['t_factor']:.1f} s + GMRES {r['t_gmres']:.1f} s ({r['its']} iterations, converged="
            f"{r['conv']}); symbolic analysis {w.t_symbolic:.1f} s excluded like the GPU arm")


def run_reference_arm(args, cfg, world, rank):
    if rank != 0:
        return
    import multiprocessing
    w = OracleWorkload(cfg)
    # the CPU arm has nothing to warm up beyond imports: one warm-up step is a
    # small instance of the same pipeline, the K timed steps are the full workload
    small = dict(cfg, name="warmup", gen=("poisson7", (8, 8, 8)), params=dict(cfg["params"], n_c=64))
    for _ in range(args.warmup):
        OracleWorkload(small).step()
    steps = [w.step() for _ in range(args.steps)]
    t = float(np.mean([r["t"] for r in steps]))
    line = {
        "impl": "reference", "metric": METRIC, "value": t, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": w.A.n_rows, "nnz": w.A.nnz, **cfg["params"], "nd_leaf": cfg["leaf"],
                   "restart": cfg["restart"], "tol": cfg["tol"], "rhs": f"{cfg['rhs']} seed 0",
                   "parallelism": "single" if args.gpus <= 1 else f"subtree{args.gpus}"},
        "threads": "1 (OPENBLAS_NUM_THREADS=1: more BLAS threads make the reference 5-15x slower, "
                   "SURVEY 6.3 / BASELINE.md 3; rank 0 only, the reference is single-process)",
        "cpu_baseline": {"value": t, "unit": "s", "cores": 1, "kind": "port", "sample": sample_text(steps[-1], w)},
        "e2e": {"value": t, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gmres": {"iterations": steps[-1]["its"], "converged": steps[-1]["conv"]},
        "host_cores_available": multiprocessing.cpu_count(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu_arm(args, cfg, world, rank, local):
    import ctypes as C
    import torch
    import paper_1410_2697_b200 as P
    from paper_1410_2697_b200 import _lib

    os.environ.setdefault("MFH_DEVICE", str(local))
    torch.cuda.set_device(local)
    ctx = _lib.context()
    stream_ptr, _ = ctx.info()
    lib_stream = torch.cuda.ExternalStream(stream_ptr)
    A, b = make_problem(cfg)
    n = A.n_rows
    nrhs = int(cfg.get("nrhs", 1))
    from paper_1410_2697_b200 import problems as PR
    bs = [b] + [PR.seeded_rhs(n, r, cfg["rhs"]) for r in range(1, nrhs)]
    t0 = time.perf_counter()
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), cfg["leaf"]), A)
    t_sym = time.perf_counter() - t0
    params = P.MfParams(**cfg["params"])
    d_bs = [torch.from_numpy(v).cuda() for v in bs]
    d_x = torch.zeros(n, dtype=torch.float64, device="cuda")
    d_B = torch.from_numpy(np.stack(bs)).cuda() if nrhs > 1 else None  # [nrhs][n]
    d_X = torch.zeros((nrhs, n), dtype=torch.float64, device="cuda") if nrhs > 1 else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dev_op = A.device_operator()
    hist = np.empty(4000)

    split = {"factor_s": [], "solve_s": [], "gmres_inner_s": [], "apply_build_s": [], "gmres_sync_s": [],
             "gmres_apply_enqueue_s": []}

    if world > 1:
        from paper_1410_2697_b200.sharded import SubtreePartition, mf_factorize_sharded
        part = SubtreePartition(et, world)

        def factorize():
            return mf_factorize_sharded(A, et, P.ACCELERATED, params, partition=part)
    else:
        mode = P.ACCELERATED if args.mode == "accelerated" else P.CONVENTIONAL

        def factorize():
            return P.mf_factorize(A, et, mode, params)

    def step_device():
        t0 = time.perf_counter()
        F = factorize()
        t1 = time.perf_counter()
        ops = _lib.mfh_gmres_ops()
        ops.A = dev_op.handle
        ops.M = F._h
        nh, its, conv = C.c_int64(), C.c_int64(), C.c_int()
        g_ms, its0, conv0, res0 = 0.0, None, None, None
        if nrhs > 1 and world == 1:  # one factorization, nrhs solves in lockstep (C5: 8)
            cap = 4000
            hh = np.empty((nrhs, cap))
            nhs, itss = np.zeros(nrhs, dtype=np.int64), np.zeros(nrhs, dtype=np.int64)
            convs = np.zeros(nrhs, dtype=np.int32)
            _lib.check(_lib.lib().mfh_gmres_batched_device(
                ctx.handle, C.byref(ops), n, nrhs, C.c_void_p(d_B.data_ptr()), C.c_void_p(d_X.data_ptr()),
                cfg["tol"], cap, cfg["restart"], _lib.ptr(hh), cap, _lib.ptr(nhs), _lib.ptr(itss), _lib.ptr(convs)))
            g_ms = F.timing()["gmres_ms"]
            its0, conv0, res0 = int(itss[0]), bool(convs[0]), hh[0, max(0, nhs[0] - 1)]
        if world > 1:  # distributed GMRES on the sharded factor: rank-local vectors, halo SpMV, CGS2
            from paper_1410_2697_b200.sharded import gmres_sharded
            for bv in bs:
                xs, hs = gmres_sharded(A, bv, F, tol=cfg["tol"], restart=cfg["restart"])
                g_ms += F.timing()["gmres_ms"]
                if its0 is None:
                    its0, conv0, res0 = hs.iterations, hs.converged, hs.residuals[-1]
        for d_b in (d_bs if not (nrhs > 1 and world == 1) and world == 1 else []):  # one solve per right-hand side
            _lib.check(_lib.lib().mfh_gmres_device(ctx.handle, C.byref(ops), n, C.c_void_p(d_b.data_ptr()),
                                                   C.c_void_p(d_x.data_ptr()), cfg["tol"], 4000, cfg["restart"],
                                                   _lib.ptr(hist), C.byref(nh), C.byref(its), C.byref(conv)))
            g_ms += F.timing()["gmres_ms"]
            if its0 is None:
                its0, conv0, res0 = its.value, bool(conv.value), hist[max(0, nh.value - 1)]
        t2 = time.perf_counter()
        ti = F.timing()
        split["factor_s"].append(t1 - t0)
        split["solve_s"].append(t2 - t1)
        split["gmres_inner_s"].append(g_ms / 1e3)
        split["apply_build_s"].append((ti["apply_build_ms"] + ti["apply_instantiate_ms"]) / 1e3)
        split["gmres_sync_s"].append(ti["gmres_sync_ms"] / 1e3)
        split["gmres_apply_enqueue_s"].append(ti["gmres_apply_ms"] / 1e3)
        return F, its0, conv0, res0

    def step_e2e():  # public API, host b -> host x (every RHS)
        F = factorize()
        if world > 1:
            from paper_1410_2697_b200.sharded import gmres_sharded
            out = [gmres_sharded(A, v, F, tol=cfg["tol"], restart=cfg["restart"]) for v in bs]
            return F, out[0][0], out[0][1]
        M = P.mf_preconditioner(F)
        if nrhs > 1 and world == 1:
            X, hs = P.gmres_batched(A, np.stack(bs, axis=1), M, tol=cfg["tol"], restart=cfg["restart"])
            return F, X[:, 0], hs[0]
        out = [P.gmres(A, v, M=M, tol=cfg["tol"], restart=cfg["restart"]) for v in bs]
        return F, out[0][0], out[0][1]

    if args.profile:  # exactly one factorization + solve, for ncu launch lists
        F, its, conv, res = step_device()
        torch.cuda.synchronize()
        print(json.dumps({"profile_step": True, "iterations": its, "converged": conv}), flush=True)
        return
    clocks = ClockSampler(local).start()
    cold_s = None
    for w in range(args.warmup):
        F = None  # release the previous factorization first (C5's factor is tens of GB)
        F, its, conv, res = step_device()
        if w == 0:  # first call on this tree: symbolic caches, maps and patterns built inside it
            cold_s = split["factor_s"][0]
    barrier(world)
    times, e2e_times = [], []
    launches0 = ctx.info()[1]
    clocks.activate(True)
    if True:
        for _ in range(args.steps):
            F = None  # the previous factorization is released before the next step
            flush.fill_(1)
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lib_stream)
            F, its, conv, res = step_device()
            e1.record(lib_stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        launches = (ctx.info()[1] - launches0) / max(1, args.steps)
        per_step = {k: [round(x, 5) for x in v[-args.steps:]] for k, v in split.items()
                    if k in ("factor_s", "gmres_inner_s")}
        split = {k: float(np.mean(v[-args.steps:])) for k, v in split.items()}
        # everything read from the timed factor, then it is released before the
        # e2e steps (at C5 two factorizations do not fit in HBM together)
        tim = F.timing()
        apply_ms, apply_bytes = F.apply_bench(20)
        spmv_ms = C.c_double()
        _lib.check(_lib.lib().mfh_spmv_bench(dev_op.handle, 50, C.byref(spmv_ms)))
        spmv_ms = spmv_ms.value
        st = F.stats
        fstats = {"structured_fronts": st.structured_fronts, "dense_fronts": st.dense_fronts,
                  "peak_stored_reals": st.peak_stored_reals, "device_bytes": st.device_bytes}
        F = st = None
        import gc
        gc.collect()
        Fe = None
        for _ in range(max(1, min(args.steps, 3))):
            Fe = None  # the previous factorization is released before the next step
            flush.fill_(1)
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lib_stream)
            Fe, xe, he = step_e2e()
            e1.record(lib_stream)
            torch.cuda.synchronize()
            e2e_times.append(e0.elapsed_time(e1) / 1e3)
    clocks.activate(False)
    clocks.stop()
    t_step = max_over_ranks(float(np.mean(times)), world)
    t_e2e = max_over_ranks(float(np.mean(e2e_times)), world)
    true_res = float(np.linalg.norm(A._csc @ xe - b) / np.linalg.norm(b))
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    # dominant kernel: complete-pivot LU (k_full_pivot_lu); 8 algorithmic bytes per
    # trailing-entry visit, per launch = per structured height
    plu_ms = tim["pivot_lu_ms"]
    plu_gbs = 8.0 * tim["pivot_lu_visits"] / (plu_ms * 1e-3) / 1e9 if plu_ms > 0 else 0.0
    pr = phase_rooflines(tim, hbm, fp64_peak_tflops(), apply_ms, apply_bytes, spmv_ms, A.nnz, n)
    tr = traffic_record(args.config) if args.mode == "accelerated" else None
    plu_traffic = None
    if tr and "k_plu" in tr:
        plu_traffic = tr["k_plu"]["dram_bytes_per_launch"]
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": n, "nnz": A.nnz, **cfg["params"], "nd_leaf": cfg["leaf"],
                   "restart": cfg["restart"], "tol": cfg["tol"], "rhs": f"{cfg['rhs']} seed 0" if nrhs == 1 else f"{cfg['rhs']} seeds 0..{nrhs - 1} (one factorization, {nrhs} GMRES solves in lockstep sharing each preconditioner apply)",
                   "parallelism": f"subtree{world}" if world > 1 else "single"},
        "l2": "flushed (256 MiB write) before every timed step",
        "mode": args.mode,
        "gmres": {"iterations": its, "converged": conv, "final_rel_residual": float(res),
                  "true_rel_residual_e2e": true_res, "e2e_iterations": he.iterations},
        "split_s": split,
        "per_step_s": {"step": [round(x, 5) for x in times], **per_step},
        "factor": {"device_ms": tim["total_ms"], "host_plan_ms": tim["host_ms"],
                   "host_ms": {k: tim[k] for k in ("host_preamble_ms", "host_select_ms", "host_sync_wait_ms",
                                                   "wall_ms", "apply_build_ms", "apply_instantiate_ms",
                                                   "gmres_ms", "gmres_apply_ms")},
                   "phases_ms": {k: tim[k] for k in ("sample_ms", "pivot_lu_ms", "skeleton_ms",
                                                     "hodlr_factor_ms", "dense_front_ms", "eliminate_ms",
                                                     "materialize_ms", "idle_gap_ms")},
                   **fstats,
                   "symbolic_s": t_sym, "cold_first_factor_s": cold_s},
        "apply": {"ms": apply_ms, "bytes": apply_bytes, "gbs": apply_bytes / (apply_ms * 1e-3) / 1e9,
                  "frac_of_hbm": apply_bytes / (apply_ms * 1e-3) / 1e9 / hbm},
        "phase_roofline": pr,
        "roofline": {"kernel": "k_plu_* (complete-pivot LU, a10)", "bound": "hbm", "achieved": plu_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": plu_gbs / hbm, "traffic": plu_traffic,
                     "peak_kind": pk_kind, "latency": pr.get("pivot_lu", {}).get("latency"),
                     "note": "nominal HBM fraction (8 B per trailing-entry visit, SURVEY 8d); the cores live in "
                             "shared memory, so traffic (ncu DRAM bytes per launch) is far below the "
                             "algorithmic bytes and the binding limit is the per-step latency"},
        "e2e": {"value": t_e2e, "unit": "s",
                "h2d_bytes_per_step": int(8 * n * nrhs + 8 * A.nnz + 4 * A.nnz + 8 * (n + 1)),
                "d2h_bytes_per_step": int(8 * n * nrhs)},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        w = OracleWorkload(cfg)
        r = w.step()
        line["cpu_baseline"] = {"value": r["t"], "unit": "s", "cores": 1, "kind": "port",
                                "sample": sample_text(r, w)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="accelerated", choices=["accelerated", "conventional"],
                    help="conventional = every front dense (the GPU dense multifrontal baseline, "
                         "multifrontal.py:470)")
    ap.add_argument("--profile", action="store_true", help="one untimed step (for ncu)")
    ap.add_argument("--param", action="append", default=[], metavar="KEY=VALUE",
                    help="override an MfParams field of the config (exploration only)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.param:
        cfg["params"] = dict(cfg["params"])
        for kv in args.param:
            k, v = kv.split("=", 1)
            cfg["params"][k] = float(v) if k == "eps" else int(float(v))
    world, rank, local = (1, 0, 0)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, cfg, world, rank)
        return
    world, rank, local = dist_setup(args.gpus)
    run_gpu_arm(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
