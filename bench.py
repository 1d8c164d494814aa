"""Benchmark: IBPM time steps/s on the B200 hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|s4m|c2a|cavity|flapping|c5-N]
                  [--impl ours|reference] [--parallel slab|replicas] [--min-dist-rows R]

N > 1 (torchrun, one process per GPU): the coupled solve runs row-slab distributed over NCCL
(csrc/dist.cu) — one simulation, strong scaling; --parallel replicas runs N independent copies.

A "step" is one Stepper::advance (stepper.hpp:231-356): explicit terms, PCG-diag momentum solve,
SA-PCG coupled solve, projection and invariants, all resident in HBM (device-built operators and
SA hierarchy). Prints ONE JSON line (rank 0). Default workload: S-4M = the north-star case,
impulsively started cylinder at ~4M cells (cylinder_re3000.cfg geometry at h_min 0.001 ->
2040^2, BASELINE.json configs[2]). Alongside: C2 (configs[1], 1042^2) under "c2", the
moving-body case (configs[3]) under "flapping", the synthetic C5 grids 1024^2..8192^2
(configs[4]) under "grid_sweep", and the reference CPU Stepper under "cpu_baseline".

--impl reference runs the reference's own CPU implementation (oracle/_ref/libibmref.so, the
unmodified reference headers) on the same case with all host threads; it never touches the GPU.
Its steps are a bounded sample (at most --ref-warmup / --ref-steps steps, default 1 / 2) so the
run ends within minutes at S-4M, where one reference step takes ~30 s on 16 cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CASES = os.path.join(ROOT, "cases")

WORKLOADS = {
    # name: (cfg, h_min override, dt override, description)
    "c2": ("cylinder_re40", 0.002, 0.001, "Re40 impulsively started cylinder, h_min 0.002 (1042^2, ~1.09M-row lhs2)"),
    # dt 1.25e-4 (CFL 0.125): at SURVEY's dt 2.5e-4 this case blows up in the reference itself (max |q|
    # 0.198 / 3.76 / 1006 at steps 4 / 5 / 6, identical on the device; tools/diag/ref_s4m_growth.py)
    "s4m": ("cylinder_re3000", 0.001, 1.25e-4, "Re3000 impulsively started cylinder, h_min 0.001 (2040^2, "
                                               "4.17M-row lhs2), dt 1.25e-4"),
    "c2a": ("cylinder_re40", 0.0, 0.0, "Re40 cylinder 330^2 (reference cfg)"),
    "cavity": ("cavity", 0.0, 0.0, "lid-driven cavity Re100 128^2, no body"),
    "flapping": ("flapping", 0.0, 0.0, "flapping ellipse 930x654, moving body (lhs2 rebuilt every step)"),
}


def config_of(name: str) -> dict:
    """The `config` object of both arms (identical keys and values, so the lines compare)."""
    cfg, h_min, dt, desc = workload(name)
    return {"workload": name, "case": cfg + ".cfg", "h_min": h_min or None, "dt": dt or None, "desc": desc}


def workload(name: str):
    if name.startswith("c5-"):
        N = int(name[3:])
        h = 30.72 / N
        return ("uniform_cylinder", h, 0.5 * h, f"synthetic uniform cylinder {N}^2")
    return WORKLOADS[name]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for k, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- algorithmic bytes
def spmv_bytes(rows, cols, nnz):
    """12 nnz + 4 (rows+1) + 8 cols + 8 rows."""
    return 12 * nnz + 4 * (rows + 1) + 8 * cols + 8 * rows


def hier_bytes(h) -> tuple[float, dict]:
    """Algorithmic bytes of one solve-2 SA-PCG iteration as the solve applies it.
    B_it2 counts the reference CSR of every operator the reference V-cycle streams (12 B per
    entry, both P_l and P_l^T). With the level-0 transfers through the stencil (csrc/xfer.cuh) the
    solve never streams P_0 / P_0^T: their 24 nnz(P_0) bytes are replaced by the aggregate id per
    fine row (4 n_0), the member lists (4 n_0 + 4 n_1) and t_a (8 n_1). The reference count stays
    in info["b_it2_reference"]."""
    nl, _, nc = h.info()
    L0 = h.level(0)["A"] if nl else h.coarse_A()
    n0, nnz0 = L0.rows(), L0.nnz()
    b = 12 * nnz0 + 92 * n0
    levels = []
    for l in range(nl):
        lv = h.level(l)
        A, P = lv["A"], lv["P"]
        n_l, n_next = A.rows(), P.cols()
        b += 24 * A.nnz() + 24 * P.nnz() + 100 * n_l + 20 * n_next
        levels.append(dict(rows=n_l, nnz_A=A.nnz(), nnz_P=P.nnz()))
    b += 8 * nc * nc + 16 * nc
    applied = b
    xfer = bool(nl) and h.transfers()
    if xfer:
        applied = b - 24 * levels[0]["nnz_P"] + 8 * n0 + 12 * h.level(0)["P"].cols()
    return float(applied), dict(levels=levels, n_c=nc, b_it2_reference=float(b), level0_transfers=xfer)


def load_traffic(workload: str):
    """Measured DRAM bytes per solve-2 iteration from the committed ncu launch list
    (profiles/r01/traffic.json, tools/traffic_per_iteration.py); None if not captured."""
    for rnd in ("r02", "r01"):  # newest capture first
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                d = json.load(f).get(workload)
            if d:
                return d
        except Exception:
            continue
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int):
    import numpy as np

    from paper_1109_3524_b200 import ibm

    cfg, h_min, dt, desc = workload(args.workload)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    slab = world > 1 and args.parallel == "slab"
    if slab:
        # one NCCL communicator over the ranks; the id travels over the host (gloo) group
        import torch
        import torch.distributed as dist
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            # rank 0 logs its communicator init (NCCL_DEBUG=INFO, INIT subsystem) to a file, so the
            # line can show that the communicator really spans `world` ranks
            if "NCCL_DEBUG" not in os.environ:
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT",
                                  NCCL_DEBUG_FILE=os.path.join(ROOT, "gpurun_out", "nccl_rank0.%p.log"))
            idt = torch.frombuffer(bytearray(ibm.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(idt, 0)
        ctx = ibm.Context(local, nranks=world, rank=rank, nccl_id=bytes(idt.numpy().tobytes()))
    else:
        ctx = ibm.Context(local)
    t0 = time.time()
    st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt, ctx=ctx)
    if slab:
        st.distribute(min_dist_rows=args.min_dist_rows)
    setup_s = time.time() - t0
    h = st.hierarchy()
    b_it2, hinfo = hier_bytes(h)
    A = st.op("A")
    b_it1 = 12 * A.nnz() + 108 * st.n_q
    Lm, QT, Q, BN = st.op("L"), st.op("QT"), st.op("Q"), st.op("BN")
    b_fixed = (spmv_bytes(Lm.rows(), Lm.cols(), Lm.nnz()) + 2 * spmv_bytes(QT.rows(), QT.cols(), QT.nnz())
               + spmv_bytes(Q.rows(), Q.cols(), Q.nnz()) + spmv_bytes(BN.rows(), BN.cols(), BN.nnz())
               + 48 * st.n_q)

    for _ in range(args.warmup):
        r = st.advance()
        if not r.ok:
            raise RuntimeError(r.message)
    launches0 = ctx.launches()
    reps = []
    solve2_ms = []
    # Timed region: K steps. Device time per step from CUDA events on the context stream (inputs
    # resident in HBM); end-to-end time per step = wall clock around the public C-ABI calls a user
    # makes (advance: body kinematics H2D + report D2H; forces; f~ D2H), same steps.
    dev_ms = 0.0
    e2e_s = 0.0
    with ClockSampler(local) as clk:
        ctx.sync()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        for _ in range(args.steps):
            t1 = time.perf_counter()
            ctx.timer_start()
            r = st.advance()
            dev_ms += ctx.timer_stop()
            if not r.ok:
                raise RuntimeError(r.message)
            st.forces()
            if st.n_b:
                _ = st.get("f_tilde")  # 2 n_b force entries
            e2e_s += time.perf_counter() - t1
            reps.append(r)
            solve2_ms.append(st.phase_ms()["solve2"])
        ctx.sync()
        if world > 1:
            dist.barrier()
        launches = ctx.launches() - launches0
    clocks = clk.summary()

    K = args.steps
    its2 = [r.solve2_iters for r in reps]
    its1 = [r.solve1_iters for r in reps]
    steps_per_s = K / (dev_ms * 1e-3)
    # dominant launch: the solve-2 SA-PCG graph (89-99% of the step); algorithmic bytes per launch
    s2_ms = sum(solve2_ms) / K
    s2_bytes = sum(its2) / K * b_it2 + spmv_bytes(st.n_lambda, st.n_lambda, st.nnz_lhs2)
    peak, peak_kind = load_peaks()
    tr = load_traffic(args.workload)
    achieved = s2_bytes / (s2_ms * 1e-3) / 1e9
    b_step = sum(its1) / K * b_it1 + sum(its2) / K * b_it2 + b_fixed
    n_b = st.n_b
    h2d = 5 * 8 * n_b  # body x, y, ds, u_B (2 n_b)
    d2h = 8 * 2 * n_b + 32 + 40 + 2 * 96  # f~, forces, step report, 2 PCG states
    out = {
        "metric": "time steps/sec (IBPM step: explicit + PCG-diag + SA-PCG + projection)",
        "value": round(steps_per_s * (1 if slab else world), 4),
        "unit": "steps/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(dev_ms / K, 4),
        "higher_is_better": True,
        "scaling": "strong" if slab else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (deterministic case file; no datasets)",
        "config": config_of(args.workload),
        "parallelism": (f"row-slab x{world} (solve 2 distributed over NCCL, min_dist_rows "
                        f"{args.min_dist_rows}; explicit terms + solve 1 replicated)") if slab else
                       ("replicas" if world > 1 else "single-gpu"),
        "l2": "inputs larger than L2 (per-iteration working set >> 126 MB)" if b_it2 > 5e8 else
              "working set partly L2-resident",
        "problem": {"grid": [st.nx, st.ny], "n_lambda": st.n_lambda, "nnz_lhs2": st.nnz_lhs2, "n_b": n_b,
                    "sa_levels": len(hinfo["levels"]), "n_c": hinfo["n_c"]},
        "cg_iters_per_step": round(sum(its2) / K, 2),
        "momentum_iters_per_step": round(sum(its1) / K, 2),
        "cg_iters_per_s": round(sum(its2) / (sum(solve2_ms) * 1e-3), 1),
        "cg_iteration_ms": round(s2_ms / max(sum(its2) / K, 1), 4),
        "setup_s": round(setup_s, 3),
        "step_hbm_gbs": round(b_step / (dev_ms / K * 1e-3) / 1e9, 1),
        "roofline": {"kernel": "solve-2 SA-PCG graph launch (SpMV + V-cycle + fused reductions)",
                     "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "frac_of_8tbs": round(achieved / 8000, 4),
                     "bytes_per_launch": s2_bytes, "b_it2": b_it2, "b_it2_reference": hinfo["b_it2_reference"],
                     "bytes_definition": ("SURVEY 8(d) B_it2 as applied: level-0 P/P^T applied through the stencil "
                                          "(not streamed) when level0_transfers"),
                     "level0_transfers": hinfo["level0_transfers"],
                     "traffic": (round(sum(its2) / K * tr["dram_bytes_per_iteration"]) if tr else None),
                     "traffic_per_iteration": tr["dram_bytes_per_iteration"] if tr else None,
                     "traffic_source": tr["source"] if tr else None},
        "e2e": {"value": round(K / e2e_s * (1 if slab else world), 4), "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if slab and rank == 0:
        out["comm"] = nccl_init_record(world)
    return out, st


def nccl_init_record(world: int) -> dict:
    """Rank 0's NCCL init log (bench.py sets NCCL_DEBUG=INFO/INIT with a per-process file): the
    communicator size NCCL reported, so the line shows whether it really spans all ranks."""
    import re
    path = os.path.join(ROOT, "gpurun_out", "nccl_rank0.%d.log" % os.getpid())
    rec = {"backend": "nccl", "log": os.path.relpath(path, ROOT), "nranks_logged": None, "nranks_ok": None}
    try:
        txt = open(path).read()
    except OSError:
        return rec
    n = [int(m) for m in re.findall(r"ncclCommInitRank comm \S+ rank \d+ nranks (\d+)", txt)]
    if n:
        rec["nranks_logged"] = n[-1]
        rec["nranks_ok"] = n[-1] == world
    m = re.search(r"NCCL version (\S+)", txt)
    if m:
        rec["version"] = m.group(1)
    return rec


def case_probe(args, name: str) -> dict:
    """Steps/s and the per-CG-iteration roofline of another cylinder workload (device-timed phases)."""
    from paper_1109_3524_b200 import ibm
    cfg, h_min, dt, desc = WORKLOADS[name]
    t0 = time.time()
    st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt)
    setup = time.time() - t0
    b_it2, hinfo = hier_bytes(st.hierarchy())
    for _ in range(3):
        st.advance()
    ms, its = [], []
    step_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        r = st.advance()
        ph = st.phase_ms()
        ms.append(ph["solve2"])
        step_ms.append(sum(ph.values()))  # device-timed phases of the whole step
        its.append(r.solve2_iters)
    peak, kind = load_peaks()
    it_ms = sum(ms) / sum(its)
    ach = b_it2 / (it_ms * 1e-3) / 1e9
    return {"config": config_of(name), "grid": [st.nx, st.ny], "n_lambda": st.n_lambda, "setup_s": round(setup, 2),
            "cg_iters_per_step": sum(its) / len(its), "cg_iteration_ms": round(it_ms, 4),
            "b_it2_gb": round(b_it2 / 1e9, 3), "achieved_gbs": round(ach, 1), "frac_measured": round(ach / peak, 4),
            "frac_of_8tbs": round(ach / 8000, 4), "steps_per_s": round(1e3 / (sum(step_ms) / len(step_ms)), 3),
            "sa_levels": len(hinfo["levels"]), "n_c": hinfo["n_c"]}


def flapping_probe(args) -> dict:
    """The moving-body probe in its own process, as the reference's own runner would run the case.
    In the bench process, after the S-4M and C2 runs, it still swings (30-104 steps/s on one build;
    fresh processes 100-104), with the operator pipeline's waits growing; see DESIGN.md (d)."""
    import subprocess
    code = ("import json, sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench.flapping_probe_inproc(None)))" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError("flapping probe failed: " + r.stderr[-500:])
    out = json.loads(lines[-1])
    out["process"] = "separate"
    return out


def flapping_probe_inproc(args) -> dict:
    """Moving body (BASELINE configs[3]): E, H, Q, Q^T, lhs2 rebuilt every step and the SA hierarchy
    every n_pc steps, all on the device. Wall clock around whole Stepper.advance calls."""
    from paper_1109_3524_b200 import ibm
    cfg, h_min, dt, _ = WORKLOADS["flapping"]
    st = ibm.Stepper(os.path.join(CASES, cfg + ".cfg"), h_min=h_min, dt=dt)
    # steady state: the operator pipeline's workers start cold (empty aggregate caches, first
    # rebuilds mapping fresh pool memory), so the first steps are not timed
    for _ in range(6):
        st.advance()
    st.ctx.sync()
    n = 40
    t0 = time.perf_counter()
    reps = [st.advance() for _ in range(n)]
    st.ctx.sync()
    wall = time.perf_counter() - t0
    return {"case": cfg + ".cfg", "grid": [st.nx, st.ny], "n_lambda": st.n_lambda, "steps": n,
            "steps_per_s": round(n / wall, 3),
            "operator_rebuild_ms_per_step": round(1e3 * sum(r.t_assembly for r in reps) / n, 3),
            "hierarchy_rebuild_ms_per_step": round(1e3 * sum(r.t_precond for r in reps) / n, 3),
            "hierarchy_rebuilds": sum(r.rebuilt_hierarchy for r in reps),
            "cg_iters_per_step": sum(r.solve2_iters for r in reps) / n}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_phase_seconds(reports) -> dict:
    """The reference's own per-phase timing (StepReport, stepper.hpp:139-144; runner.hpp:18-42)."""
    keys = ("t_assembly", "t_precond", "t_explicit", "t_solve1", "t_solve2", "t_projection")
    return {k[2:]: round(sum(r[k] for r in reports) / len(reports), 4) for k in keys}


def cpu_baseline(args) -> dict:
    """Reference CPU path (oracle/_ref) on a bounded sample of the same workload (rank 0 only):
    --cpu-steps timed steps after one warm-up step, all host threads."""
    from oracle import oracle as O
    cfg, h_min, dt, _ = workload(args.workload)
    R = O.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    t0 = time.time()
    c = R.case(os.path.join(CASES, cfg + ".cfg"), h_min, dt)
    setup = time.time() - t0
    n = args.cpu_steps
    c.step()  # first step (forward Euler bootstrap) excluded
    t1 = time.time()
    reps = [c.step() for _ in range(n)]
    el = time.time() - t1
    return {"value": round(n / el, 5), "unit": "steps/s", "cores": cores, "kind": "reference",
            "cpu_model": cpu_model(), "setup_s": round(setup, 1), "phase_s": ref_phase_seconds(reps),
            "sample": f"{n} Stepper::advance step(s) of {args.workload} after 1 warm-up step "
                      f"(setup {setup:.1f}s excluded), OMP_NUM_THREADS={cores}"}


def cpu_threads_figure(name: str = "c2") -> dict:
    """The reference Stepper on C2 with all host threads and with one thread (one step each after a
    warm-up step): the CPU model's scaling, next to the all-core figure of the headline case."""
    from oracle import oracle as O
    cfg, h_min, dt, _ = workload(name)
    R = O.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    c = R.case(os.path.join(CASES, cfg + ".cfg"), h_min, dt)
    c.step()
    out = {"config": config_of(name), "cpu_model": cpu_model(), "unit": "steps/s"}
    for threads in (cores, 1):
        R.set_threads(threads)
        t1 = time.time()
        rep = c.step()
        el = time.time() - t1
        out[f"threads_{threads}"] = {"value": round(1 / el, 5), "phase_s": ref_phase_seconds([rep])}
    R.set_threads(cores)
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU Stepper on the same config (GPU untouched)."""
    from oracle import oracle as O
    cfg, h_min, dt, desc = workload(args.workload)
    if not O.have_ref():
        return {"impl": "reference", "unavailable": "oracle/_ref/libibmref.so not built"}
    R = O.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    t0 = time.time()
    c = R.case(os.path.join(CASES, cfg + ".cfg"), h_min, dt)
    setup = time.time() - t0
    # bounded sample: at most --ref-warmup / --ref-steps steps (a reference S-4M step is ~30 s)
    W = min(args.warmup, args.ref_warmup)
    K = max(1, min(args.steps, args.ref_steps))
    for _ in range(W):
        c.step()
    t1 = time.time()
    reps = [c.step() for _ in range(K)]
    el = time.time() - t1
    its = sum(r["solve2_iters"] for r in reps)
    v = K / el
    sample = (f"{K} timed Stepper::advance step(s) after {W} warm-up (bounded sample of the requested "
              f"--steps {args.steps} --warmup {args.warmup}; setup {setup:.1f}s excluded), OMP_NUM_THREADS={cores}")
    return {"impl": "reference", "metric": "time steps/sec (IBPM step: explicit + PCG-diag + SA-PCG + projection)",
            "value": round(v, 5), "unit": "steps/s", "n_gpus": 1, "steps": K, "warmup": W,
            "ms_per_step": round(el / K * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic case file)",
            "config": config_of(args.workload), "parallelism": f"host OpenMP x{cores}",
            "cg_iters_per_step": its / K, "setup_s": round(setup, 2), "phase_s": ref_phase_seconds(reps),
            "cpu_baseline": {"value": round(v, 5), "unit": "steps/s", "cores": cores, "kind": "reference",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": round(v, 5), "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="s4m")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--ref-steps", type=int, default=2, help="--impl reference: at most this many timed steps")
    ap.add_argument("--ref-warmup", type=int, default=1, help="--impl reference: at most this many warm-up steps")
    ap.add_argument("--no-cpu-threads", action="store_true", help="skip the C2 all-core / 1-thread CPU figure")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-s4m", action="store_true", help="skip the S-4M / C2 side probe")
    ap.add_argument("--no-flapping", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C5 grid-size sweep (1024^2..8192^2)")
    ap.add_argument("--parallel", default="slab", choices=["slab", "replicas"],
                    help="N>1: row-slab distributed solve 2 over NCCL (one simulation), or N replicas")
    ap.add_argument("--min-dist-rows", type=int, default=200000,
                    help="SA levels with fewer rows are replicated on every rank")
    ap.add_argument("--watchdog", type=float, default=900.0, help="N>1: abort after this many seconds")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        # A wedged collective must not hang the job: if the whole run has not finished within
        # --watchdog seconds, this rank reports and exits (the other ranks' watchdogs do the same).
        def _watchdog():
            time.sleep(args.watchdog)
            print(json.dumps({"error": f"rank {rank}: no completion within {args.watchdog}s (watchdog)"}),
                  file=sys.stderr, flush=True)
            os._exit(3)
        threading.Thread(target=_watchdog, daemon=True).start()
    out, st = run_ours(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([out["ms_per_step"], 1e3 / out["e2e"]["value"] * (1 if args.parallel == "slab" else world)],
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
        out["ms_per_step"] = float(t[0].item())
        mult = 1 if args.parallel == "slab" else world  # slab: one simulation; replicas: N of them
        out["value"] = round(mult * 1e3 / out["ms_per_step"], 4)
        out["e2e"]["value"] = round(mult * 1e3 / float(t[1].item()), 4)
        dist.barrier()
    if rank == 0:
        del st
        if not args.no_s4m and world == 1:  # the other cylinder workload of the pair C2 / S-4M
            side = "c2" if args.workload == "s4m" else "s4m"
            if args.workload in ("s4m", "c2"):
                try:
                    out[side] = case_probe(args, side)
                except Exception as e:  # report, never hide
                    out[side] = {"error": str(e)}
        if not args.no_flapping and args.workload != "flapping" and world == 1:
            try:
                out["flapping"] = flapping_probe(args)
            except Exception as e:
                out["flapping"] = {"error": str(e)}
        if not args.no_sweep and world == 1 and args.workload in ("s4m", "c2"):
            try:  # BASELINE metric "CG iters/sec vs grid size" (configs[4] synthetic grids)
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                import sweep as _sweep
                keys = ("grid", "setup_s", "cg_iters_per_s", "cg_iteration_ms", "cg_frac_measured", "spmv_lhs2_us",
                        "spmv_format_gbs", "spmv_format_frac_measured", "spmv_format_frac_of_8tbs", "steps_per_s")
                out["grid_sweep"] = [{k: r[k] for k in keys}
                                     for r in _sweep.sweep([1024, 2048, 4096, 8192], spmv_reps=10)]
            except Exception as e:
                out["grid_sweep"] = {"error": str(e)}
        if not args.no_cpu and world == 1:
            try:
                out["cpu_baseline"] = cpu_baseline(args)
            except Exception as e:
                out["cpu_baseline"] = {"error": str(e)}
            if not args.no_cpu_threads:
                try:
                    out["cpu_threads"] = cpu_threads_figure("c2")
                except Exception as e:
                    out["cpu_threads"] = {"error": str(e)}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
