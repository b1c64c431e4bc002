"""bench.py — exponential-DG step throughput on B200 (BASELINE.json metric).

Workload (N=1): config C4 of BASELINE.json — 2D compressible Euler, strength-5
isentropic vortex on [0,10]^2, 1024 x 1024 quads, N = 4 LGL (104,857,600 DOF),
Lax-Friedrichs, EPI2 at Cr_a = 5, Krylov tol 1e-10, max dim 40 — the largest
configuration of the reference's own physics that fits one GPU (configs[1], C2,
fails in the reference algorithm itself: KrylovError -> blew_up at step 1, see
DESIGN.md).  One "step" = one EPI2 step (relinearise, R, phi_1 by the adaptive
augmented Krylov engine, u update).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints one JSON line (rank 0).  value = DOF-steps/s with the state resident in
HBM (device CUDA events around the step loop); e2e = the same metric through the
public API with host buffers (H2D + D2H of u inside every step); roofline = the
JVP + Arnoldi phi engine's canonical algorithmic bytes over the
step time against the measured HBM copy peak; cpu_baseline = the oracle (CPU
restatement of the reference, single-threaded like the reference) on a bounded
sample of the same physics.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL logs (e.g. its version banner) go to stderr: stdout carries exactly one JSON line
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
            return
        # nvidia-smi takes ~0.1-0.5 s to print its first row: wait for it, so that a short timed
        # region (C3: ~0.1 s) still has samples
        t0 = time.time()
        while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# EXPDG_BENCH_SHARED_GPU=1: a FUNCTIONAL check of the N > 1 code path with every rank on the one
# visible GPU (gloo for the bench's own small collectives, the library's peer-memory communicator
# between the processes) -- never a timing: ranks that share a device and spin on each other's
# collectives say nothing about multi-GPU speed.
SHARED_GPU = os.environ.get("EXPDG_BENCH_SHARED_GPU") == "1"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU:
        local = 0
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if SHARED_GPU else "nccl", init_method="env://")
    return world, rank, local


def _coll_dev(local):
    """Device of the bench's own small collective tensors (CPU under gloo)."""
    return "cpu" if SHARED_GPU else f"cuda:{local}"


def cpu_sample(workload, steps: int = 1, nx: int = 128, warmup: int = 0):
    """The oracle (CPU restatement of the reference) on a bounded sample of the
    same physics: same config, Courant rule and Krylov settings on nx x nx.  Loads
    only oracle/ (the dt rule takes the oracle's LGL nodes), never the CUDA library."""
    import numpy as np

    import oracle
    from paper_2011_01316_b200 import configs
    w = configs.scaled(workload, nx, steps=steps)
    spec = w.spec()
    u0 = oracle.initial_condition(w.config, w.nx, w.order, configs.SEEDS[w.config], w.noise)
    dt = w.time_step(u0, nodes=oracle.lgl(w.order)[0])
    P = oracle.Problem(spec.kind, spec.order, spec.nx, spec.ny, spec.nz, box=spec.box, periodic=spec.periodic,
                       kappa=spec.kappa, flux=spec.flux, sigma=spec.sigma, euler_flux=spec.euler_flux,
                       gamma=spec.gamma)
    u = u0
    if warmup:
        u = P.integrate("epi2", u, dt, warmup * dt, tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis).u
    r = P.integrate("epi2", u, dt, steps * dt, tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis)
    dofs = P.dim
    per_step = np.diff(np.concatenate([[0], np.asarray(r.iters_per_step)])).astype(int).tolist()
    return {"value": dofs * r.steps / r.seconds, "seconds": r.seconds, "steps": r.steps, "dofs": dofs,
            "nx": nx, "iterations": r.krylov_iterations, "iters_per_step": per_step}


def _ref_worker(a):
    name, steps, nx, warmup = a
    from paper_2011_01316_b200 import configs
    w = next(v for v in configs.ALL.values() if v.name == name)
    return cpu_sample(w, steps=steps, nx=nx, warmup=warmup)


SPEC_HBM_GBPS = 8000.0  # B200 HBM3e spec (the north star's "~8 TB/s"); `peak` is the measured copy bandwidth


def roofline(dominant, step_achieved, peak, peak_kind, traffic, steps):
    """Roofline of the dominant kernel (live CUDA-event timing of its launches) plus the
    whole step's algorithmic bandwidth."""
    step = {"achieved": step_achieved, "frac": step_achieved / peak, "frac_spec": step_achieved / SPEC_HBM_GBPS,
            "what": "phi engine (JVP + DCGS2 passes + combine + controller): algorithmic bytes of the realised "
                    "trajectory (pipelined DCGS2: JVP 32n + merged pass 8n(k+6) per column; two-pass DCGS2 "
                    "32n + 8n(2k+6); SURVEY's CGS2 count 32n + 8n(3k+6)) / step-loop time",
            "alg_bytes_per_step": traffic["alg_bytes"] / steps, "columns": traffic["columns"],
            "avnorms": traffic["avnorms"], "combines": traffic["combines"]}
    if not dominant or dominant["launches"] == 0 or dominant["ms"] <= 0:
        return {"bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s",
                "frac": step_achieved / peak, "traffic": None, "kernel": "phi engine step", "peak_kind": peak_kind,
                "step": step}
    per_launch_bytes = dominant["bytes"] / dominant["launches"]
    ach = dominant["bytes"] / (dominant["ms"] * 1e-3) / 1e9
    traffic_launch, ncu = None, None
    try:
        if dominant["ncu_file"] is None:
            raise FileNotFoundError
        with open(os.path.join(ROOT, "profiles", dominant["ncu_file"])) as f:
            ncu = json.load(f)
        traffic_launch = ncu["dram_over_alg"] * per_launch_bytes
    except Exception:
        pass
    out = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
           "frac_spec": ach / SPEC_HBM_GBPS,
           "traffic": traffic_launch, "kernel": dominant["kernel"],
           "alg_bytes_per_launch": per_launch_bytes, "launch_ms": dominant["ms"] / dominant["launches"],
           "launches": dominant["launches"], "peak_kind": peak_kind,
           "traffic_source": (ncu or {}).get("source"),
           "step": step}
    if dominant.get("other"):
        o = dominant["other"]
        out["next_kernel"] = {"kernel": o["kernel"], "achieved": o["bytes"] / (o["ms"] * 1e-3) / 1e9,
                              "launch_ms": o["ms"] / o["launches"], "launches": o["launches"],
                              "share_ms": o["ms"]}
        out["share_ms"] = dominant["ms"]
    return out


def run_reference(args, workload):
    """--impl reference: the reference's CPU path (the oracle port; the reference
    itself cannot be built here) on the host cores, bounded samples per step.  The
    reference has no intra-step parallelism (single-threaded by design,
    proj/README.md:43-45), so all host cores are used as independent single-threaded
    instances of the same sample; value = their aggregate DOF-steps/s (total work /
    slowest instance)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    nx = args.ref_nx if args.ref_nx > 0 else (10 if workload.kind == "euler3d" else 96)
    procs = args.ref_procs if args.ref_procs > 0 else (os.cpu_count() or 1)
    if procs == 1:
        samples = [cpu_sample(workload, steps=args.steps, nx=nx, warmup=args.warmup)]
    else:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            samples = pool.map(_ref_worker, [(workload.name, args.steps, nx, args.warmup)] * procs)
    slowest = max(x["seconds"] for x in samples)
    s0 = samples[0]
    value = sum(x["dofs"] * x["steps"] for x in samples) / slowest
    mesh = "x".join([str(nx)] * (3 if workload.kind == "euler3d" else 2))
    line = {
        "impl": "reference", "metric": "DOF-steps/s per exponential-DG step", "value": value,
        "unit": "DOF-steps/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * slowest / max(1, s0["steps"]), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload.name,
                   "sample": f"{mesh} elements per instance (same physics, Cr_a, Krylov tol / max dim as the "
                             f"workload; DOF-steps/s is per DOF, so the per-DOF work is comparable when the "
                             f"Krylov iterations per step match)",
                   "dofs": s0["dofs"], "instances": procs, "cores": procs,
                   "krylov_iters_per_step": s0["iters_per_step"]},
        "cpu_baseline": {"value": value, "unit": "DOF-steps/s", "cores": procs, "kind": "port",
                         "sample": f"oracle EPI2 (CPU restatement of the reference; the reference itself needs "
                                   f"Eigen, absent here), {workload.name} physics on {mesh} elements, "
                                   f"{args.steps} timed steps after {args.warmup} warm-up, {procs} concurrent "
                                   f"single-threaded instances on {procs} host cores (the reference is "
                                   f"single-threaded, proj/README.md:43-45); Krylov iterations per step "
                                   f"{s0['iters_per_step']}"},
        "e2e": {"value": value, "unit": "DOF-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--nz", type=int, default=0,
                    help="3D configs: z element count override (C5L --nz 32: one rank's share of the 4-GPU "
                         "128^3 job on a single GPU; same box, so the same dt)")
    ap.add_argument("--ref-nx", type=int, default=0,
                    help="elements per direction of the reference-arm sample (0: 96 in 2D, 10 in 3D)")
    ap.add_argument("--ref-procs", type=int, default=0, help="--impl reference instances (0: all host cores)")
    ap.add_argument("--cpu-nx", type=int, default=0,
                    help="elements per direction of the CPU baseline sample (0: 128 in 2D, 12 in 3D)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dominant", action="store_true", help="skip the dominant-kernel event timing")
    ap.add_argument("--partition", action="store_true",
                    help="slab-partitioned NCCL path even at N = 1 (always used for N > 1)")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent full-size replicas instead")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="partitioned runs: device-resident peer-memory collectives (graph control) or NCCL "
                         "(host-stepped control)")
    ap.add_argument("--host-control", action="store_true",
                    help="host-stepped controller (same kernels, no graph WHILE nodes): for ncu, which "
                         "cannot profile kernel nodes of graphs with conditional nodes")
    args = ap.parse_args()

    from dataclasses import replace

    from paper_2011_01316_b200 import configs
    workload = configs.ALL[args.config]
    if args.nz > 0:
        if workload.kind != "euler3d":
            raise SystemExit("--nz: 3D configs only")
        workload = replace(workload, nz=args.nz, name=f"{workload.name}@{workload.nx}x{workload.ny}x{args.nz}")
    if args.impl == "reference":
        run_reference(args, workload)
        return

    import numpy as np
    import torch

    import paper_2011_01316_b200 as pkg

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    ctx = pkg.Context(local)
    w = workload
    spec = w.spec()
    n_global = w.dofs
    # N > 1: element-row slabs of the one C4 mesh (strong scaling), halo rows and the
    # Gram-Schmidt / norm sums between the ranks; --partition forces the
    # partitioned path at N = 1 (a world of one) to exercise it on a single GPU.  --comm peer
    # (default): the device-resident peer-memory communicator (kernel allreduce / halo over
    # NVLink P2P through CUDA IPC mappings, graph control kept); --comm nccl: NCCL with
    # host-stepped control.
    partitioned = (world > 1 or args.partition) and not args.replicas
    if partitioned:
        from paper_2011_01316_b200.partition import slab_ranges

        npe = spec.order + 1
        layers, blk = {"burgers1d": (spec.nx, npe), "burgers2d": (spec.ny, spec.nx * npe ** 2),
                       "euler2d": (spec.ny, spec.nx * npe ** 2 * 4),
                       "euler3d": (spec.nz, spec.nx * spec.ny * npe ** 3 * 5)}[spec.kind]
        if args.comm == "peer":
            handle = ctx.peer_export(world, blk)
            handles = [handle]
            if world > 1:
                handles = [None] * world
                torch.distributed.all_gather_object(handles, handle)
            ctx.attach_peer(handles, rank, world)
        else:
            uid = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                uid = torch.tensor(list(pkg.nccl_unique_id()), dtype=torch.uint8)
            if world > 1:
                t_uid = uid.to(_coll_dev(local))
                torch.distributed.broadcast(t_uid, 0)
                uid = t_uid.cpu()
            ctx.attach_nccl(bytes(uid.tolist()), rank, world)
        rows = slab_ranges(layers, world)[rank]
        spec.part = rows
        if w.config == 5:  # each rank builds only its z-slab (C5L: 5.4 GB global state)
            u0 = w.initial_condition_slab(*rows)
        else:
            u0 = w.initial_condition()[rows[0] * blk:rows[1] * blk].copy()
    else:
        u0 = w.initial_condition()
    # dt = cfl dx_min / c_max over the whole state: the min over ranks of the local rule
    dt = w.time_step(u0) if w.dt is None else w.dt
    if world > 1:
        t_dt = torch.tensor([dt], dtype=torch.float64, device=_coll_dev(local))
        torch.distributed.all_reduce(t_dt, op=torch.distributed.ReduceOp.MIN)
        dt = float(t_dt.item())
    op = pkg.Operator(ctx, spec)
    n = op.dim
    kw = dict(tol=w.tol, max_basis=w.max_basis, orth_length=w.max_basis, use_graph=not args.host_control)
    u = torch.tensor(u0, device=f"cuda:{local}")

    # warm-up steps (untimed)
    rw = pkg.integrate(ctx, op, u, "epi2", dt, args.warmup * dt, **kw)
    if rw.status != "completed":
        raise RuntimeError(f"warm-up blew up at step {rw.blow_up_step}")
    # the e2e leg replays the timed trajectory from this same state (same steps, same
    # Krylov dimensions), from pinned host memory
    u_start = None if args.no_e2e else torch.empty(n, dtype=torch.float64, pin_memory=True)
    if u_start is not None:
        u_start.copy_(u)

    # timed region: barrier + synchronize on both sides, device events inside the library
    clocks = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.kernel_launches
    r = pkg.integrate(ctx, op, u, "epi2", dt, args.steps * dt, **kw)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        torch.distributed.barrier()
    launches = ctx.kernel_launches - l0
    traffic = ctx.traffic()
    dominant = None
    if not args.no_dominant:
        # the dominant kernel: CUDA events around each launch of the two largest kernels (the
        # DCGS2 update pass; the operator sweep, which at C4 also takes the DCGS2 dots) on the
        # context stream over one host-stepped step of the same trajectory; the one with the
        # larger summed time is reported (its algorithmic bytes are accumulated on the device)
        timed = []
        # the operator sweep of this workload, and the ncu capture (DRAM / algorithmic bytes of
        # one launch) made on the same config, if any
        # pipelined DCGS2: per column one operator application (the lookahead, stage 2: reads W,
        # q~, b_1, writes Y = 32 n bytes; the first column of a substep also runs stage 1 with the
        # fused pass-1 dots) and one merged basis pass k_ts3 (8 n (j + 6) bytes)
        sweep = {
            "euler2d": ("k_e2_phi_strip_fw<5,LF,4> (Euler strip JVP with a face warp: the lookahead application "
                        "dt A (s_j W) -> Y, reads W, q~, b_1, writes Y; + k_e2_phi_strip<5,LF,8,DOT> with the "
                        "pass-1 dots at substep starts)",
                        "r02f_ncu_dominant_strip.json"),
            "burgers2d": ("k_b2_phi_strip<5,*> (2D Burgers strip JVP: reads x, u~, b_1, writes y; + the pass-1 "
                          "dots at substep starts)", None),
            "euler3d": ("k_e3_phi_march_fw<4> (3D Euler z-march JVP with face warps: reads x, q~, b_1, writes y; "
                        "+ k_e3_phi_march<4,DOT> with the pass-1 dots at substep starts)", None),
        }.get(w.kind, ("operator sweep (JVP of slot j)", None))
        for kind, name, ncu_file in (
                (1, "k_ts3 (pipelined DCGS2 merged pass, column j: u <- u - V a, W <- W - g u - V mu, "
                    "Y <- Arnoldi-relation image, + column j+1 pass-1 dots; reads V_0..V_{j-1}, u, W, Y, "
                    "writes u, W, Y; k_ts2<TS2_UPD> on substep-final avnorm cycles)",
                 "r02f_ncu_dominant_ts3.json" if w.kind == "euler2d" else None),
                (2, sweep[0], sweep[1])):
            ud = u.clone()
            ctx.time_dominant(kind)
            pkg.integrate(ctx, op, ud, "epi2", dt, dt, **{**kw, "use_graph": False})
            d = ctx.dominant_stats()
            ctx.time_dominant(False)
            del ud
            if d["launches"] > 0 and d["bytes"] > 0:
                timed.append({**d, "kernel": name, "ncu_file": ncu_file})
        if timed:
            timed.sort(key=lambda d: -d["ms"])
            dominant = timed[0]
            if len(timed) > 1:
                dominant["other"] = timed[1]
    if r.status != "completed" or r.steps != args.steps:
        raise RuntimeError(f"timed run: {r.status} after {r.steps} steps")
    loop_s = r.loop_ms / 1e3
    if world > 1:
        t = torch.tensor([loop_s], device=_coll_dev(local))
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        loop_s = float(t.item())
    total_dofs = n_global if partitioned else world * n
    value = total_dofs * args.steps / loop_s
    peak, peak_kind = hbm_peak()
    achieved = traffic["alg_bytes"] / (r.loop_ms / 1e3) / 1e9
    iters_per_step = np.diff(np.concatenate([[0], r.iters_per_step])) if len(r.iters_per_step) else []

    # e2e: public API with host buffers, H2D + D2H of u inside every step, from the
    # timed region's start state over the same K steps (one integrate call per step)
    e2e = None
    if not args.no_e2e:
        uh_np = u_start.numpy()
        if world > 1:
            torch.distributed.barrier()
        e_iters = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            re = pkg.integrate(ctx, op, uh_np, "epi2", dt, dt, **kw)
            if re.status != "completed":
                raise RuntimeError("e2e step blew up")
            e_iters.append(int(re.krylov_iterations))
        t1 = time.perf_counter()
        e_s = t1 - t0
        if world > 1:
            tt = torch.tensor([e_s], device=_coll_dev(local))
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e_s = float(tt.item())
        e2e = {"value": total_dofs * args.steps / e_s, "unit": "DOF-steps/s", "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n, "seconds": e_s, "krylov_iters_per_step": e_iters,
               "same_trajectory": [int(v) for v in iters_per_step] == e_iters}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.cpu_nx <= 0:
            args.cpu_nx = 12 if w.kind == "euler3d" else 128
        s = cpu_sample(w, steps=1, nx=args.cpu_nx)
        cpu = {"value": s["value"], "unit": "DOF-steps/s", "cores": 1, "kind": "port",
               "sample": f"oracle EPI2 (CPU restatement of the reference, single-threaded), {w.name} physics "
                         f"on {'x'.join([str(args.cpu_nx)] * (3 if w.kind == 'euler3d' else 2))} elements ({s['dofs']} DOF), 1 step, "
                         f"{s['seconds']:.1f} s"}

    if rank == 0:
        line = {
            "metric": "DOF-steps/s per exponential-DG step", "value": value, "unit": "DOF-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * loop_s / args.steps, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": {"euler2d": "synthetic (seeded strength-5 isentropic vortex + 1e-6 N(0,1) density noise)",
                     "euler3d": "synthetic (Taylor-Green vortex, Mach 0.1, analytic; per-rank z-slabs)",
                     "burgers2d": "synthetic (sin(2 pi x) sin(2 pi y) + 0.01 N(0,1) seeded noise)",
                     "burgers1d": "synthetic (seeded Burgers initial state)"}[w.kind],
            "config": {"workload": w.name, "dofs": n_global, "dofs_per_rank": n,
                       "elements": "x".join(str(v) for v in ((w.nx, w.ny, w.nz) if w.kind == "euler3d"
                                                              else (w.nx, w.ny))),
                       "order": w.order,
                       "dt": dt, "cr_a": w.cfl, "krylov": {"tol": w.tol, "max_basis": w.max_basis,
                                                           "orth_length": w.max_basis},
                       "integrator": "epi2", "l2": "inputs larger than L2 (Krylov workspace "
                       f"{(w.max_basis + 2) * 8 * n / 1e9:.1f} GB vs 126 MB L2)",
                       "parallelism": (f"{world}-way element slabs ({args.comm} halo + allreduce)" if partitioned
                                       else "single GPU" if world == 1 else f"{world} independent replicas"),
                       "krylov_iters_per_step": [int(v) for v in iters_per_step]},
            "roofline": roofline(dominant, achieved, peak, peak_kind, traffic, args.steps),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
