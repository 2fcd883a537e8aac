#!/usr/bin/env python
"""SISPH hot-path benchmark (BASELINE.json metric: PPE Jacobi sweeps x particles / s
and ms / timestep; % HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sisph|reference]

A step is one full SISPH step (Algorithm 1: two neighbour
builds, density, wall BCs, forces + predictors, RHS/D_ii, the iterated PPE,
pressure-gradient correction, K GTVF sub-steps, advance) on the per-GPU slab of
BASELINE configs[4] (3D dam break, fp32).  Inputs are synthetic (synth/).

value = (sum over the K timed steps of PPE sweeps x fluid particles) x n_gpus
        / (device time of the K whole steps)       [particle-sweeps / s]
ms_per_step = device time of one whole step.
The oracle (oracle/, fp64 C) is timed on the host as cpu_baseline, and is the
--impl reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

# stdout carries exactly one JSON line: the real stdout is kept aside for it and file
# descriptor 1 points at stderr, so that whatever libraries print there (NCCL's "NCCL version"
# banner, CUDA / torch notices) cannot interleave with the result
_JSON_FD = None   # set by main()

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PPE Jacobi particle-sweeps/s (sweeps x fluid particles per second of whole SISPH-step time)"
UNIT = "particle-sweeps/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sisph", choices=["sisph", "reference"])
    ap.add_argument("--workload", default="dambreak3d",
                    choices=["dambreak3d", "tgv3d", "dambreak2d", "hydrostatic", "tgv2d"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--slab-self", action="store_true",
                    help="ablation on one GPU: the slab path (halos over NCCL to itself across the periodic y)")
    ap.add_argument("--ppe-loop", type=int, default=0,
                    help="PPE loop form: 0 auto, 1 host-polled batches, 2 CUDA-graph WHILE node, 3 persistent kernel")
    ap.add_argument("--matrix-free", action="store_true",
                    help="ablation: the sweep recomputes fac_ij every sweep (PAPER.md:785-801)")
    return ap.parse_args()


def workload(name, ranks=1):
    import synth
    if name == "dambreak3d":
        c = synth.dambreak3d(ranks=ranks)
        desc = ("3D dam break per-GPU slab (BASELINE configs[4]): fluid 256x64x128 at dx=1/256, "
                "3 wall layers, y periodic, fp32, tol 1e-2, K=10")
        if ranks > 1:
            desc += f"; {ranks} slabs along y, global fluid 256x{64 * ranks}x128 = {c.n_fluid} particles"
    elif name == "tgv3d":
        c = synth.tgv3d()
        desc = "3D Taylor-Green 128^3 periodic (BASELINE configs[3]), fp32, tol 1e-3"
    elif name == "dambreak2d":
        c = synth.dambreak2d()
        desc = "2D dam break 500x1000 fluid in a 4x4 tank (BASELINE configs[2]), fp32, tol 1e-2"
    elif name == "tgv2d":
        c = synth.tgv2d()
        desc = "2D Taylor-Green 50x50 periodic (BASELINE configs[0]), fp64, tol 1e-4, 10 steps as configured"
    else:
        c = synth.hydrostatic()
        desc = "2D hydrostatic column 200x400 (BASELINE configs[1]), fp32, tol 1e-3"
    return c, desc


def sample_case(name, small=False):
    """Bounded CPU sample of the same workload.  small: the reference arm's per-step
    sample, so that --steps K --warmup W of the oracle ends within a few minutes."""
    import synth
    if name == "dambreak3d" and small:
        # same dx, parameters and recipe; a 64 x 12 x 64 block in a quarter-length tank
        return (synth.dambreak3d(nfx=64, nfy=12, nfz=64, tank_nx=206, wall_nz=77),
                "64 x 12 x 64 block of the same dam-break recipe (dx = 1/256, quarter-length tank)")
    if name == "dambreak3d":
        # 12 of the 64 spanwise rows: the periodic y axis keeps 4 cells of 3h (>= 3, R26)
        return synth.dambreak3d(nfy=12), "12/64 spanwise slab of the per-GPU workload (nfy=12)"
    if name == "tgv3d":
        return synth.tgv3d(n=64), "64^3 instance of the same TGV-3D recipe"
    if name == "dambreak2d":
        return synth.dambreak2d(nx=250, ny=500, dx=0.004), "dx=0.004 instance of the same dam break"
    if name == "tgv2d":
        return synth.tgv2d(), "the full workload"
    return synth.hydrostatic(), "the full workload"


class ClockSampler:
    """SM clock + throttle reasons via NVML every 20 ms while the timed region runs."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def sweep_traffic(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum of one k_sweep launch from the committed
    ncu --set full capture of THIS workload (profiles/traffic_<workload>.json), else None."""
    p = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def kernel_instr(workload):
    """Warp instructions per launch of the issue-bound kernels (sm__inst_executed.sum from the
    committed ncu --set full captures of this workload), profiles/instr_<workload>.json."""
    p = os.path.join(ROOT, "profiles", f"instr_{workload}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def alu_peak(device):
    """The FP32 issue roof of this GPU at its current clocks:
    libsisph_tools.so's FFMA / MUFU micro-benchmark (csrc/sisph_tools.cu)."""
    import ctypes
    from paper_1908_01762_b200 import build as B
    lib = ctypes.CDLL(B.build_tools())
    out = (ctypes.c_double * 4)()
    rc = lib.sisph_tools_alu_peak(int(device), out)
    if rc != 0:
        return None
    return {"ffma_warp_instr_per_s": out[0], "fp32_tflops": out[0] * 64 / 1e12,
            "mufu_rsq_warp_instr_per_s": out[1], "issue_warp_instr_per_s": out[2],
            "sm_mhz_during": out[3],
            "how": "8 independent FFMA (MUFU.RSQ) chains per thread, 8 x SMs blocks of 256 threads, CUDA events"}


def cpu_baseline(name, max_seconds=20.0):
    """The oracle as it stands, on a bounded sample, on all host cores (fp64):
    whole SISPH steps, same metric definition as `value`."""
    import oracle
    oracle.build()
    case, desc = sample_case(name)
    o = oracle.Sim(case)
    sweeps, steps = 0, 0
    t0 = time.perf_counter()
    while True:
        it, _, _ = o.step(case.dt)
        sweeps += it
        steps += 1
        t = time.perf_counter() - t0
        if t > max_seconds or steps >= 50:
            break
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    return {"value": sweeps * case.n_fluid / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "ms_per_step": 1e3 * t / steps,
            "sample": f"{desc}: {steps} full SISPH steps ({sweeps} PPE sweeps) over {case.n_fluid} fluid "
                      f"particles, {t:.1f} s, fp64"}


def emit(d):
    if _JSON_FD is None:
        print(json.dumps(d), flush=True)
        return
    sys.stdout.flush()
    os.write(_JSON_FD, (json.dumps(d) + "\n").encode())


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if "RANK" in os.environ and os.environ.get("OMP_NUM_THREADS") == "1":
        # torchrun's default of one thread per rank: rank 0 alone runs the oracle here, on all
        # host cores as at N = 1 (OpenMP reads this when the oracle library first runs)
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    import oracle
    oracle.build()
    case, sdesc = sample_case(args.workload, small=True)
    _, desc = workload(args.workload)
    o = oracle.Sim(case)
    for _ in range(args.warmup):
        o.step(case.dt)
    t0 = time.perf_counter()
    sweeps = 0
    for _ in range(args.steps):
        it, _, _ = o.step(case.dt)
        sweeps += it
    t = time.perf_counter() - t0
    v = sweeps * case.n_fluid / t
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic", "config": {"workload": desc, "reference_sample": sdesc,
                                          "n_fluid_sample": case.n_fluid},
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                           "sample": f"{sdesc}: {args.steps} full SISPH steps, fp64"},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


SLAB_AXIS = {"dambreak3d": 1, "tgv3d": 0, "dambreak2d": 0, "hydrostatic": 0, "tgv2d": 0}


def run_sisph(args):
    import numpy as np
    import torch

    from paper_1908_01762_b200 import Simulation, default_nccl_lib
    from paper_1908_01762_b200 import dist as D

    rank, world, local = D.env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # weak scaling: the per-GPU problem is fixed, the global problem has `world` slabs
    case, desc = workload(args.workload, ranks=world)
    stream = torch.cuda.current_stream()
    over = dict(stream=stream.cuda_stream, device=local, matrix_free=1 if args.matrix_free else 0)
    if args.ppe_loop:
        over["ppe_loop"] = args.ppe_loop
    if world > 1:
        # one process per GPU: torch.distributed (NCCL) carries the NCCL id; the halo
        # exchanges and per-sweep allreduce run inside libsisph over NCCL
        D.init_process_group("nccl")
        nccl_lib = default_nccl_lib()
        uid = D.share_nccl_id(rank, nccl_lib)
        sim = D.create_rank(case, SLAB_AXIS[args.workload], rank, world, uid, nccl_lib, **over)
    elif args.slab_self:
        from paper_1908_01762_b200 import make_dist, nccl_unique_id
        nccl_lib = default_nccl_lib()
        d = make_dist(1, 0, SLAB_AXIS[args.workload], nccl_id=nccl_unique_id(nccl_lib), nccl_lib=nccl_lib,
                      always_slab=True)
        sim = Simulation.from_case(case, dist=d, **over)
    else:
        sim = Simulation.from_case(case, **over)
    nf, n = sim.n_fluid, sim.n            # global counts
    nf_own = sim.owned_counts()[0]

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as td
            td.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sim.step(case.dt)
    barrier()
    reps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one event per step boundary as well (the median step)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        e0.record(stream)
        for k in range(args.steps):
            reps.append(sim.step(case.dt))
            ev[k].record(stream)
        e1.record(stream)
        barrier()
    ms_rank = e0.elapsed_time(e1)
    step_ms = [e0.elapsed_time(ev[0])] + [ev[k - 1].elapsed_time(ev[k]) for k in range(1, args.steps)]
    ms = D.max_over_ranks(ms_rank, dev) if world > 1 else ms_rank   # the job's time: its slowest rank
    sweeps = sum(r.iters for r in reps)   # identical on every rank (allreduced decision)
    value = sweeps * nf / (ms / 1e3)      # all ranks' fluid particles
    # instrumented steps after the timed region (per-phase and per-sweep CUDA events; the
    # PPE loop then runs host-polled so that each sweep launch can be bracketed)
    sim.set_timing(True)
    ireps = [sim.step(case.dt) for _ in range(max(3, min(args.steps, 10)))]
    sim.set_timing(False)
    barrier()
    ms_solve_i = sum(r.ms_solve for r in ireps)
    sweeps_i = sum(r.iters for r in ireps)
    # roofline of the dominant hot-path kernel: the Jacobi sweep (A12), timed on one more
    # step whose solve runs a fixed 21 sweeps (tol 0): 20 standalone sweep launches, each
    # bracketed by CUDA events on the handle's stream
    sim.set_timing(True)
    sim.predict(case.dt)
    sim.ppe_solve(0.0, 21)
    ms_sw, n_sw = sim.sweep_timing()
    sim.correct(case.dt)
    sim.set_timing(False)
    barrier()
    pairs = reps[-1].pairs
    n_loc = nf_own + (n - nf) // world if world > 1 else n     # this rank's rows (roofline: per-GPU kernel)
    nf_loc = nf_own
    nw_loc = n_loc - nf_loc
    tb = 4 if case.params["precision"] == 32 else 8
    d = case.dim
    # SURVEY.md §8(d) M3(a), design (i): the ALGORITHMIC bytes of one sweep = the state of every
    # fluid row read or written once (r: d s, rho, p^k, RHS, D_ii, p^{k+1}: 5 s, fs: 1 byte;
    # 33 B in 3D fp32) + the stored neighbour structure, a 4-byte index per interaction
    state_b = d * tb + 5 * tb + 1
    b_alg = state_b * nf_loc + 4 * pairs
    # what this design actually streams per launch (reported apart, it is not "useful" bytes):
    if args.matrix_free:
        # pos (x, y, z, m), rho, p^k of every particle; rhs, diag, cnt, p^{k+1} (+ fs) of every
        # fluid row; the 4-byte index of every pair
        b_str = (6 * tb) * n_loc + (3 * tb + 5) * nf_loc + 4 * pairs
    else:
        # p^k of every particle; rho, rhs, diag, cnt, p^{k+1} (+ fs) of every fluid row; per pair
        # the 4-byte index and the stored factor of fac_ij
        b_str = tb * n_loc + (4 * tb + 5) * nf_loc + (4 + tb) * pairs
    avg_s = ms_sw / max(n_sw, 1) / 1e3
    achieved = b_alg / avg_s / 1e9
    peak, peak_src = peaks()
    # M1 = sum(sweeps x N_f) / t_PPE with t_PPE from the start of A11 (wall p^0, RHS, D_ii and the
    # fused first sweep) to the final decision of the solve
    ms_ppe_i = sum(r.ms_ppe for r in ireps)
    # the neighbour-build + PPE pipeline (north_star's ">= 60 % of the HBM roofline"): algorithmic
    # bytes per step of
    #   sort / reorder (A1-A4): hash reads r (4 s) and writes key + rank (8 B), the scatter moves
    #     key, rank, slot (12 B), the reorder reads and writes the carried state (r, u, u~: 3 x 4 s,
    #     p, rho: 2 s, id 4 B, fs 1 B) -> 32 s + 30 B per fluid particle (158 B in fp32)
    #   the exact r* neighbour list (A5 / A9): positions read once (4 s per particle), the list
    #     written once (4 B per interaction)
    #   A11: r*, u* (2 x 4 s), rho, fs read, RHS, D_ii written (3 s + 1 B) per fluid row, walls'
    #     r and u* (2 x 4 s), the list read once (4 B per interaction)
    #   every sweep: b_alg (A11's fused first sweep included)
    # over the device time of those phases (CUDA events: ms_build + ms_filter + ms_ppe)
    sw_i = sweeps_i / len(ireps)
    vb = 4 * tb   # one (x, y, z, m) / (u, rho) record
    pipe_b = ((32 * tb + 30) * nf_loc + vb * n_loc + 4 * pairs
              + (2 * vb + 3 * tb + 1) * nf_loc + 2 * vb * nw_loc + 4 * pairs
              + sw_i * b_alg)
    pipe_ms = sum(r.ms_build + r.ms_filter + r.ms_ppe for r in ireps) / len(ireps)
    alu = alu_peak(local)
    instr = kernel_instr(args.workload)
    m3 = None
    if alu and instr:
        # M3(b) issue fraction of the issue-bound kernels: the committed ncu warp-instruction count
        # of one launch over this run's launch time x the measured issue roof; M3(c) binding
        # roofline: max(bytes / HBM peak, instructions / issue roof) / launch time
        m3 = {}
        ph = {"k_sweep": avg_s}
        for kname, rec in instr.items():
            t = ph.get(kname)
            if t is None and rec.get("us_ncu"):
                t = rec["us_ncu"] * 1e-6
            if not t:
                continue
            ins = rec["warp_instr"]
            byt = rec.get("dram_bytes", 0.0)
            m3[kname] = {"issue_frac": ins / t / alu["issue_warp_instr_per_s"],
                         "binding_frac": max(byt / (peak * 1e9), ins / alu["issue_warp_instr_per_s"]) / t,
                         "time_source": "live CUDA events" if kname in ph else "ncu gpu__time_duration",
                         "warp_instr": ins}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.workload == "dambreak3d" else "strong",
        "vs_baseline": None, "dtype": "f32" if case.params["precision"] == 32 else "f64",
        "data": "synthetic",
        "config": {"workload": desc, "n_fluid": nf, "n_wall": n - nf, "dt": case.dt,
                   "l2": "inputs larger than L2 (neighbour list %.2f GB, state %.0f MB per GPU)"
                         % (4 * pairs / 1e9, 24 * n_loc / 1e6),
                   "parallelism": f"slab x{world}" + (f" along axis {SLAB_AXIS[args.workload]}, NCCL halos + "
                                                      "per-sweep allreduce" if world > 1 else "")},
        "ms_per_step_median": float(np.median(step_ms)),
        # t_PPE from the start of A11 to the final decision (the fused first sweep
        # and the wall passes included); instrumented steps after the timed region
        "ppe_phase_particle_sweeps_per_s": sweeps_i * nf / (ms_ppe_i / 1e3) if ms_ppe_i > 0 else None,
        "sweeps_per_step": sweeps / args.steps,
        "single_build_steps": sum(r.single_build for r in reps),
        "ms_per_step_phases": {"predict": sum(r.ms_predict for r in ireps) / len(ireps),
                               "solve": sum(r.ms_solve for r in ireps) / len(ireps),
                               "correct": sum(r.ms_correct for r in ireps) / len(ireps),
                               "build_rn": sum(r.ms_build for r in ireps) / len(ireps),
                               "rstar_sets": sum(r.ms_filter for r in ireps) / len(ireps),
                               "a11": sum(r.ms_rhs for r in ireps) / len(ireps),
                               "ppe_from_a11": ms_ppe_i / len(ireps),
                               "note": f"{len(ireps)} instrumented steps after the timed region "
                                       "(events between phases, host-polled PPE loop)"},
        "roofline": {"kernel": "k_sweep (A12 Jacobi sweep + fused residual reduction, "
                               + ("fac_ij recomputed per sweep)" if args.matrix_free else "stored fac_ij streamed)"),
                     "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": sweep_traffic(args.workload),
                     "algorithmic_bytes_per_launch": b_alg,
                     "algorithmic_bytes_def": f"SURVEY §8(d) M3(a) design (i): {state_b} B of state per fluid row "
                                              "+ 4 B per interaction",
                     "bytes_streamed_per_launch": b_str,
                     "streamed_frac": b_str / avg_s / 1e9 / peak,
                     "pairs_per_launch": pairs,
                     "avg_launch_us": avg_s * 1e6, "launches_timed": n_sw,
                     # interactions/s and the logical gather bandwidth (the
                     # p_j each interaction gathers; served by L1/L2, not an HBM fraction)
                     "interactions_per_s": pairs / avg_s,
                     "gather_logical_GBs": tb * pairs / avg_s / 1e9,
                     "how": "20 sweep launches of a fixed-sweep solve after the timed region, CUDA events "
                            "on the handle's stream",
                     "peak_source": peak_src + " (burst copy figure; the sweep is timed alone)"},
        "pipeline_roofline": {"phases": "build at r^n (A1-A5) + r* sets (A9) + A11 + PPE sweeps to the decision",
                              "algorithmic_bytes": pipe_b, "ms": pipe_ms,
                              "achieved": pipe_b / (pipe_ms / 1e3) / 1e9 if pipe_ms > 0 else None,
                              "peak": peak, "unit": "GB/s",
                              "frac": pipe_b / (pipe_ms / 1e3) / 1e9 / peak if pipe_ms > 0 else None,
                              "bytes_def": "158 B / fluid particle (hash, sort, reorder) + 16 B / particle + "
                                           "4 B / interaction (the exact r* list) + A11 state + 4 B / "
                                           "interaction + sweeps x (state + 4 B / interaction)"},
        "alu_peak": alu,
        "m3_issue_bound": m3,
        "gpu_launches": int(sum(r.launches for r in reps)),
        "halo": {"ghost_fluid_per_rank": int(reps[-1].n_ghost_fluid),
                 "bytes_sent_per_step_rank0": int(sum(r.halo_bytes for r in reps) / args.steps)}
                if (world > 1 or args.slab_self) else None,
        "clocks": clk.summary(),
    }
    # end to end through the public API with host buffers
    if not args.no_e2e:
        dim = case.dim
        # host buffers at the handle's precision (fp32 handles: sisph_{get,set}_field_f32)
        f32 = case.params["precision"] == 32
        hdt, hb = (torch.float32, 4) if f32 else (torch.float64, 8)
        pin = lambda shape: torch.empty(shape, dtype=hdt, pin_memory=True)
        hx, hu, hut, hp = pin((n, dim)), pin((n, dim)), pin((n, dim)), pin((n,))
        sim.get_ptr("POSITION", hx.data_ptr(), n * dim, f32)
        sim.get_ptr("VELOCITY", hu.data_ptr(), n * dim, f32)
        sim.get_ptr("TRANSPORT_VELOCITY", hut.data_ptr(), n * dim, f32)
        sim.get_ptr("PRESSURE", hp.data_ptr(), n, f32)
        if world > 1:
            # each rank filled its own particles: sum the ranks' arrays into the whole state,
            # so that every rank can feed any particle it comes to own
            import torch.distributed as td
            for hbuf in (hx, hu, hut, hp):
                t = hbuf.to(dev)
                td.all_reduce(t)
                hbuf.copy_(t.cpu())
        out_p = pin((n,))
        K2 = args.e2e_steps
        fields = (("POSITION", hx, n * dim), ("VELOCITY", hu, n * dim), ("TRANSPORT_VELOCITY", hut, n * dim),
                  ("PRESSURE", hp, n))

        def e2e(pipelined):
            """K2 steps, each fed its input state from pinned host memory and read back (p).
            pipelined: sisph_stage_field uploads step k+1's inputs while step k computes,
            sisph_commit_staged applies them (the public pipelined-input API); else
            sisph_set_field before each step (upload, then compute)."""
            sw = 0
            barrier()
            t0 = time.perf_counter()
            if pipelined:
                for f, buf, cnt in fields:
                    sim.stage_ptr(f, buf.data_ptr(), cnt, f32)
            for k in range(K2):
                if pipelined:
                    sim.commit_staged()
                    if k + 1 < K2:
                        for f, buf, cnt in fields:
                            sim.stage_ptr(f, buf.data_ptr(), cnt, f32)
                else:
                    for f, buf, cnt in fields:
                        sim.set_ptr(f, buf.data_ptr(), cnt, f32)
                sw += sim.step(case.dt).iters
                if pipelined:
                    # the read of step k's p overlaps step k + 1 (waited for before the next fetch)
                    sim.fetch_wait()
                    sim.fetch_ptr("PRESSURE", out_p.data_ptr(), n, f32)
                else:
                    sim.get_ptr("PRESSURE", out_p.data_ptr(), n, f32)
            if pipelined:
                sim.fetch_wait()
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            if world > 1:
                t = D.max_over_ranks(t, dev)
            return t, sw

        # untimed warm-up of the pipelined calls: their staging / download buffers and streams are
        # allocated on first use
        for f, buf, cnt in fields:
            sim.stage_ptr(f, buf.data_ptr(), cnt, f32)
        sim.commit_staged()
        sim.fetch_ptr("PRESSURE", out_p.data_ptr(), n, f32)
        sim.fetch_wait()
        torch.cuda.synchronize()
        t_s, sw_s = e2e(False)
        t, sw2 = e2e(True)
        out["e2e"] = {"value": sw2 * nf / t, "unit": UNIT, "h2d_bytes_per_step": hb * n * (3 * dim + 1),
                      "d2h_bytes_per_step": hb * n, "host_dtype": "f32" if f32 else "f64", "steps": K2,
                      "ms_per_step": 1e3 * t / K2,
                      "how": "sisph_stage_field uploads of step k+1's inputs (pinned host) overlap step k, "
                             "sisph_fetch_field's read of step k's p overlaps step k+1; per step "
                             "sisph_commit_staged, sisph_step, sisph_fetch_wait + sisph_fetch_field(PRESSURE)",
                      # every e2e step repeats the step from the uploaded state (the one after the
                      # timed steps), so its sweep count can differ from theirs (same on C5)
                      "sweeps_per_step": sw2 / K2,
                      "serial": {"value": sw_s * nf / t_s, "ms_per_step": 1e3 * t_s / K2,
                                 "how": "sisph_set_field of every input, the step, sisph_get_field(PRESSURE)"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.workload)
    del np
    if rank == 0:
        emit(out)
    if world > 1:
        sim.close()
        import torch.distributed as td
        td.barrier()
        td.destroy_process_group()


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1, exactly as the driver launches it;
    rank 0 prints the JSON line on the inherited stdout.  Returns the launcher's exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    global _JSON_FD
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rf = os.environ.get("SISPH_BENCH_RANKFILE")
    if rf:   # CPU test hook: every rank records that it started
        with open(rf, "a") as f:
            f.write(f"{os.environ.get('RANK', '0')}/{max(world, 1)}\n")
        if os.environ.get("SISPH_BENCH_DRYRUN"):
            return
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sisph(args)


if __name__ == "__main__":
    main()
