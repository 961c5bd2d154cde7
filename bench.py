#!/usr/bin/env python3
"""ISDC hot-path benchmark (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--mode isdc|sdc] [--impl ours|reference]

A "step" is one ISDC time step of a BASELINE.json config -- every row of SURVEY.md §8(a) over one
batch of synthetic input: RHS assembly (Eq. 5), 2 V(2,2)-cycles per node solve, f^E, the SDC residual
after every sweep, sweeps until ||r~|| < 1e-10.  The default workload is config 5 (3D advection-
diffusion, 511^3, M = 5, CD4 advection, a 5-step trajectory that restarts from u0 after its 5th
step): the LARGEST single-GPU config, one of the two sizes of the north-star roofline target.  The
other target size, config 3 (2D, 4095^2), is measured in the same run and reported in "extra".

N > 1 (torchrun): replicas -- every rank runs its own independent problem on its own GPU with no
collective on the data path ("replicas only"); value = all ranks' steps / max time.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the host cores.  It cannot
run a full step in minutes (config 5: ~30 min per step on 16 cores), so every "step" of that arm is
a bounded full-size sample -- one of {RHS, one V-cycle, f^E, residual}, in rotation -- and the
step time is EXTRAPOLATED from the per-component means and the (identical) sweep count per step;
the line says so in its fields ("extrapolated", "sample", "wall_s").
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "ISDC steps/s + V-cycles/s (fp64, 1 B200); HBM GB/s as fraction of ~8 TB/s peak"
# fine-level kernel classes (isdc_profile classes 0-2) -> the kernel that implements them
KERNEL_NAMES = {
    (2, "fine_defect_restrict"): "f2d::k_smooth2r: 2 Jacobi sweeps + defect + full weighting (26 B/pt)",
    (2, "fine_prolong_correct"): "f2d::k_smooth2<MODE 2>: bilinear prolongation + correction + 2 Jacobi sweeps (26 B/pt)",
    (2, "fine_smoother"): "f2d::k_smooth2: 2 Jacobi sweeps (24 B/pt)",
    (3, "fine_smoother"): "f3d::k_smooth2ws: 2 Jacobi sweeps, warp-specialised z-streaming (24 B/pt)",
    (3, "fine_defect_restrict"): "f3d::k_restrict: defect + full weighting (17 B/pt)",
    (3, "fine_prolong_correct"): "f3d::k_prolong: trilinear prolongation + correction (17 B/pt)",
    (3, "residual"): "f3d residual pass (DESIGN.md §6.10)",
    (2, "residual"): "f2d::k_resid_s residual (DESIGN.md §6.6)",
}
WORKLOAD = {1: "cfg1_heat2d_63_M3", 2: "cfg2_allencahn2d_1023_M5", 3: "cfg3_forced_heat2d_4095_M5",
            4: "cfg4_heat3d_255_M3", 5: "cfg5_advdiff3d_511_M5"}
RESIDUAL_NOTE = ("stop test on the weighted residual ||B_h r||_inf (DESIGN.md reading R15); the paper's unweighted "
                 "||r||_inf = ||W^-1 r~|| is residual_kind 1 (2D only, W-cycles counted apart)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--mode", choices=["isdc", "sdc"], default="isdc")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--extra", type=str, default="3", help="comma-separated extra configs measured in the same run")
    ap.add_argument("--pfasst", type=int, default=4, help="slices of the one-GPU PFASST block in 'extra' (0: off)")
    ap.add_argument("--pfasst-config", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 0)
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def golden_sweeps(cid, seed, mode):
    """Sweeps per step of the whole trajectory recorded by scripts/oracle_golden.py, or None."""
    name = os.path.join(ROOT, "tests", "golden", f"full_cfg{cid}_seed{seed}_{mode}.json")
    try:
        with open(name) as f:
            rec = json.load(f)
        return float(np.mean([s["sweeps"] for s in rec["steps"]])), len(rec["steps"])
    except Exception:
        return None, 0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0])); mx = float(f[1]); pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(sm)}


def replica_seed(seed, rank):
    """Replicas only: rank r solves its own independent problem, seed + r."""
    return seed + rank


def aggregate_ranks(el_ms, steps, world, reduce_max):
    """Whole-job throughput of N independent replicas: every rank ran `steps` steps in `el_ms`
    device milliseconds; the job time is the max over ranks (reduce_max: all-reduce MAX of one
    float).  Returns (max_ms, steps/s of all ranks)."""
    el_max = float(reduce_max(float(el_ms)))
    return el_max, world * steps / (el_max / 1e3)


# ------------------------------------------------------------------------------ the CPU oracle
def oracle_components(cfg, u0, G, mode, which):
    """Time one full-size application of an oracle component on the host cores; returns seconds.
    which: 'rhs' (substep 0 of Eq. 5), 'vcycle' (one V(2,2) cycle of node 0), 'fe' (f^E of one node
    field; 0 when f^E needs no stored field), 'residual' (all nodes)."""
    import oracle
    prob = oracle.Problem(cfg, G, mode=mode)
    M = cfg.M
    state = [u0] * M
    t0 = time.perf_counter()
    if which == "rhs":
        oracle.rhs(prob, 0.0, 0, state, state)
    elif which == "vcycle":
        tau, Q, S, dtau = oracle.tables(M)
        gamma = cfg.nu * (cfg.dt * dtau[0])
        oracle.vcycle(u0, u0, gamma, nu1=cfg.nu1, nu2=cfg.nu2, omega=cfg.omega)
    elif which == "fe":
        if cfg.fe == synth.FE_NONE:
            return 0.0
        oracle.fe_eval(cfg.fe, u0, a=cfg.fe_a, G=G, ct=1.0)
    else:
        oracle.residual(prob, 0.0, state)
    return time.perf_counter() - t0


def compose_step(cfg, t, sweeps_per_step):
    """Oracle seconds per step from component times t: per sweep (M-1) x (RHS + L V-cycles + f^E) +
    residual (the oracle's own loop structure, isdc_oracle.c ora_sweep_state / ora_step)."""
    t_sweep = (cfg.M - 1) * (t["rhs"] + cfg.L * t["vcycle"] + t["fe"]) + t["residual"]
    return t_sweep * sweeps_per_step, t_sweep


def cpu_baseline(cfg, u0, G, mode, sweeps_per_step):
    """The oracle (as it stands) on all host cores, one full-size sample of each component (about
    10-30 s of CPU work), composed into steps/s with the measured sweep count."""
    import oracle
    t = {w: oracle_components(cfg, u0, G, mode, w) for w in ("rhs", "vcycle", "fe", "residual")}
    t_step, t_sweep = compose_step(cfg, t, sweeps_per_step)
    return {"value": 1.0 / t_step, "unit": "steps/s", "cores": oracle.num_threads(), "kind": "oracle",
            "cpu_model": cpu_model(), "extrapolated": True,
            "component_s": t, "sweep_s": t_sweep, "sweeps_per_step": sweeps_per_step,
            "sample": f"one full-size RHS, V(2,2)-cycle, f^E and residual of {WORKLOAD[cfg.cid]} on "
                      f"{oracle.num_threads()} threads; step = {sweeps_per_step:g} sweeps x ((M-1)(RHS + L V-cycles "
                      f"+ f^E) + residual)"}


def run_reference(a):
    """--impl reference: the CPU oracle on the host cores.  Step k times component k mod 4 at full
    size (a bounded sample); the line reports the extrapolated step rate and the real wall time."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t_start = time.perf_counter()
    mode = synth.MODE_SDC if a.mode == "sdc" else synth.MODE_ISDC
    cfg, u0, G = synth.problem_inputs(a.config, a.seed)
    kt, kt_steps = golden_sweeps(a.config, a.seed, a.mode)
    kt_src = "tests/golden (oracle trajectory)"
    if kt is not None and kt_steps < cfg.steps:
        kt_src = f"tests/golden (oracle trajectory, steps 1-{kt_steps} of {cfg.steps})"
    if cfg.fixed_sweeps > 0:
        kt, kt_src = float(cfg.fixed_sweeps), "fixed sweeps per step"
    elif kt is None:
        kt, kt_src = 1.0, "unknown: per-sweep rate"
    comps = ["rhs", "vcycle", "fe", "residual"]
    for i in range(a.warmup):
        oracle_components(cfg, u0, G, mode, comps[i % 4])
    times = {c: [] for c in comps}
    t0 = time.perf_counter()
    for i in range(max(a.steps, 4)):
        c = comps[i % 4]
        times[c].append(oracle_components(cfg, u0, G, mode, c))
    timed_s = time.perf_counter() - t0
    t = {c: float(np.mean(v)) for c, v in times.items()}
    t_step, t_sweep = compose_step(cfg, t, kt)
    cores = oracle.num_threads()
    # single-thread rate: the RHS sample on one thread, against the same sample on all threads
    oracle.set_num_threads(1)
    t1 = oracle_components(cfg, u0, G, mode, "rhs")
    oracle.set_num_threads(cores)
    speedup = t1 / t["rhs"] if t["rhs"] > 0 else None
    val = 1.0 / t_step
    sample = (f"step k = one full-size {{RHS, V(2,2)-cycle, f^E, residual}}[k mod 4] of {WORKLOAD[a.config]} on "
              f"{cores} threads; ms_per_step EXTRAPOLATED = {kt:g} sweeps/step ({kt_src}) x "
              f"((M-1)(RHS + L V-cycles + f^E) + residual)")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[a.config], "seed": a.seed, "mode": a.mode, "residual": RESIDUAL_NOTE},
            "extrapolated": True, "timed_samples_s": timed_s, "wall_s": time.perf_counter() - t_start,
            "component_s": t, "sweep_s": t_sweep, "sweeps_per_step": kt,
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample,
                             "single_thread": {"value": (val / speedup) if speedup else None, "unit": "steps/s",
                                               "rhs_s_1thread": t1, "speedup_all_cores": speedup,
                                               "method": "all-core rate / (1-thread RHS time / all-core RHS time)"}},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ the CUDA path
class Runner:
    """One handle stepping a config's trajectory (restarting from u0 after its last step)."""

    def __init__(self, pk, torch, cid, seed, mode):
        self.torch = torch
        self.cfg, self.u0, G = synth.problem_inputs(cid, seed)
        self.h = pk.ISDC.from_config(self.cfg, None if G is None else torch.from_numpy(G), mode=mode)
        self.u0_dev = torch.from_numpy(self.u0).cuda()
        self.G = G
        self.k = 0

    def step(self):
        if self.k % self.cfg.steps == 0:
            self.h.set_initial(self.u0_dev, 0)
        self.k += 1
        return self.h.step()

    def goto(self, k):
        """Put the trajectory where it was after k steps (deterministic: same bits)."""
        self.k = k - k % self.cfg.steps
        while self.k < k:
            self.step()
        if self.k % self.cfg.steps == 0:
            self.h.set_initial(self.u0_dev, 0)


def measure(pk, torch, a, cid, rank, world, local, barrier, reduce_max, with_e2e, with_cpu, peak, peak_kind):
    mode = synth.MODE_SDC if a.mode == "sdc" else synth.MODE_ISDC
    R = Runner(pk, torch, cid, replica_seed(a.seed, rank), mode)
    cfg, h = R.cfg, R.h
    P = cfg.n ** cfg.dim
    for _ in range(a.warmup):
        R.step()
    k0 = R.k
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    l0 = h.launches
    stream = h.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = [R.step() for _ in range(a.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = h.launches - l0
    el_ms = ev0.elapsed_time(ev1)
    barrier()
    el_max, steps_per_s = aggregate_ranks(el_ms, a.steps, world, reduce_max)
    sweeps = sum(s["sweeps"] for s in stats)
    vcyc = sum(s["vcycles"] for s in stats)
    vcyc_per_s = world * vcyc / (el_max / 1e3)

    # Replay A: the SAME K steps (same starting state, same sweep counts) with CUDA events (on the
    # handle's stream, inside the CUDA graphs) around every launch -> per-class device time and
    # algorithmic bytes; the step's algorithmic GB/s divides those bytes by the event-free timed time.
    R.goto(k0)
    h.profile(2)
    h.profile_reset()
    for _ in range(a.steps):
        R.step()
    prof = h.profile_get()
    h.profile(0)
    alg_bytes = sum(v[2] for v in prof.values())
    tot_ms = sum(v[0] for v in prof.values())
    kernels = {k: {"ms_per_step": v[0] / a.steps, "launches_per_step": v[1] / a.steps,
                   "alg_GBps": (v[2] / (v[0] * 1e-3) / 1e9) if v[0] else None,
                   "share": v[0] / tot_ms if tot_ms else None} for k, v in prof.items()}
    kernels["_note"] = "replay of the K timed steps with events around every launch (shares of the summed event time)"
    # dominant kernel = the class with the largest device time among the fine-level kernels and the
    # residual (each a single kernel at the fine level)
    cands = {k: v for k, v in prof.items() if (k.startswith("fine_") or k == "residual") and v[1] > 0}
    dom = max(cands, key=lambda k: cands[k][0])
    # Replay B: the same K steps with events around the dominant class only (less event overhead)
    R.goto(k0)
    h.profile(16 + pk.PROFILE_CLASS_IDS[dom])
    h.profile_reset()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(a.steps):
        R.step()
    r1.record(stream)
    torch.cuda.synchronize()
    replay_ms = r0.elapsed_time(r1)
    sm_ms, sm_n, sm_b = h.profile_get()[dom]
    h.profile(0)
    achieved = (sm_b / sm_n) / (sm_ms / sm_n * 1e-3) / 1e9 if sm_n else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ent = json.load(f).get(WORKLOAD[cid], {}).get(dom)
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": KERNEL_NAMES.get((cfg.dim, dom), dom), "class": dom,
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "alg_bytes_per_launch": (sm_b / sm_n) if sm_n else None,
                "avg_launch_ms": (sm_ms / sm_n) if sm_n else None, "launches": sm_n,
                "share_of_step": sm_ms / replay_ms if replay_ms else None,
                "measured": "CUDA events around every launch of this class (on the handle's stream) during a replay "
                            "of the K timed steps (%.1f ms/step with the events)" % (replay_ms / a.steps)}
    step_ms = el_ms / a.steps
    line = {
        "value": steps_per_s, "unit": "steps/s", "ms_per_step": el_max / a.steps,
        "config": {"workload": WORKLOAD[cid], "grid": [cfg.n] * cfg.dim, "M": cfg.M, "dt": cfg.dt,
                   "nu": cfg.nu, "L": cfg.L, "mode": a.mode, "seed": a.seed, "trajectory_steps": cfg.steps,
                   "residual": RESIDUAL_NOTE,
                   "l2": "inputs larger than L2 (working set %.2f GB > 126 MB)" % (h.workspace_bytes / 1e9)
                   if h.workspace_bytes > 126e6 else "working set fits in L2 (latency-bound config)",
                   "parallelism": f"replicas{world}"},
        "vcycles_per_s": vcyc_per_s, "sweeps_per_step": sweeps / a.steps, "vcycles_per_step": vcyc / a.steps,
        "point_updates_per_s": vcyc_per_s * P,
        "step_alg_GBps": alg_bytes / a.steps / (step_ms * 1e-3) / 1e9,
        "step_alg_frac_of_peak": alg_bytes / a.steps / (step_ms * 1e-3) / 1e9 / peak,
        "roofline": roofline, "kernels": kernels, "gpu_launches": launches, "clocks": clocks,
        "final_residual": stats[-1]["final_residual"], "converged": all(s["converged"] for s in stats),
    }
    if with_e2e:
        # e2e through the C-ABI with host buffers: every step uploads its input state u_n from pinned
        # host memory and reads u_{n+1} back (the trajectory round-trips through the host; bits equal)
        u_host = torch.from_numpy(R.u0).pin_memory().numpy()
        out_host = torch.empty(R.u0.shape, dtype=torch.float64).pin_memory().numpy()
        k = max(1, min(a.steps, cfg.steps))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(k):
            h.set_initial(u_host if i == 0 else out_host, i)
            h.step()
            h.solution_host(-1, out_host)
        torch.cuda.synchronize()
        el2 = time.perf_counter() - t0
        e2e_s = reduce_max(el2)
        line["e2e"] = {"value": world * k / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": int(R.u0.nbytes),
                       "d2h_bytes_per_step": int(R.u0.nbytes), "steps": k,
                       "note": "wall clock; steps 1..k of the trajectory, each H2D of u_n (pinned) + step + D2H of u_n+1"}
    if with_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, R.u0, R.G, mode, sweeps / a.steps)
    del R, h
    torch.cuda.empty_cache()
    return line


def measure_pfasst(pk, torch, cid, P, seed=0):
    """PFASST (NEXT f4b, R33) on ONE GPU: a block of P time slices of config cid, every slice an
    MLSDC handle on the same stream, scheduled by the product driver's one-GPU transport (the
    slices run one after another).  Reported: the block's device time (CUDA events around the
    block, after an identical warm-up block), its iterations and sweeps, and the same P steps as
    serial single-level ISDC steps for comparison.  `model_p_gpu_ms` is a MODEL, not a measurement:
    the block's critical path on P GPUs = predictor (P coarse stages) + iterations x (one fine sweep
    + P chained coarse sweeps), from the measured per-phase times (transfers not included)."""
    from paper_1401_7824_b200 import pfasst
    cfg, u0, G = synth.problem_inputs(cid, seed)
    Gt = None if G is None else torch.from_numpy(G)
    stream = torch.cuda.current_stream()
    hs = [pk.ISDC.from_config(cfg, Gt, mode=synth.MODE_ISDC, mlsdc_levels=2, coarse_sweeps=1) for _ in range(P)]
    u0d = torch.from_numpy(u0).cuda()
    kw = dict(max_iters=cfg.max_sweeps, fixed_iters=cfg.fixed_sweeps, tol=cfg.sweep_tol, predictor=True)

    def block():
        sl = [pfasst.CudaSlice(hs[p], u0d, p) for p in range(P)]
        return sl, pfasst.run_block_local(sl, **kw)

    block()                                   # warm-up (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sl, out = block()
    e1.record(stream)
    torch.cuda.synchronize()
    blk_ms = e0.elapsed_time(e1)
    it = out[0].iterations
    # per-phase device times on slice P-1 (fine sweep; coarse sweep) for the critical-path model
    h = hs[-1]
    f0, f1, c1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    f0.record(stream); h.sweep(); f1.record(stream)
    h.pfasst_restrict(); h.pfasst_coarse(None); c1.record(stream)
    torch.cuda.synchronize()
    t_fine, t_coarse = f0.elapsed_time(f1), f1.elapsed_time(c1)
    # the same P steps as serial single-level ISDC steps
    hi = pk.ISDC.from_config(cfg, Gt, mode=synth.MODE_ISDC)
    hi.set_initial(u0d, 0); hi.step(); torch.cuda.synchronize()
    hi.set_initial(u0d, 0)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    ser = [hi.step() for _ in range(P)]
    s1.record(stream)
    torch.cuda.synchronize()
    ser_ms = s0.elapsed_time(s1)
    # ... and as serial two-level MLSDC steps (the slice handle's own isdc_step)
    hm = hs[0]
    hm.set_initial(u0d, 0)
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m0.record(stream)
    serm = [hm.step() for _ in range(P)]
    m1.record(stream)
    torch.cuda.synchronize()
    res = {"workload": WORKLOAD[cid], "slices": P, "block_ms_1gpu": blk_ms, "iterations": it,
           "converged": out[0].converged, "fine_sweeps": P * it, "vcycles": sum(o.vcycles for o in out),
           "coarse_vcycles": sum(o.coarse_vcycles for o in out),
           "serial_isdc_ms": ser_ms, "serial_isdc_sweeps": sum(s["sweeps"] for s in ser),
           "serial_mlsdc_ms": m0.elapsed_time(m1), "serial_mlsdc_fine_sweeps": sum(s["sweeps"] for s in serm),
           "serial_mlsdc_coarse_vcycles": sum(s["coarse_vcycles"] for s in serm),
           "fine_sweep_ms": t_fine, "restrict_coarse_ms": t_coarse,
           "model_p_gpu_ms": P * t_coarse + it * (t_fine + P * t_coarse),
           "note": "1 GPU runs the P slices one after another; model_p_gpu_ms is a critical-path MODEL "
                   "(P GPUs, transfers excluded), not a measurement"}
    del sl, hs, hi
    torch.cuda.empty_cache()
    return res


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_1401_7824_b200 as pk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    peak, peak_kind = peaks()
    main_line = measure(pk, torch, a, a.config, rank, world, local, barrier, reduce_max, not a.no_e2e,
                        rank == 0 and world == 1 and not a.no_cpu_baseline, peak, peak_kind)
    extra = {}
    for c in [int(x) for x in a.extra.split(",") if x.strip()]:
        if c == a.config:
            continue
        ln = measure(pk, torch, a, c, rank, world, local, barrier, reduce_max, False, False, peak, peak_kind)
        extra[WORKLOAD[c]] = {k: ln[k] for k in ("value", "unit", "ms_per_step", "vcycles_per_s", "sweeps_per_step",
                                                 "vcycles_per_step", "point_updates_per_s", "step_alg_GBps",
                                                 "step_alg_frac_of_peak", "roofline", "kernels", "clocks",
                                                 "gpu_launches", "config")}
    if a.pfasst > 1 and world == 1:
        extra["pfasst"] = measure_pfasst(pk, torch, a.pfasst_config, a.pfasst)
    if rank == 0:
        line = {"metric": METRIC, "value": main_line["value"], "unit": "steps/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": main_line["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
        line.update({k: v for k, v in main_line.items() if k not in line})
        if extra:
            line["extra"] = extra
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
