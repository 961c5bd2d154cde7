#!/usr/bin/env python3
"""ISDC hot-path benchmark (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--mode isdc|sdc] [--impl ours|reference]

A "step" is one ISDC time step of the BASELINE.json config (default config 3: 2D heat with
forcing, 4095^2, M = 5, sweeps until ||r~|| < 1e-10, 2 V(2,2)-cycles per node solve), i.e. every
row of SURVEY.md §8(a) over one batch of synthetic input.  Multi-step configs (2: 10 steps,
5: 5 steps) advance their trajectory and restart from u0 after their last step.

N > 1 (torchrun): replicas -- every rank runs its own independent problem on its own GPU with no
collective on the data path ("replicas only"); value = all ranks' steps / max time.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the host cores on a
bounded sample (one full-size sweep + residual per "step"), extrapolated to steps/s with the
config's sweep count per step.
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

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "ISDC steps/s + V-cycles/s (fp64, 1 B200); HBM GB/s as fraction of ~8 TB/s peak"
# fine-level kernel classes (isdc_profile classes 0-2) -> the kernel that implements them
KERNEL_NAMES = {
    (2, "fine_defect_restrict"): "f2d::k_smooth2r: 2 Jacobi sweeps + defect + full weighting (26 B/pt)",
    (2, "fine_prolong_correct"): "f2d::k_smooth2<MODE 2>: bilinear prolongation + correction + 2 Jacobi sweeps (26 B/pt)",
    (2, "fine_smoother"): "f2d::k_smooth2: 2 Jacobi sweeps (24 B/pt)",
    (3, "fine_smoother"): "f3d::k_smooth2: 2 Jacobi sweeps, z-streaming (24 B/pt)",
    (3, "fine_defect_restrict"): "f3d::k_restrict: defect + full weighting (17 B/pt)",
    (3, "fine_prolong_correct"): "f3d::k_prolong: trilinear prolongation + correction (17 B/pt)",
}
WORKLOAD = {1: "cfg1_heat2d_63_M3", 2: "cfg2_allencahn2d_1023_M5", 3: "cfg3_forced_heat2d_4095_M5",
            4: "cfg4_heat3d_255_M3", 5: "cfg5_advdiff3d_511_M5"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--mode", choices=["isdc", "sdc"], default="isdc")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def golden_sweeps(cid, seed, mode):
    """Sweeps per step recorded by scripts/oracle_golden.py (oracle-only), or None."""
    name = os.path.join(ROOT, "tests", "golden", f"full_cfg{cid}_seed{seed}_{mode}.json")
    try:
        with open(name) as f:
            rec = json.load(f)
        return float(np.mean([s["sweeps"] for s in rec["steps"]]))
    except Exception:
        return None


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
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0])); mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def replica_seed(seed, rank):
    """Replicas only: rank r solves its own independent problem, seed + r."""
    return seed + rank


def aggregate_ranks(el_ms, steps, world, reduce_max):
    """Whole-job throughput of N independent replicas: every rank ran `steps` steps in `el_ms`
    device milliseconds; the job time is the max over ranks (reduce_max: all-reduce MAX of one
    float).  Returns (max_ms, steps/s of all ranks)."""
    el_max = float(reduce_max(float(el_ms)))
    return el_max, world * steps / (el_max / 1e3)


def cpu_baseline(cfg, u0, G, mode, sweeps_per_step, reps=1):
    """Time the oracle (as it stands) on this host: `reps` full-size sweeps + residual."""
    import oracle
    prob = oracle.Problem(cfg, G, mode=mode)
    state = [u0] * cfg.M
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        state, _ = oracle.sweep(prob, 0.0, state)
        oracle.residual(prob, 0.0, state)
        times.append(time.perf_counter() - t0)
    t_sweep = float(np.mean(times))
    return {"value": 1.0 / (t_sweep * sweeps_per_step), "unit": "steps/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{reps} full-size sweep(s) + residual of {WORKLOAD[cfg.cid]} ({t_sweep:.2f} s each); "
                      f"steps/s = 1/(t_sweep * {sweeps_per_step:g} sweeps per step)"}


def run_reference(a):
    """--impl reference: the CPU oracle on host cores, bounded sample per step."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mode = synth.MODE_SDC if a.mode == "sdc" else synth.MODE_ISDC
    cfg, u0, G = synth.problem_inputs(a.config, a.seed)
    kt = golden_sweeps(a.config, a.seed, a.mode)
    kt_src = "tests/golden (oracle)"
    if kt is None:
        kt, kt_src = 1.0, "unknown (per-sweep rate)"
    prob = oracle.Problem(cfg, G, mode=mode)
    state = [u0] * cfg.M
    for _ in range(a.warmup):
        state, _ = oracle.sweep(prob, 0.0, state)
        oracle.residual(prob, 0.0, state)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        state, _ = oracle.sweep(prob, 0.0, state)
        oracle.residual(prob, 0.0, state)
    el = time.perf_counter() - t0
    t_sweep = el / a.steps
    val = 1.0 / (t_sweep * kt)
    sample = (f"each step = 1 full-size sweep + residual of {WORKLOAD[a.config]} ({t_sweep:.2f} s); "
              f"steps/s = 1/(t_sweep * {kt:g} sweeps per step, from {kt_src})")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t_sweep * kt, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[a.config], "seed": a.seed, "mode": a.mode},
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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

    mode = synth.MODE_SDC if a.mode == "sdc" else synth.MODE_ISDC
    cfg, u0, G = synth.problem_inputs(a.config, replica_seed(a.seed, rank))
    h = pk.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=mode)
    u0_dev = torch.from_numpy(u0).cuda()
    P = cfg.n ** cfg.dim
    state = {"k": 0}

    def one_step():
        if state["k"] % cfg.steps == 0:
            h.set_initial(u0_dev, 0)
        state["k"] += 1
        return h.step()

    for _ in range(a.warmup):
        one_step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    l0 = h.launches
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = [one_step() for _ in range(a.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = h.launches - l0
    el_ms = ev0.elapsed_time(ev1)
    barrier()

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    el_max, steps_per_s = aggregate_ranks(el_ms, a.steps, world, reduce_max)
    sweeps = sum(s["sweeps"] for s in stats)
    vcyc = sum(s["vcycles"] for s in stats)
    vcyc_per_s = world * vcyc / (el_max / 1e3)
    peak, peak_kind = peaks()

    # Dominant kernel (roofline): the fine-level kernel class with the largest device time in one
    # step with events around every fine-level launch; then the same K steps are replayed from the
    # same state with CUDA events (on the handle's stream, inside the CUDA graphs) around that
    # class only.  The events cost graph throughput, so `value` comes from the event-free timed
    # region above and the kernel average from this replay.
    h.profile(1)
    h.profile_reset()
    state["k"] = 0
    one_step()
    pre = {k: v for k, v in h.profile_get().items() if k.startswith("fine_") and v[1] > 0}
    dom = max(pre, key=lambda k: pre[k][0])
    h.profile(16 + pk.PROFILE_CLASS_IDS[dom])
    h.profile_reset()
    state["k"] = a.warmup
    if state["k"] % cfg.steps:
        h.set_initial(u0_dev, 0)
        for _ in range(state["k"] % cfg.steps):
            h.step()
        h.profile_reset()
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(a.steps):
        one_step()
    r1.record(stream)
    torch.cuda.synchronize()
    replay_ms = r0.elapsed_time(r1)
    prof_timed = h.profile_get()
    h.profile(0)
    sm_ms, sm_n, sm_b = prof_timed[dom]
    achieved = (sm_b / sm_n) / (sm_ms / sm_n * 1e-3) / 1e9 if sm_n else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        ent = tr.get(WORKLOAD[a.config], {})
        if ent.get("class") == dom:
            traffic = ent.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": KERNEL_NAMES.get((cfg.dim, dom), dom), "class": dom,
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "alg_bytes_per_launch": (sm_b / sm_n) if sm_n else None,
                "avg_launch_ms": (sm_ms / sm_n) if sm_n else None, "launches": sm_n,
                "share_of_step": sm_ms / replay_ms if replay_ms else None,
                "measured": "CUDA events around every launch of this class during a replay of the K timed "
                            "steps (%.1f ms/step with the events)" % (replay_ms / a.steps),
                "fine_classes_one_step": {k: {"ms": v[0], "launches": v[1]} for k, v in pre.items()}}
    # per-class breakdown: one extra (untimed) step with events around every launch
    h.profile(2)
    h.profile_reset()
    state["k"] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    br_ms = e0.elapsed_time(e1)
    prof = h.profile_get()
    h.profile(0)
    alg_bytes = sum(v[2] for v in prof.values())
    kernels = {k: {"ms": v[0], "launches": v[1], "alg_GBps": (v[2] / (v[0] * 1e-3) / 1e9) if v[0] else None,
                   "share": v[0] / br_ms} for k, v in prof.items()}
    kernels["_note"] = "from one extra step with events around every launch (%.1f ms incl. event overhead)" % br_ms

    # e2e: through the C-ABI with host buffers (H2D of u0 and D2H of u_M inside the timed region)
    e2e = None
    if not a.no_e2e:
        u0_host = torch.from_numpy(u0).pin_memory().numpy()
        out_host = torch.empty(u0.shape, dtype=torch.float64).pin_memory().numpy()
        k = max(1, min(a.steps, 3))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(k):
            h.set_initial(u0_host, 0)
            h.step()
            h.solution_host(-1, out_host)
        torch.cuda.synchronize()
        el2 = time.perf_counter() - t0
        t2 = torch.tensor([el2], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e = {"value": world * k / float(t2.item()), "unit": "steps/s", "h2d_bytes_per_step": int(u0.nbytes),
               "d2h_bytes_per_step": int(u0.nbytes), "steps": k, "note": "restarts from u0 each step"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(cfg, u0, G, mode, sweeps / a.steps)

    if rank == 0:
        line = {
            "metric": METRIC, "value": steps_per_s, "unit": "steps/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": el_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[a.config], "grid": [cfg.n] * cfg.dim, "M": cfg.M, "dt": cfg.dt,
                       "nu": cfg.nu, "L": cfg.L, "mode": a.mode, "seed": a.seed,
                       "l2": "inputs larger than L2 (working set %.2f GB > 126 MB)" % (h.workspace_bytes / 1e9)
                       if h.workspace_bytes > 126e6 else "working set fits in L2 (latency-bound config)",
                       "parallelism": f"replicas{world}"},
            "vcycles_per_s": vcyc_per_s, "sweeps_per_step": sweeps / a.steps, "vcycles_per_step": vcyc / a.steps,
            "point_updates_per_s": vcyc_per_s * P,
            "step_alg_GBps": alg_bytes / (el_ms / a.steps * 1e-3) / 1e9,
            "step_alg_frac_of_peak": alg_bytes / (el_ms / a.steps * 1e-3) / 1e9 / peak,
            "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "final_residual": stats[-1]["final_residual"],
            "converged": all(s["converged"] for s in stats),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
