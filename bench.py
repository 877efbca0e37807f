"""Benchmark of the B200 hot path (BASELINE config 2 by default).

A "step" = one F(u), one J(u)v and one J(u)^T w apply over the full config-2
field (E = 2^22 elements, N = 7, 29,360,128 DOF, fp64), inputs resident in
HBM.  value = 3 * DOF / step time ("apply-DOF/s" summed over the three
operators).  Each field is 235 MB, larger than the 126 MB L2, so no flush is
needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (stock semopt 0.1.0,
installed unmodified into baseline/_ref) on the host cores, on the same full
config-2 step.
Under torchrun (N > 1) the ranks share ONE periodic ring of N * 2^22 elements,
element-sharded (dist.py): every operator input gets a ghost-node exchange with
the two neighbouring ranks over NCCL (weak scaling); timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_DOF = {"F": 16, "J": 24, "JT": 24}
# BASELINE.json "metric", verbatim.  `value` is the config-2 step (F(u), J(u)v, J(u)^T w once
# each, BASELINE configs[1]) as 3 * DOF / step time; per_op reports F and J^T alone, roofline
# the % of HBM bandwidth, ratios the adjoint/forward cost ratios.
METRIC = "fp64 DOF/s for F(u) and J^T\u00b7w apply; % HBM roofline; adjoint/forward cost ratio"
VALUE_DEF = "3 * DOF / time of one config-2 step (F(u), J(u)v and J(u)^T w once each)"


def flop_per_dof(N, op):
    n = N + 1
    per_elem = 4 * n * n + 3 * n + N + 1 if op == "F" else 6 * n * n + 5 * n + N + 1
    return per_elem / N


def executed_flop_per_dof(N, op):
    """FP64 work the reflection-split kernels execute for n = N + 1 a multiple of 16 (plain applies,
    sem1d_device.cuh WS_EO): every n x n product runs as two (n/2) x (n/2) products on the sums and
    differences of mirrored nodes, n^2 flops instead of 2 n^2, plus n adds to form them and n to
    recombine the rows."""
    n = N + 1
    per_elem = (2 * n * n + 4 * n) + 3 * n + N + 1 if op == "F" else (3 * n * n + 7 * n) + 5 * n + N + 1
    return per_elem / N


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--sweep-steps", type=int, default=64)
    p.add_argument("--no-cfg5", action="store_true")
    p.add_argument("--cfg5-steps", type=int, default=8)
    # test-only: exercise the sharded path with every rank on cuda:0 and a gloo exchange
    # (safe on one GPU: no kernel waits on another rank)
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    p.add_argument("--same-device", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU arm


def cpu_reference_step_sample(E_sample, reps, seed):
    """Time the reference algorithm (oracle port) on E_sample elements of config 2."""
    import numpy as np

    from oracle import semref as R
    from paper_1806_01422_b200 import configs

    c = configs.CFG2
    h = (c["xb"] - c["xa"]) / c["E"]
    mesh = R.Mesh1D(0.0, E_sample * h, E_sample, c["N"], True)   # same h, N, nu as config 2
    op = R.BurgersOracle(mesh, c["nu"])
    u, v, w = configs.operator_inputs(mesh.ndof, seed)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        op.rhs(u)
        op.jac(u, v)
        op.jact(u, w)
        times.append(time.perf_counter() - t0)
    del np
    return mesh.ndof, times


def workload_config(world):
    """The `config` object shared by both arms (same workload, same keys)."""
    from paper_1806_01422_b200 import configs
    c = configs.CFG2
    return {"workload": "BASELINE config 2: 1D Burgers, E=2^22, N=7, nu=0.01, periodic [-1,1]",
            "value": VALUE_DEF, "E": c["E"], "N": c["N"], "dof": c["E"] * c["N"],
            "l2": "inputs 235 MB/field > 126 MB L2, no flush",
            "parallelism": "single GPU" if world == 1 else
            f"x{world} independent config-2 replicas at N=1's size + strong-scaled config-5 sweep (see scaling)"}


REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def import_stock_reference():
    """The unmodified reference package (semopt 0.1.0), installed into baseline/_ref by
    `pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of
    /root/reference/pkg>`.  Returns None when it is absent."""
    if not os.path.isdir(os.path.join(REF_PATH, "semopt")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import semopt.grid
    import semopt.ops
    return semopt


def run_reference_arm(args):
    """The reference's own CPU path, timed on the host cores: stock semopt
    SemOperator.apply_rhs / apply_jacobian / apply_jacobian_transpose (ops.py:232-257) on the
    FULL config-2 field, numpy/OpenBLAS with every host thread.  Falls back to the
    bit-identical numpy port (oracle/semref.py) only if baseline/_ref is missing."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from paper_1806_01422_b200 import configs
    c = configs.CFG2
    semopt = import_stock_reference()
    cores = host_cores()
    u = v = w = None
    if semopt is not None:
        g = semopt.grid.grid_1d(c["xa"], c["xb"], c["E"], c["N"])
        op = semopt.ops.SemOperator(g, semopt.ops.PdeCoefficients(c["nu"]))
        ndof = g.nglobal
        kind, what = "reference", "stock semopt 0.1.0 from baseline/_ref (ops.py:232-257)"
        f_rhs, f_jac, f_jact = op.apply_rhs, op.apply_jacobian, op.apply_jacobian_transpose
    else:
        from oracle import semref as R
        op = R.BurgersOracle(R.Mesh1D(c["xa"], c["xb"], c["E"], c["N"], True), c["nu"])
        ndof = op.mesh.ndof
        kind, what = "port", "numpy port of semopt ops.py (oracle/semref.py; baseline/_ref absent)"
        f_rhs, f_jac, f_jact = op.rhs, op.jac, op.jact
    u, v, w = configs.operator_inputs(ndof, c["seed"])
    times = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        f_rhs(u)
        f_jac(u, v)
        f_jact(u, w)
        times.append(time.perf_counter() - t0)
    timed = times[args.warmup:]
    total = sum(timed)
    value = 3 * ndof * len(timed) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded u~U(-1,1), v,w~N(0,1) per node)",
        "config": workload_config(1),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores, "kind": kind,
                         "sample": f"the full config-2 step (F+J+J^T once each on all {ndof} DOF), "
                                   f"{what}, numpy {np.__version__} / OpenBLAS, {cores} host threads"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover - depends on the box
            self.nvml = None
            self.err = str(exc)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # pragma: no cover
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nvml is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- GPU arm


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return {}


def timed_ops(op, ud, vd, wd, outs, steps, stream, per_launch=True):
    """Run `steps` steps of (F, J, J^T) on the launching stream.  per_launch: CUDA events
    around every launch (per-kernel durations for the roofline); otherwise only around the
    whole region, so consecutive launches keep their programmatic-dependent-launch overlap
    (an event between two kernels serialises them)."""
    import torch
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    sharded = hasattr(op, "refresh")
    if not per_launch:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for s in range(steps):
                if sharded:
                    op.refresh([ud, vd, wd])
                    op.launch_rhs(ud, outs[0], refresh=False)
                    op.launch_jac(ud, vd, outs[1], refresh=False)
                    op.launch_jact(ud, wd, outs[2], refresh=False)
                else:
                    op.launch_rhs(ud, outs[0])
                    op.launch_jac(ud, vd, outs[1])
                    op.launch_jact(ud, wd, outs[2])
            ev1.record(stream)
        stream.synchronize()
        return ev0.elapsed_time(ev1), None
    with torch.cuda.stream(stream):
        for s in range(steps):
            e = ev[s]
            e[0].record(stream)
            if sharded:          # one batched ghost exchange of the step's inputs u, v, w
                op.refresh([ud, vd, wd])
                op.launch_rhs(ud, outs[0], refresh=False)
            else:
                op.launch_rhs(ud, outs[0])
            e[1].record(stream)
            if sharded:
                op.launch_jac(ud, vd, outs[1], refresh=False)
            else:
                op.launch_jac(ud, vd, outs[1])
            e[2].record(stream)
            if sharded:
                op.launch_jact(ud, wd, outs[2], refresh=False)
            else:
                op.launch_jact(ud, wd, outs[2])
            e[3].record(stream)
    stream.synchronize()
    per = {"F": [], "J": [], "JT": []}
    for e in ev:
        per["F"].append(e[0].elapsed_time(e[1]))
        per["J"].append(e[1].elapsed_time(e[2]))
        per["JT"].append(e[2].elapsed_time(e[3]))
    total = ev[0][0].elapsed_time(ev[-1][3])
    return total, per


def sweep_ratio(op, torch, steps=8):
    """Forward RK4 sweep vs discrete-adjoint sweep on the config-2 field (store-all), with the
    stage states held in HBM (what evaluate() does when they fit) and with the reference's
    stage recompute.  h = 4.8e-7 on config 2 makes the explicit limit ~5e-14 (rho*h^2 ~ 13
    at nu=0.01), so dt = 1e-14: this measures cost, not physics."""
    from paper_1806_01422_b200 import adjoint, checkpoint, timeloop
    dt = 1e-14
    ts = timeloop.TsConfig(scheme="rk4", t0=0.0, t_end=steps * dt, dt=dt)
    u0 = torch.sin(torch.linspace(0, 6.283185307179586, op.ndof, dtype=torch.float64,
                                  device=op.device))

    def one(keep):
        fw = timeloop.integrate(op, u0, ts, keep_stages=keep)   # warm-up (allocations)
        _, lam = adjoint.terminal_condition(op.grid, fw.u_final, 0.5 * u0, op=op)
        adjoint.sweep(op, ts, fw, checkpoint.plan_store_all(fw.n_steps), lam)
        del fw, lam
        torch.cuda.synchronize()
        a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        a.record()
        fwd = timeloop.integrate(op, u0, ts, keep_stages=keep)
        b.record()
        sched = checkpoint.plan_store_all(fwd.n_steps)
        _, lam = adjoint.terminal_condition(op.grid, fwd.u_final, 0.5 * u0, op=op)
        c.record()
        adjoint.sweep(op, ts, fwd, sched, lam)
        d.record()
        torch.cuda.synchronize()
        del fwd, lam
        return a.elapsed_time(b), c.elapsed_time(d)

    f_ms, a_ms = one(True)
    fr_ms, ar_ms = one(False)
    return {"scheme": "rk4", "steps": steps, "forward_ms": f_ms, "adjoint_ms": a_ms,
            "adjoint_over_forward": a_ms / f_ms, "ms_per_forward_step": f_ms / steps,
            "ms_per_adjoint_step": a_ms / steps,
            "stage_states": "held in HBM by the forward step (no adjoint recompute)",
            "recompute": {"forward_ms": fr_ms, "adjoint_ms": ar_ms, "adjoint_over_forward": ar_ms / fr_ms,
                          "ms_per_forward_step": fr_ms / steps, "ms_per_adjoint_step": ar_ms / steps},
            "kernels": "one temporally blocked launch per RK4 step and per adjoint step"
                       if getattr(op, "step_fused_supported", lambda: False)() else "per-stage"}


FP64_PEAK_TFS = 36.98   # measured DMMA m8n8k4 f64 peak on this pool's B200 (profiles/r1_dmma_chains.jsonl)
# whole-step kernels, per DOF of the ring: FP64 work (reference flop counts)
# and algorithmic HBM bytes (each input read once, each output written once)
STEP_BYTES = {"fwd": 16, "fwd_st": 40, "adj": 24, "adj_st": 48}


def step_flops(kind, N=7):
    f, j = flop_per_dof(N, "F"), flop_per_dof(N, "J")
    return {"fwd": 4 * f, "fwd_st": 4 * f, "adj": 3 * f + 4 * j, "adj_st": 4 * j}[kind]


def roofline_entry(us, flops_per_dof, bytes_per_dof, dof, hbm_gbs):
    t_flop = flops_per_dof * dof / (FP64_PEAK_TFS * 1e12) * 1e6
    t_byte = bytes_per_dof * dof / (hbm_gbs * 1e9) * 1e6
    bound = "fp64" if t_flop >= t_byte else "hbm"
    return {"us": us, "fp64_tflops": flops_per_dof * dof / (us * 1e-6) / 1e12,
            "achieved_gbs": bytes_per_dof * dof / (us * 1e-6) / 1e9, "bound": bound,
            "roofline_us": max(t_flop, t_byte), "frac": max(t_flop, t_byte) / us}


def tile_kernel_times(op, torch, hbm_gbs, reps=20):
    """The RK4 whole-step kernels on the config-2 field, CUDA events around `reps`
    back-to-back launches on the launching stream: forward step (run-ahead form), forward
    step writing its stage states, adjoint step with stage recompute, adjoint step reading
    the stored stages.  Roofline = the slower of FP64 work at the measured DMMA peak and
    algorithmic bytes at the measured HBM bandwidth."""
    if not getattr(op, "step_fused_supported", lambda: False)():
        return None
    u = torch.sin(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device=op.device))
    lam = torch.cos(torch.linspace(0, 50, op.ndof, dtype=torch.float64, device=op.device))
    o = op.empty()
    st = [op.empty() for _ in range(3)]
    slot = op.flag_slots(1)
    dt = 1e-14
    # every kernel in the form the run-ahead integrate / sweep launches it (per-step flag word,
    # outputs-only check; a flagged step is re-run with the classifying check)
    runs = {"fwd": lambda: op.launch_rk_step(u, o, dt, "rk4", flag=slot.data_ptr()),
            "fwd_st": lambda: op.launch_rk_step_stages(u, o, st, dt, "rk4", flag=slot.data_ptr()),
            "adj": lambda: op.launch_adj_step(u, lam, o, dt, "rk4", flag=slot.data_ptr()),
            "adj_st": lambda: op.launch_adj_step_stages(u, st, lam, o, dt, "rk4", flag=slot.data_ptr())}
    out = {}
    for k, fn in runs.items():
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        us = 1e3 * a.elapsed_time(b) / reps
        out[k] = roofline_entry(us, step_flops(k), STEP_BYTES[k], op.ndof, hbm_gbs)
    if op.flags() or int(slot[0]):
        raise RuntimeError("non-finite flag in the tile-kernel timing")
    del u, lam, o, st
    return out


def graph_us(torch, fn, reps):
    """Average time of `reps` launches captured in one CUDA graph and replayed (no host
    launch path between kernels; best of 5 replays)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, 1e3 * a.elapsed_time(b) / reps)
    del g
    return best


def cfg3_ops(torch, dev, hbm_gbs, reps=20):
    """BASELINE config 3 (E = 2^18, N = 31, nu = 1e-3): F, J v, J^T w per launch (CUDA events
    around each launch).  frac_of_dmma_peak counts the reference algorithm's flops
    against the measured DMMA peak; the kernels run the reflection split, which executes about
    half of them (executed_fp64_tflops), so the roofline is the slower of the executed FP64 work
    at the DMMA peak and the algorithmic bytes at the measured HBM bandwidth."""
    from paper_1806_01422_b200 import configs
    c = configs.CFG3
    op = configs.cfg_operator(c, device=dev)
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    ud, vd, wd = (torch.from_numpy(a).to(dev) for a in (u, v, w))
    o = op.empty()
    runs = {"F": lambda: op.launch_rhs(ud, o), "J": lambda: op.launch_jac(ud, vd, o),
            "JT": lambda: op.launch_jact(ud, wd, o)}
    out = {}
    for k, fn in runs.items():
        for _ in range(3):
            fn()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        for r in range(reps):
            ev[2 * r].record()
            fn()
            ev[2 * r + 1].record()
        torch.cuda.synchronize()
        us = 1e3 * sum(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps)) / reps
        ev[0].record()                          # back to back (PDL overlap kept), events at the ends
        for r in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        us_b2b = 1e3 * ev[0].elapsed_time(ev[1]) / reps
        us_graph = graph_us(torch, fn, reps)
        fl = flop_per_dof(c["N"], "F" if k == "F" else "J") * op.ndof
        fx = executed_flop_per_dof(c["N"], "F" if k == "F" else "J") * op.ndof
        by = (16 if k == "F" else 24) * op.ndof
        t_roof = max(fx / (FP64_PEAK_TFS * 1e12), by / (hbm_gbs * 1e9)) * 1e6
        out[k] = {"us": us, "fp64_tflops": fl / (us * 1e-6) / 1e12,
                  "executed_fp64_tflops": fx / (us_b2b * 1e-6) / 1e12,
                  "achieved_gbs": by / (us_b2b * 1e-6) / 1e9, "hbm_frac": by / (us_b2b * 1e-6) / 1e9 / hbm_gbs,
                  "roofline_us": t_roof, "bound": "fp64" if fx / (FP64_PEAK_TFS * 1e12) >= by / (hbm_gbs * 1e9) else "hbm",
                  "frac_roofline_back_to_back": t_roof / us_b2b,
                  "frac_of_dmma_peak": fl / (us * 1e-6) / 1e12 / FP64_PEAK_TFS,
                  "us_back_to_back": us_b2b, "frac_back_to_back": fl / (us_b2b * 1e-6) / 1e12 / FP64_PEAK_TFS,
                  "us_graph": us_graph, "frac_graph": fl / (us_graph * 1e-6) / 1e12 / FP64_PEAK_TFS}
    if op.flags():
        raise RuntimeError("non-finite flag in config 3")
    return {"workload": "BASELINE config 3: E=2^18, N=31, nu=1e-3, periodic [-1,1]", "dof": op.ndof,
            "fp64_peak_tflops": FP64_PEAK_TFS, "algorithm": "reflection (even/odd) split of K, Dw, Dw^T: "
            "half the DMMAs of the full-matrix products", "per_op": out}


def cfg5_sweep(torch, dist, world, rank, dev, steps, backend="nccl"):
    """BASELINE config 5's ring (E = 2^25, N = 7, h = 1/64, nu = 1e-3, 234,881,024 DOF),
    strong-scaled: the same global ring at every N, `steps` fused RK4 forward steps then
    `steps` fused adjoint steps (stage recompute, as the binomial-checkpointed gradient runs
    them), dt = 2e-4, smooth 32-mode u0.  Sharded (N > 1): contiguous element blocks, 8-element
    ghost zones, one NCCL halo exchange per step overlapped with the interior tiles.
    Times on the device (CUDA events), max over ranks."""
    from paper_1806_01422_b200 import configs
    from paper_1806_01422_b200 import dist as sd
    from paper_1806_01422_b200.grid import grid_1d
    from paper_1806_01422_b200.ops import PdeCoefficients, SemOperator
    c = configs.CFG5
    E = c["E"]
    g = grid_1d(0.0, E * c["h"], E, c["N"])
    if world == 1:
        op = SemOperator(g, PdeCoefficients(c["nu"]), device=dev)
        u0 = configs.fourier_field_device(g, c["modes"], c["seed"], dev) / 8.0
        lam0 = configs.fourier_field_device(g, c["modes"], c["seed"] + 1, dev)
    else:
        op = sd.ShardedOperator(g, PdeCoefficients(c["nu"]), rank, world, device=dev)
        sl = slice(op.part.g_lo, op.part.g_lo + op.part.n_own)
        u0 = op.field((configs.fourier_field_device(g, c["modes"], c["seed"], dev) / 8.0)[sl].contiguous())[0]
        lam0 = op.field(configs.fourier_field_device(g, c["modes"], c["seed"] + 1, dev)[sl].contiguous())[0]
    dt = c["dt"]
    states = [u0] + [op.empty() for _ in range(steps)]
    lam = [lam0.clone(), op.empty()]
    # the forward steps in the form the gradient's run-ahead integrate launches them: each
    # step ORs into a flag word and checks only its new state (timeloop.integrate)
    slot = op.flag_slots(1)

    def run(k):
        for i in range(k):
            op.launch_rk_step(states[i], states[i + 1], dt, "rk4", flag=slot.data_ptr())
        f1 = torch.cuda.Event(enable_timing=True)
        f1.record()
        for i in range(k - 1, -1, -1):
            op.launch_adj_step(states[i], lam[0], lam[1], dt, "rk4", flag=slot.data_ptr())
            lam.reverse()
        return f1

    run(1)                                       # warm-up (allocations, first launches)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    mid = run(steps)
    z.record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(mid), mid.elapsed_time(z)]
    if world > 1:
        tt = torch.tensor(t, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.tolist()
    if op.flags() or int(slot[0]):
        raise RuntimeError("non-finite flag in the config-5 sweep")
    dof = E * c["N"]
    del states, lam, u0, lam0
    return {"n_gpus": world, "E": E, "dof": dof, "steps": steps, "forward_ms": t[0], "adjoint_ms": t[1],
            "ms_per_step_pair": (t[0] + t[1]) / steps,
            "dof_steps_per_s": 2 * dof * steps / ((t[0] + t[1]) * 1e-3),
            "forward_dof_per_s": dof * steps / (t[0] * 1e-3), "adjoint_dof_per_s": dof * steps / (t[1] * 1e-3)}


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1806_01422_b200 import configs

    rank, world, local = dist_env()
    if args.same_device:
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")      # communicator ranks in the log
        dist.init_process_group(args.dist_backend)
        print(f"[bench] rank {rank}/{world} local_rank {local} device {torch.cuda.get_device_name(local)} "
              f"backend {dist.get_backend()}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    c = configs.CFG2
    if world == 1:
        op = configs.cfg_operator(c, device=dev)
        ndof = op.ndof
        u, v, w = configs.operator_inputs(ndof, c["seed"])
        ud, vd, wd = (torch.from_numpy(a).to(dev) for a in (u, v, w))
    else:
        # element-sharded weak scaling: one periodic ring of world * 2^22 elements, each
        # rank owns 2^22 of them and exchanges ghost nodes with its two neighbours (NCCL)
        from paper_1806_01422_b200 import dist as sd
        from paper_1806_01422_b200.grid import grid_1d
        from paper_1806_01422_b200.ops import PdeCoefficients
        h = (c["xb"] - c["xa"]) / c["E"]
        g = grid_1d(c["xa"], c["xa"] + world * c["E"] * h, world * c["E"], c["N"])
        op = sd.ShardedOperator(g, PdeCoefficients(c["nu"]), rank, world, device=dev)
        ndof = op.part.n_own
        u, v, w = configs.operator_inputs(ndof, c["seed"] + rank)
        ud, vd, wd = (op.field(torch.from_numpy(a).to(dev))[0] for a in (u, v, w))
    op.sync_checks = False
    outs = [op.empty() for _ in range(3)]
    stream = torch.cuda.current_stream(dev)

    # warm-up
    timed_ops(op, ud, vd, wd, outs, max(1, args.warmup), stream)
    if op.flags():
        raise RuntimeError("non-finite flag raised on config-2 inputs")

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        # the timed region: K steps back to back, events only at its ends
        total_ms, _ = timed_ops(op, ud, vd, wd, outs, args.steps, stream, per_launch=False)
        torch.cuda.synchronize()
        # per-kernel durations for the roofline: a second pass of K steps with an event
        # around every launch (which serialises consecutive launches)
        _, per = timed_ops(op, ud, vd, wd, outs, args.steps, stream)
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([total_ms], device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_step = total_ms / args.steps
    value = 3 * ndof * world / (ms_step * 1e-3)

    # e2e through the public API with pinned host buffers, copies inside the timed region
    uh, vh, wh = (torch.from_numpy(a).pin_memory() for a in (u, v, w))
    oh = [torch.empty(ndof, dtype=torch.float64).pin_memory() for _ in range(3)]
    e2e_steps = max(2, min(5, args.steps))

    streaming = world == 1 and hasattr(op, "apply_host")

    def e2e_step():
        if streaming:
            # public streaming API: element-chunked H2D / kernels / D2H overlap
            op.apply_host(uh, vh, wh, out={"rhs": oh[0], "jac": oh[1], "jact": oh[2]})
            return
        du = uh.to(dev, non_blocking=True)
        dv = vh.to(dev, non_blocking=True)
        dw = wh.to(dev, non_blocking=True)
        f = op.apply_rhs(du)
        jv = op.apply_jacobian(du, dv)
        jt = op.apply_jacobian_transpose(du, dw)
        oh[0].copy_(f, non_blocking=True)
        oh[1].copy_(jv, non_blocking=True)
        oh[2].copy_(jt, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(e2e_steps):
        e2e_step()
    s1.record()
    torch.cuda.synchronize()
    e2e_ms = s0.elapsed_time(s1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = 3 * ndof * world / (e2e_ms * 1e-3)
    if op.flags():
        raise RuntimeError("non-finite flag raised in e2e")

    sweep = tiles = cfg3 = dropin = None
    if not args.no_sweep and world == 1:
        sweep = sweep_ratio(op, torch, steps=args.sweep_steps)
        tiles = tile_kernel_times(op, torch, load_peaks()[0])
        # the drop-in as a semopt user calls it: numpy in, numpy out, three serial applies
        hu, hv, hw = u, v, w
        op.apply_rhs(hu)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            op.apply_rhs(hu)
            op.apply_jacobian(hu, hv)
            op.apply_jacobian_transpose(hu, hw)
        dms = 1e3 * (time.perf_counter() - t0) / 3
        dropin = {"value": 3 * ndof / (dms * 1e-3), "unit": "DOF/s", "ms_per_step": dms,
                  "h2d_bytes_per_step": 5 * 8 * ndof, "d2h_bytes_per_step": 3 * 8 * ndof,
                  "path": "SemOperator.apply_rhs / apply_jacobian / apply_jacobian_transpose on numpy "
                          "arrays (what stock semopt code calls): serial applies; numpy inputs stream through a "
                          "ring of pinned chunks, results come back into pinned numpy arrays"}
        cfg3 = cfg3_ops(torch, dev, load_peaks()[0])
    # BASELINE config 5 strong-scaled: at N > 1 rank 0 first times the same ring alone
    strong = None
    if not args.no_cfg5:
        t1 = None
        if world > 1:
            if rank == 0:
                t1 = cfg5_sweep(torch, dist, 1, 0, dev, args.cfg5_steps)
            dist.barrier()
        strong = cfg5_sweep(torch, dist, world, rank, dev, args.cfg5_steps, args.dist_backend)
        if t1 is not None:
            strong["n1_reference"] = t1
            strong["efficiency_vs_n1"] = t1["ms_per_step_pair"] / (world * strong["ms_per_step_pair"])
        strong["note"] = ("strong scaling: the same 2^25-element ring at every N; N = 1's time is "
                          "measured by rank 0 alone in the same job")
        torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = load_peaks()
    per_op = {}
    for k, lst in per.items():
        # an event interval also contains any time the GPU waited for the host to enqueue the
        # launch (one Python hiccup of 2 ms adds 20 us to a 100-launch mean): intervals above
        # 1.25x the median are host gaps, not kernel time, and are dropped and counted
        med = sorted(lst)[len(lst) // 2]
        kept = [t for t in lst if t <= 1.25 * med]
        avg_ms = sum(kept) / len(kept)
        gbs = BYTES_PER_DOF[k] * ndof / (avg_ms * 1e-3) / 1e9
        per_op[k] = {"avg_us": 1e3 * avg_ms, "launches_timed": len(lst),
                     "launches_dropped_host_gap": len(lst) - len(kept),
                     "avg_us_all_intervals": 1e3 * sum(lst) / len(lst), "dof_per_s": ndof / (avg_ms * 1e-3),
                     "achieved_gbs": gbs, "hbm_frac": gbs / peak,
                     "fp64_tflops": flop_per_dof(c["N"], "F" if k == "F" else "J") * ndof
                     / (avg_ms * 1e-3) / 1e12}
    dom = max(per_op, key=lambda k: per_op[k]["avg_us"])
    traffic = load_traffic().get({"F": "rhs", "J": "jac", "JT": "jact"}[dom])
    cpu = None
    if not args.no_cpu_baseline:
        ndof_s, times = cpu_reference_step_sample(1 << 20, 3, seed=12)
        cpu_v = 3 * ndof_s / min(times)
        cores = host_cores()
        cpu = {"value": cpu_v, "unit": "DOF/s", "cores": cores, "kind": "port",
               "sample": f"F+J+J^T once each on E=2^20 of config 2 (same h, N, nu; {ndof_s} DOF), "
                         f"min of 3 reps, numpy/OpenBLAS port of semopt ops.py, {cores} threads"}
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded u~U(-1,1), v,w~N(0,1) per node)",
        "config": workload_config(1) if world == 1 else
                  {"workload": "BASELINE config 2: 1D Burgers, E=2^22, N=7, nu=0.01, periodic [-1,1]",
                   "value": VALUE_DEF, "E": c["E"], "N": c["N"], "dof": ndof,
                   "per_rank_problem": "2^22 elements" + ("" if world == 1 else
                                       " of one element-sharded ring (ghost exchange per input)"),
                   "l2": "inputs 235 MB/field > 126 MB L2, no flush",
                   "parallelism": "single GPU" if world == 1 else
                   f"element-sharded x{world} (NCCL P2P halo: u, v, w ghosts in one batched exchange per step)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": per_op[dom]["achieved_gbs"],
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": per_op[dom]["hbm_frac"], "traffic": traffic,
                     "algorithmic_bytes_per_launch": BYTES_PER_DOF[dom] * ndof,
                     "timing": "CUDA events around every launch (mean over the launches without the intervals above "
                               "1.25x the median, which contain host enqueue gaps; per_op counts them), a second pass of K steps after the "
                               "timed region (value/ms_per_step: K steps with events only at the ends, "
                               "so consecutive launches keep their programmatic-dependent-launch overlap)"},
        "per_op": per_op,
        "ratios": {"JT_over_J": per_op["JT"]["avg_us"] / per_op["J"]["avg_us"],
                   "JT_over_F": per_op["JT"]["avg_us"] / per_op["F"]["avg_us"],
                   "sweep": sweep},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "DOF/s", "h2d_bytes_per_step": 3 * 8 * ndof,
                "d2h_bytes_per_step": 3 * 8 * ndof, "ms_per_step": e2e_ms,
                "path": ("SemOperator.apply_host: pinned host fields streamed in element chunks, "
                         "H2D / kernels / D2H overlapped on three streams") if streaming else
                        "SemOperator.apply_* on pinned host->device copies, results copied back"},
        "tile_kernels": tiles and {"field": "config-2 ring (E=2^22, N=7), RK4, events around 20 "
                                            "back-to-back launches", "fp64_peak_tflops": FP64_PEAK_TFS,
                                   "bytes_per_dof": STEP_BYTES, **tiles},
        "cfg3": cfg3,
        "strong_scaling_cfg5": strong,
        "e2e_dropin": dropin,
        "gpu_launches": 3 * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    del np


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
