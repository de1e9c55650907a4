"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workloads are the BASELINE.json configs; the default,
C=2, is configs[1]: trace(A*B), diagmat(v)*B and A*diagmat(v) on float64
4096x4096 A, B and a length-4096 v, entries U(-1,1) (seeded synthetic
data, no dataset is involved).  A *step* is one evaluation of the
config's expressions through the public API.

value        algorithmic bytes (or flops) per step x steps, all ranks, / the
             max-over-ranks device time of K steps (CUDA events around CUDA-
             graph replays of the compiled plans; inputs resident in HBM).
e2e          the same metric through evaluate() from pinned HOST buffers:
             H2D of the inputs and D2H of every result inside the timed
             region (rewrite + device structure scans included).
roofline     the dominant kernel's algorithmic bytes / its CUDA-event
             duration vs the measured HBM copy peak (MEASURED_PEAKS.json).
cpu_baseline the reference's loops restated in C (oracle/, single thread,
             same inputs) on a bounded sample -- a reported baseline only.
--impl reference  times that CPU restatement as the reference arm.

Multi-GPU: these configs do not shard (replicas only) --
every rank runs the same workload independently; value = total work of
all ranks / max rank time.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def seeded(config: int, k: int, shape, seed: int = 42) -> np.ndarray:
    """Operand k of config c: default_rng(1000003*seed + 101*c + k).uniform(-1,1), F-order."""
    rng = np.random.default_rng(1000003 * seed + 101 * config + k)
    return np.asfortranarray(rng.uniform(-1.0, 1.0, shape))


# ---------------------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------------------

class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during a region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------------------

class Workload:
    """One BASELINE config: host inputs, expressions, work per step."""

    config = 0
    unit = "GB/s"
    workload = ""
    dtype = "f64"

    def host_inputs(self) -> dict:
        raise NotImplementedError

    def expressions(self, lm, mats) -> list:
        raise NotImplementedError

    def work_per_step(self) -> float:  # bytes (GB/s) or flops (TFLOP/s)
        raise NotImplementedError

    def kernels_for_roofline(self, lm, mats):
        """[(name, work_per_launch, thunk)] candidate dominant kernels."""
        return []

    def cpu_step(self, O, host) -> None:
        raise NotImplementedError

    def scale(self) -> float:
        return 1e9 if self.unit == "GB/s" else 1e12


class Config2(Workload):
    config = 2
    N = 4096
    workload = "trace(A*B), diagmat(v)*B, A*diagmat(v); float64 A,B 4096x4096, v 4096x1, U(-1,1)"

    def host_inputs(self):
        n = self.N
        return {"A": seeded(2, 0, (n, n)), "B": seeded(2, 1, (n, n)), "v": seeded(2, 2, (n, 1))}

    def expressions(self, lm, m):
        return [lm.trace(m["A"] * m["B"]), lm.diagmat(m["v"]) * m["B"], m["A"] * lm.diagmat(m["v"])]

    def work_per_step(self):
        n = self.N
        return 2 * n * n * 8 + 2 * (2 * n * n * 8 + 8 * n)  # each operand once, each output once

    def kernels_for_roofline(self, lm, m):
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.matrix import fortran_empty
        import torch
        n = self.N
        A, B, v = m["A"].data, m["B"].data, m["v"].data
        out = fortran_empty(n, n)
        s = torch.empty(1, dtype=torch.float64, device=A.device)
        return [("trace_of_product", 2 * n * n * 8, lambda: K.trace_of_product(A, B, out=s)),
                ("diag_scale", 2 * n * n * 8 + 8 * n, lambda: K.diag_scale(v[:, 0], B, "left", out))]

    def cpu_step(self, O, h):
        n = self.N
        out = np.empty((n, n), order="F")
        O.trace_of_product(h["A"], h["B"])
        O.diag_scale(np.ascontiguousarray(h["v"][:, 0]), h["B"], "left", out)
        O.diag_scale(np.ascontiguousarray(h["v"][:, 0]), h["A"], "right", out)


class Config1(Workload):
    config = 1
    N = 4096
    workload = "D = 2*A + B % C - A / (1 + abs(B)); float64 A,B,C 4096x4096 U(-1,1); one fused pass"

    def host_inputs(self):
        n = self.N
        return {k: seeded(1, i, (n, n)) for i, k in enumerate("ABC")}

    def expressions(self, lm, m):
        A, B, C = m["A"], m["B"], m["C"]
        return [2 * A + B % C - A / (1 + abs(B))]

    def work_per_step(self):
        return 4 * self.N * self.N * 8

    def kernels_for_roofline(self, lm, m):
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.matrix import fortran_empty
        n = self.N
        out = fortran_empty(n, n)
        srcs = [m[k].data for k in "ABC"]
        return [("fused_expr", 4 * n * n * 8,
                 lambda: K.fused_expr("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -", (2.0, 1.0), srcs, out))]

    def cpu_step(self, O, h):
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
        out = np.empty((self.N, self.N), order="F")
        O.program(ops.numpy(), args.numpy(), [2.0, 1.0], [h["A"], h["B"], h["C"]], out)


WORKLOADS = {1: Config1, 2: Config2}


# ---------------------------------------------------------------------------------------
# measurement
# ---------------------------------------------------------------------------------------

def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_cpu(O, wl, host, budget_s: float = 10.0, min_steps: int = 1, max_steps: int = 1000):
    """Run the C restatement of the reference loops for ~budget_s."""
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps and (steps < min_steps or time.perf_counter() - t0 < budget_s):
        wl.cpu_step(O, host)
        steps += 1
    el = time.perf_counter() - t0
    return steps, el


def run_ours(args, wl, ws, rank, local):
    import torch

    import paper_2502_03000_b200 as lm
    from paper_2502_03000_b200 import _native

    torch.cuda.set_device(local)
    host = wl.host_inputs()
    mats = {k: lm.DenseMatrix(v) for k, v in host.items()}
    exprs = wl.expressions(lm, mats)
    plans = [lm.rewrite(e) for e in exprs]

    def step():
        return [lm.execute(p, host_scalar=False) for p in plans]

    sampler = ClockSampler(local)
    with sampler:
        # warm-up (JIT compiles, allocator pools), launch count of one step
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        c0 = _native.launch_count()
        step()
        torch.cuda.synchronize()
        launches_per_step = _native.launch_count() - c0
        # capture the step as one CUDA graph (plans are static)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            step()
        for _ in range(max(args.warmup, 3)):
            g.replay()
        torch.cuda.synchronize()
        _barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        _barrier(ws)
        ms = e0.elapsed_time(e1) / args.steps

        # per-kernel durations for the roofline (CUDA events, same stream, graph replays)
        kern = []
        for name, work, thunk in wl.kernels_for_roofline(lm, mats):
            thunk()
            torch.cuda.synchronize()
            gk = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gk):
                thunk()
            gk.replay()
            torch.cuda.synchronize()
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record()
            for _ in range(args.steps):
                gk.replay()
            k1.record()
            torch.cuda.synchronize()
            kern.append((name, work, k0.elapsed_time(k1) / args.steps))
    ms_max = _max_over_ranks(ms, ws)

    # end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        pinned = {k: torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory().t() for k, v in host.items()}
        outs = {}

        def e2e_step():
            m = {k: lm.DenseMatrix(t) for k, t in pinned.items()}
            res = []
            for e in wl.expressions(lm, m):
                r = lm.evaluate(e)
                if isinstance(r, float):
                    res.append(r)
                else:
                    key = len(res)
                    if key not in outs or outs[key].shape != r.data.shape:
                        outs[key] = torch.empty(r.data.shape[::-1], dtype=r.data.dtype).pin_memory().t()
                    outs[key].copy_(r.data)
                    res.append(outs[key])
            torch.cuda.synchronize()
            return res

        for _ in range(2):
            e2e_step()
        h2d = sum(t.numel() * t.element_size() for t in pinned.values())
        res = e2e_step()
        d2h = sum(8 if isinstance(r, float) else r.numel() * r.element_size() for r in res)
        _barrier(ws)
        k_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            e2e_step()
        el = (time.perf_counter() - t0) / k_e2e
        el = _max_over_ranks(el, ws)
        e2e = {"value": wl.work_per_step() * ws / el / wl.scale(), "unit": wl.unit,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": el * 1e3,
               "steps": k_e2e, "includes": "H2D inputs, rewrite (+device scans), kernels, D2H results"}

    # CPU restatement of the reference loops (rank 0, N=1 only)
    cpu = None
    if not args.no_cpu and ws == 1 and rank == 0:
        from oracle import lm_oracle as O
        steps, el = time_cpu(O, wl, host, budget_s=args.cpu_budget)
        cpu = {"value": wl.work_per_step() * steps / el / wl.scale(), "unit": wl.unit, "cores": 1, "kind": "port",
               "sample": f"{steps} full steps of the same workload ({el:.1f} s), oracle/lm_oracle.c single thread"}

    peak, peak_kind = _peaks()
    roof = None
    if kern:
        name, work, kms = max(kern, key=lambda x: x[2])
        achieved = work / (kms * 1e-3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(f"config{wl.config}", {}).get(name)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": work, "ms_per_launch": kms,
                "all": {n: {"ms": t, "GB/s": w / (t * 1e-3) / 1e9} for n, w, t in kern}}

    out = {"metric": METRIC, "value": wl.work_per_step() * ws / (ms_max * 1e-3) / wl.scale(), "unit": wl.unit,
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": wl.dtype,
           "data": "synthetic: seeded U(-1,1) (SURVEY.md 8(d)); no public dataset",
           "config": {"workload": wl.workload, "baseline_config": wl.config,
                      "work_per_step": wl.work_per_step(),
                      "l2": "every input > 126 MB L2 (4096^2 f64 = 134 MB); no flush needed",
                      "parallelism": "replicas" if ws > 1 else "single GPU",
                      "timing": "CUDA events around CUDA-graph replays of the compiled plans"},
           "impl": "ours", "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
           "clocks": sampler.summary(), "gpu_launches": launches_per_step * args.steps}
    return out


def run_reference(args, wl, ws, rank):
    """Reference arm: the reference's loops (C restatement, oracle/) on the host cores."""
    if rank != 0:
        return None
    from oracle import lm_oracle as O
    host = wl.host_inputs()
    for _ in range(args.warmup):
        wl.cpu_step(O, host)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.cpu_step(O, host)
    el = (time.perf_counter() - t0) / args.steps
    v = wl.work_per_step() / el / wl.scale()
    return {"metric": METRIC, "value": v, "unit": wl.unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": wl.dtype, "data": "synthetic: seeded U(-1,1) (SURVEY.md 8(d))",
            "config": {"workload": wl.workload, "baseline_config": wl.config, "work_per_step": wl.work_per_step()},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": wl.unit, "cores": 1, "kind": "port",
                             "sample": f"{args.steps} full steps, oracle/lm_oracle.c (the reference's numba loops "
                                       f"restated in C, single thread like the reference)"},
            "e2e": {"value": v, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    ws, rank, local = _dist()
    wl = WORKLOADS[args.config]()
    if args.impl == "reference":
        out = run_reference(args, wl, ws, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    out = run_ours(args, wl, ws, rank, local)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
