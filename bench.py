"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workloads are the BASELINE.json configs.  The default,
C=5a, is the largest single-GPU configuration (configs[4]): 262144
independent instances of E = A.t()*B + C % D and s = trace(A*B), float64,
square sizes drawn uniformly from {32, 64, 128}, U(-1,1) entries (75 GB of
operands resident in HBM).  Inputs are seeded synthetic data, generated on
the device bit-identical to the numpy scheme of SURVEY.md 8(d)
(paper_2502_03000_b200/datagen.py); no dataset is involved.  A *step* is
one evaluation of the config's expressions through the public API.

verified     before anything is timed, a sample of the step's own outputs
             is compared with the oracle (oracle/, the reference loops
             restated in C) at the north-star tolerance -- the reference
             harness verifies before it times (lazymat/bench.py:184-190).
value        algorithmic bytes (or flops) per step x steps, all ranks, / the
             max-over-ranks device time of K steps (CUDA events around CUDA-
             graph replays of the compiled plans; inputs resident in HBM).
e2e          the same metric through the public API from pinned HOST
             buffers: H2D of the inputs and D2H of every result inside the
             timed region.
roofline     the dominant kernel's algorithmic work / its CUDA-event
             duration vs the measured HBM copy peak (MEASURED_PEAKS.json) or
             the measured FP64 peak (profiles/fp64_peak.json).
cpu_baseline the reference's loops restated in C (oracle/) on one core of
             the host, on a bounded sample; batched configs add an all-core
             process pool (`all_cores`).
--impl reference  times that CPU restatement as the reference arm, with
             every host core for the batched configs (independent instances).

Multi-GPU (`--gpus N`; without torchrun this script launches N ranks
itself): configs 4b and 5a partition the FIXED batch into contiguous
instance ranges balanced by realised n^3 (strong scaling, no collective);
5b row-shards the 32768^2 matrices (one NCCL scalar all-reduce); the
single-problem configs 1-4a run one replica per rank (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
DEFAULT_CONFIG = "5a"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback"


def seeded(config: int, k: int, shape, seed: int = 42) -> np.ndarray:
    """Operand k of config c: default_rng(1000003*seed + 101*c + k).uniform(-1,1), F-order."""
    rng = np.random.default_rng(1000003 * seed + 101 * config + k)
    return np.asfortranarray(rng.uniform(-1.0, 1.0, shape))


def _np(x):
    """Host numpy copy of a step output (DenseMatrix, tensor or float)."""
    if hasattr(x, "to_numpy"):
        return x.to_numpy()
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _bitwise(a, b) -> bool:
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                                 b.view(np.int64) if b.dtype == np.float64 else b)


def _normwise(a, b) -> float:
    """max|a - b| / max|b| (lazymat/bench.py:139-143)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b), initial=0.0))


def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------------------

class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during a region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int, enabled: bool = True):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nv = None
        if not enabled:
            return
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
# all-core CPU pool (batched configs: independent instances)
# ---------------------------------------------------------------------------------------

def _pool_worker(config, wid, conn):
    from oracle import lm_oracle as O
    wl = WORKLOADS[config]()
    state = wl.pool_prepare(O, wid)
    conn.send("ready")
    while True:
        rounds = conn.recv()
        if rounds is None:
            break
        for _ in range(rounds):
            wl.pool_round(O, state)
        conn.send("done")
    conn.close()


class CpuPool:
    """One process per host core, each running the oracle on its own
    instances of the workload (generated in the worker, untimed).  A step
    is one round on every worker; its time is the parent's wall clock from
    the first send to the last reply."""

    def __init__(self, config: str, workers: int):
        import multiprocessing as mp
        ctx = mp.get_context("fork")  # created before any CUDA context exists in this process
        self.workers = workers
        self.procs, self.conns = [], []
        for w in range(workers):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_pool_worker, args=(config, w, b), daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(a)
        for c in self.conns:
            if c.recv() != "ready":
                raise RuntimeError("pool worker failed")

    def step(self, rounds: int = 1) -> float:
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(rounds)
        for c in self.conns:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=10)


# ---------------------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------------------

class Workload:
    """One BASELINE config: host inputs, expressions, work per step."""

    config = 0
    unit = "GB/s"
    bound = "hbm"
    graphable = True  # the step has no host synchronisation -> CUDA graph replay
    workload = ""
    dtype = "f64"
    scaling = "weak"  # replicas per rank unless the workload partitions
    pool = False  # independent instances: an all-core CPU pool is meaningful

    def cpu_work_per_step(self):
        return self.work_per_step()

    def host_inputs(self) -> dict:
        raise NotImplementedError

    def expressions(self, lm, mats) -> list:
        raise NotImplementedError

    def work_per_step(self) -> float:  # bytes (GB/s) or flops (TFLOP/s), ALL ranks
        raise NotImplementedError

    def kernels_for_roofline(self, lm, mats):
        """[(name, work_per_launch, thunk)] candidate dominant kernels."""
        return []

    def cpu_step(self, O, host) -> None:
        raise NotImplementedError

    def verify(self, lm, ctx, host, outs, O):
        """(ok, details): the step's outputs vs the oracle."""
        return None, {"note": "no verification defined"}

    def scale(self) -> float:
        return 1e9 if self.unit == "GB/s" else 1e12


# The f32 n=128 batched kernel runs A.T*B as 3xTF32 on mma.sync.m16n8k8.tf32:
# 275.2 TF/s measured (tools/tf32_probe.cu, profiles/r01_tf32_probe.txt),
# three MMAs per product -> an effective f32 ceiling of a third of that.
TF32_MMA_TFLOPS = 275.2


def _tf32x3_peak():
    return TF32_MMA_TFLOPS / 3.0, "3xTF32 effective (legacy mma.sync tf32 275.2 TF/s measured / 3)"


def _fp64_peak():
    p = ROOT / "profiles" / "fp64_peak.json"
    if p.exists():
        return float(json.loads(p.read_text())["tflops"]), "measured (tools/fp64_probe.cu)"
    return 37.0, "fallback"


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

    def e2e_fn(self, lm, h):
        """Through the public API with asynchronous transfers, pipelined over
        column chunks: each chunk of diagmat(v)*B and A*diagmat(v) is
        computed and streams back to the host while the next chunk's
        operands are still arriving (PCIe carries both directions at once);
        trace(A*B) runs once A and B are complete."""
        import torch

        def pin(a):
            return torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory().t()
        pA, pB, pv = pin(h["A"]), pin(h["B"]), pin(h["v"])
        n = self.N
        o2, o3 = (torch.empty((n, n), dtype=torch.float64).pin_memory().t() for _ in range(2))
        ot = torch.empty((1, 1), dtype=torch.float64).pin_memory()

        K = 8  # column chunks: chunk k computes and streams back while chunk k+1 arrives
        w = n // K

        def run():
            from paper_2502_03000_b200.matrix import MatrixView
            v = lm.upload(pv)
            A, B = lm.empty_matrix(n, n), lm.empty_matrix(n, n)
            fs = []
            for k in range(K):
                lm.upload_into(B, pB[:, k * w:(k + 1) * w], k * w)
                Bk = MatrixView(B, 0, k * w, n, w)
                fs.append(lm.download(lm.evaluate(lm.diagmat(v) * Bk), out=o2[:, k * w:(k + 1) * w]))
            for k in range(K):
                lm.upload_into(A, pA[:, k * w:(k + 1) * w], k * w)
                Ak, vk = MatrixView(A, 0, k * w, n, w), MatrixView(v, k * w, 0, w, 1)
                fs.append(lm.download(lm.evaluate(Ak * lm.diagmat(vk)), out=o3[:, k * w:(k + 1) * w]))
            fs.append(lm.download(lm.evaluate(lm.trace(A * B), host_scalar=False), out=ot))
            for f in fs:
                f.wait()
            return [o2, o3, ot]
        return run, (pA.numel() + pB.numel() + pv.numel()) * 8, (o2.numel() + o3.numel() + 1) * 8

    def cpu_step(self, O, h):
        n = self.N
        out = np.empty((n, n), order="F")
        O.trace_of_product(h["A"], h["B"])
        O.diag_scale(np.ascontiguousarray(h["v"][:, 0]), h["B"], "left", out)
        O.diag_scale(np.ascontiguousarray(h["v"][:, 0]), h["A"], "right", out)

    def verify(self, lm, ctx, h, outs, O):
        t = float(_np(outs[0]).ravel()[0])
        tref = O.trace_of_product(h["A"], h["B"])
        v = np.ascontiguousarray(h["v"][:, 0])
        left, right = (np.empty(h["A"].shape, order="F") for _ in range(2))
        O.diag_scale(v, h["B"], "left", left)
        O.diag_scale(v, h["A"], "right", right)
        rel = abs(t - tref) / abs(tref)
        ok = rel <= 1e-12 and _bitwise(_np(outs[1]), left) and _bitwise(_np(outs[2]), right)
        return ok, {"trace_rel_err": rel, "trace_tol": 1e-12, "diag_scale": "bitwise vs oracle, both sides",
                    "size": "full 4096^2"}


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

    def e2e_fn(self, lm, h):
        """Through the public API, pipelined over column chunks: each chunk's
        result streams back to the host while the next chunk's operands are
        still arriving."""
        import torch
        from paper_2502_03000_b200.matrix import MatrixView

        def pin(a):
            return torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory().t()
        p = {k: pin(h[k]) for k in "ABC"}
        n, K = self.N, 8
        w = n // K
        out = torch.empty((n, n), dtype=torch.float64).pin_memory().t()

        def run():
            dev = {k: lm.empty_matrix(n, n) for k in "ABC"}
            fs = []
            for c in range(K):
                for k in "ABC":
                    lm.upload_into(dev[k], p[k][:, c * w:(c + 1) * w], c * w)
                A, B, C = (MatrixView(dev[k], 0, c * w, n, w) for k in "ABC")
                fs.append(lm.download(lm.evaluate(2 * A + B % C - A / (1 + abs(B))), out=out[:, c * w:(c + 1) * w]))
            for f in fs:
                f.wait()
            return [out]
        return run, 3 * n * n * 8, n * n * 8

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

    def verify(self, lm, ctx, h, outs, O):
        ref = np.empty((self.N, self.N), order="F")
        self.cpu_step_into(O, h, ref)
        return _bitwise(_np(outs[0]), ref), {"D": "bitwise vs oracle program (per-node IEEE order)",
                                             "size": "full 4096^2"}

    def cpu_step_into(self, O, h, out):
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
        O.program(ops.numpy(), args.numpy(), [2.0, 1.0], [h["A"], h["B"], h["C"]], out)


class Config3a(Workload):
    config = "3a"
    N = 4096
    workload = "A*B*C*v, float64 4096x4096 A,B,C and 4096x1 v, U(-1,1): re-associated to three GEMVs"

    def host_inputs(self):
        n = self.N
        return {"A": seeded(3, 0, (n, n)), "B": seeded(3, 1, (n, n)), "C": seeded(3, 2, (n, n)),
                "v": seeded(3, 3, (n, 1))}

    def expressions(self, lm, m):
        return [m["A"] * m["B"] * m["C"] * m["v"]]

    def work_per_step(self):
        n = self.N
        return 3 * n * n * 8 + 4 * n * 8

    def kernels_for_roofline(self, lm, m):
        from paper_2502_03000_b200 import kernels as K
        import torch
        n = self.N
        y = torch.empty(n, dtype=torch.float64, device=m["A"].data.device)
        A, v = m["A"].data, m["v"].data[:, 0]
        return [("gemv", n * n * 8 + 2 * n * 8, lambda: K.gemv(A, v, y))]

    def cpu_step(self, O, h):
        n = self.N
        t1, t2, t3 = (np.zeros((n, 1), order="F") for _ in range(3))
        O.gemm(h["C"], h["v"], t1)
        O.gemm(h["B"], t1, t2)
        O.gemm(h["A"], t2, t3)

    def verify(self, lm, ctx, h, outs, O):
        n = self.N
        t1, t2, t3 = (np.zeros((n, 1), order="F") for _ in range(3))
        O.gemm(h["C"], h["v"], t1)
        O.gemm(h["B"], t1, t2)
        O.gemm(h["A"], t2, t3)
        err = _normwise(_np(outs[0]), t3)
        return err <= 1e-12, {"normwise_err": err, "tol": 1e-12, "size": "full 4096^2 chain"}


class Config3b(Workload):
    config = "3b"
    unit = "TFLOP/s"
    bound = "fp64"
    workload = "X*Y*Z, float64 X 8000x100, Y 100x8000, Z 8000x100, U(-1,1): ordered (Y*Z first), 320 MFLOP"

    def host_inputs(self):
        return {"X": seeded(3, 10, (8000, 100)), "Y": seeded(3, 11, (100, 8000)), "Z": seeded(3, 12, (8000, 100))}

    def expressions(self, lm, m):
        return [m["X"] * m["Y"] * m["Z"]]

    def work_per_step(self):
        return 2 * 100 * 8000 * 100 * 2

    def kernels_for_roofline(self, lm, m):
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.matrix import fortran_empty
        out = fortran_empty(100, 100)
        Y, Z = m["Y"].data, m["Z"].data
        return [("gemm(Y,Z)", 2 * 100 * 8000 * 100, lambda: K.gemm(Y, Z, out))]

    def cpu_step(self, O, h):
        yz = np.zeros((100, 100), order="F")
        O.gemm(h["Y"], h["Z"], yz)
        out = np.zeros((8000, 100), order="F")
        O.gemm(h["X"], yz, out)

    def verify(self, lm, ctx, h, outs, O):
        yz = np.zeros((100, 100), order="F")
        O.gemm(h["Y"], h["Z"], yz)
        ref = np.zeros((8000, 100), order="F")
        O.gemm(h["X"], yz, ref)
        err = _normwise(_np(outs[0]), ref)
        return err <= 1e-12, {"normwise_err": err, "tol": 1e-12, "size": "full 8000x100 chain"}


class Config3c(Workload):
    config = "3c"
    unit = "TFLOP/s"
    bound = "fp64"
    workload = "A.t()*A, float64 A 16384x2048 U(-1,1): R8 SYRK (upper tiles + bitwise mirror), 68.75 GFLOP"
    M, K = 16384, 2048

    def host_inputs(self):
        return {"A": seeded(3, 20, (self.M, self.K))}

    def expressions(self, lm, m):
        return [m["A"].t() * m["A"]]

    def work_per_step(self):
        return self.K * (self.K + 1) * self.M  # lazymat/kernels.py:109-116 formula n(n+1)k

    def kernels_for_roofline(self, lm, m):
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.matrix import fortran_empty
        out = fortran_empty(self.K, self.K)
        a = m["A"].data.t()
        return [("syrk", self.work_per_step(), lambda: K.syrk(a, out))]

    cpu_sample_k = 512
    cpu_sample_desc = "the same SYRK over the first 512 of the 16384 inner terms (1/32 of the flops)"

    def cpu_step(self, O, h):
        # bounded sample: the same syrk over the first 512 of the 16384 inner terms
        a = h["A"][: self.cpu_sample_k, :].T
        out = np.zeros((self.K, self.K), order="F")
        O.syrk(a, out)

    def cpu_work_per_step(self):
        return self.K * (self.K + 1) * self.cpu_sample_k

    def verify(self, lm, ctx, h, outs, O):
        """16 sampled 64x64 output tiles (diagonal, edge, interior, both
        triangles) vs the oracle's gemm on the matching column slices of A,
        over all 16384 inner terms; plus the whole device output bitwise
        symmetric."""
        import torch
        out = outs[0].data if hasattr(outs[0], "data") else outs[0]
        sym = bool(torch.equal(out, out.t()))
        S = out.cpu().numpy()
        A = h["A"]
        starts = [0, 64, 960, 1024, 1984]
        tiles = [(i, j) for i in starts for j in starts if abs(i - j) <= 1024][:16]
        worst = 0.0
        for (i0, j0) in tiles:
            ref = np.zeros((64, 64), order="F")
            O.gemm(A[:, i0:i0 + 64].T, A[:, j0:j0 + 64], ref)
            worst = max(worst, _normwise(S[i0:i0 + 64, j0:j0 + 64], ref))
        return sym and worst <= 1e-12, {"tiles": len(tiles), "tile_normwise_err_max": worst, "tol": 1e-12,
                                        "bitwise_symmetric": sym, "size": "full 16384x2048"}


class Config4a(Workload):
    config = "4a"
    unit = "TFLOP/s"
    bound = "fp64"
    graphable = False
    N, NRHS = 8192, 64
    workload = ("inverse(A)*b -> LU solve (R9), float64 A = U(-1,1) + 8192*I (data leaf), b 8192x64; "
                "blocked LU with reference pivots, trailing updates on the FP64 tensor cores (DMMA)")

    def host_inputs(self):
        n = self.N
        a = seeded(4, 0, (n, n))
        a[np.diag_indices(n)] += n
        return {"A": a, "b": seeded(4, 1, (n, self.NRHS))}

    def expressions(self, lm, m):
        return [lm.inverse(m["A"]) * m["b"]]

    def work_per_step(self):
        n, k = self.N, self.NRHS
        return 2 * n * n * n // 3 + 2 * n * n * k  # lazymat/kernels.py:190, :215

    roofline_graphable = False

    def kernels_for_roofline(self, lm, m):
        import torch
        from paper_2502_03000_b200 import _native as N
        from paper_2502_03000_b200.matrix import fortran_empty
        n, k = self.N, self.NRHS
        A, b = m["A"].data, m["b"].data
        work, x = fortran_empty(n, n), fortran_empty(n, k)
        piv = torch.empty(n, dtype=torch.int64, device=A.device)
        info = torch.zeros(1, dtype=torch.int32, device=A.device)

        def factor():  # (out of place, as _lu_factor: the 537 MB workspace copy is inside the call)
            N.call("lm_lu_factor_from", 0, N.view(A), N.view(work), piv.data_ptr(), info.data_ptr(), N.LU_MODES["auto"])

        def solve():
            x.copy_(b)
            N.call("lm_lu_solve_mode", 0, N.view(work), piv.data_ptr(), N.view(x), N.LU_MODES["auto"])
        return [("lu_factor (pivot-free chain + DMMA trailing updates)", 2 * n ** 3 // 3, factor),
                ("lu_solve (DMMA wavefront, inverted diagonal blocks)", 2 * n * n * k, solve)]

    cpu_n = 1024
    cpu_sample_desc = "an n=1024 LU solve with 64 RHS (same unblocked algorithm; a rate, not the 8192 problem)"

    def cpu_step(self, O, h):
        n = self.cpu_n
        a = np.asfortranarray(h["A"][:n, :n] - (self.N - n) * np.eye(n))
        rc, lu, piv = O.lu_factor(a)
        x = np.array(h["b"][:n, :], order="F")
        O.lu_solve(lu, piv, x)

    def cpu_work_per_step(self):
        n, k = self.cpu_n, self.NRHS
        return 2 * n * n * n // 3 + 2 * n * n * k

    def verify(self, lm, ctx, h, outs, O):
        X = _np(outs[0])
        A, B = h["A"], h["b"]
        r = A @ X - B
        res = np.abs(r).sum(axis=1).max() / (np.abs(A).sum(axis=1).max() * np.abs(X).sum(axis=1).max() +
                                             np.abs(B).sum(axis=1).max())
        return res <= 1e-10, {"scaled_residual": float(res), "tol": 1e-10, "size": "full 8192^2, 64 rhs",
                              "norm": "inf-norm, lazymat tests/test_kernels.py:169-179 form"}


def _ws():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))


def _spread(first: int, count: int, k: int) -> list:
    """k local indices spread over [0, count): both ends and the tail included."""
    if count <= k:
        return list(range(count))
    idx = set(np.linspace(0, count - 1, k - 4).round().astype(int).tolist())
    idx.update([0, 1, count - 2, count - 1])
    return sorted(idx)


class Config4b(Workload):
    config = "4b"
    unit = "GB/s"
    graphable = False
    scaling = "strong"
    pool = True
    N, BATCH = 64, 4096
    workload = ("4096 independent inverse(A_i)*b_i, A_i = U(-1,1) + 64*I (64x64), b_i 64x1: batched structure "
                "scan + in-register LU in the reference's exact order; instances partitioned across ranks")
    POOL_SYSTEMS = 64  # per worker per round

    def __init__(self):
        from paper_2502_03000_b200.shard import partition_by_cost
        self.ws, self.rank = _ws()
        self.lo, self.hi = partition_by_cost(np.ones(self.BATCH), self.ws)[self.rank]

    def _full(self, seed_k=7):
        n, bt = self.N, self.BATCH
        rng = np.random.default_rng(1000003 * 42 + 101 * 4 + seed_k)
        a = rng.uniform(-1.0, 1.0, (bt, n, n)) + n * np.eye(n)[None]
        b = rng.uniform(-1.0, 1.0, (bt, n, 1))
        return a, b

    def host_inputs(self):
        a, b = self._full()
        return {"A": a[self.lo:self.hi], "b": b[self.lo:self.hi]}

    def setup(self, lm, h):
        from paper_2502_03000_b200.batch import stack_fortran
        return {"A": stack_fortran(h["A"]), "b": stack_fortran(h["b"])}

    def step_fn(self, lm, ctx):
        from paper_2502_03000_b200.batch import solve_batched
        return lambda: [solve_batched(ctx["A"], ctx["b"]).x]

    def verify(self, lm, ctx, h, outs, O):
        x = outs[0]
        idx = _spread(0, x.shape[0], 64)
        xs = x[idx].cpu().numpy()
        bad = []
        for t, i in enumerate(idx):
            rc, lu, piv = O.lu_factor(np.asfortranarray(h["A"][i]))
            xr = np.array(h["b"][i], order="F")
            O.lu_solve(lu, piv, xr)
            if rc != 0 or not _bitwise(xs[t], xr):
                bad.append(int(i) + self.lo)
        return not bad, {"instances_checked": len(idx), "criterion": "x bitwise vs oracle lu_factor+lu_solve",
                         "mismatches": bad[:8]}

    def e2e_fn(self, lm, h):
        import torch
        from paper_2502_03000_b200.batch import solve_batched
        pa = torch.from_numpy(np.ascontiguousarray(np.transpose(h["A"], (0, 2, 1)))).pin_memory()
        pb = torch.from_numpy(np.ascontiguousarray(h["b"])).pin_memory()
        px = torch.empty_like(pb).pin_memory()
        bt = pa.shape[0]
        K = 4 if bt >= 4 else 1  # instance chunks: chunk k is solved while chunks > k are still uploading
        bounds = [(k * bt // K, (k + 1) * bt // K) for k in range(K)]
        h2d = torch.cuda.Stream()

        def run():
            chunks = []
            h2d.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(h2d):
                for lo, hi in bounds:
                    A = pa[lo:hi].cuda(non_blocking=True).transpose(1, 2)
                    b = pb[lo:hi].cuda(non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(h2d)
                    chunks.append((A, b, ev))
            for (lo, hi), (A, b, ev) in zip(bounds, chunks):
                torch.cuda.current_stream().wait_event(ev)
                A.record_stream(torch.cuda.current_stream())
                b.record_stream(torch.cuda.current_stream())
                x = solve_batched(A, b).x
                px[lo:hi].copy_(x, non_blocking=True)
            torch.cuda.synchronize()
            return [px]
        return run, pa.numel() * 8 + pb.numel() * 8, px.numel() * 8

    def work_per_step(self):
        n, bt = self.N, self.BATCH
        return bt * (n * n * 8 + 2 * n * 8)  # A read once, b read, x written (whole batch, all ranks)

    def rank_work(self):
        n = self.N
        return (self.hi - self.lo) * (n * n * 8 + 2 * n * 8)

    exact_fp64 = True

    def kernels_for_roofline(self, lm, ctx):
        import torch
        from paper_2502_03000_b200 import _native as N
        A = ctx["A"]
        bt, n = A.shape[0], self.N
        x = torch.empty((bt, 1, n), dtype=torch.float64, device=A.device).transpose(1, 2)
        x.copy_(ctx["b"])
        info = torch.empty(bt, dtype=torch.int32, device=A.device)

        def solve():  # in place: repeated solves do the same work
            N.call("lm_lu_solve_batched", 0, n, bt, A.data_ptr(), x.data_ptr(), None, None, info.data_ptr())
        return [("lu_solve_batched", bt * (n * n * 8 + 2 * n * 8), solve, bt * (2 * n ** 3 // 3 + 2 * n * n))]

    def flops_per_step(self):
        n, bt = self.N, self.BATCH
        return bt * (2 * n * n * n // 3 + 2 * n * n)

    cpu_sample_desc = "the rank's systems, oracle lu_factor + lu_solve each"

    def cpu_step(self, O, h):
        for i in range(h["A"].shape[0]):
            rc, lu, piv = O.lu_factor(np.asfortranarray(h["A"][i]))
            x = np.array(h["b"][i], order="F")
            O.lu_solve(lu, piv, x)

    def cpu_work_per_step(self):
        return self.rank_work()

    # all-core pool: each worker solves its own 64 systems per round
    def pool_prepare(self, O, wid):
        n = self.N
        rng = np.random.default_rng([1000003 * 42 + 101 * 4 + 7, 1000 + wid])
        A = [np.asfortranarray(rng.uniform(-1, 1, (n, n)) + n * np.eye(n)) for _ in range(self.POOL_SYSTEMS)]
        b = [np.asfortranarray(rng.uniform(-1, 1, (n, 1))) for _ in range(self.POOL_SYSTEMS)]
        return A, b

    def pool_round(self, O, state):
        for A, b in zip(*state):
            rc, lu, piv = O.lu_factor(A)
            x = np.array(b, order="F")
            O.lu_solve(lu, piv, x)

    def pool_work_round(self):
        n = self.N
        return self.POOL_SYSTEMS * (n * n * 8 + 2 * n * 8)


class Config5a(Workload):
    """262144 instances of E = A.t()*B + C%D, s = trace(A*B), n in {32,64,128}."""

    config = "5a"
    BATCH = 262144
    SIZES = (32, 64, 128)
    dtype = "f64"
    scaling = "strong"
    pool = True
    workload = ("262144 independent E = A.t()*B + C % D and s = trace(A*B), square sizes drawn uniformly from "
                "{32,64,128}, U(-1,1) float64; one grouped kernel per size class; instances partitioned across "
                "ranks by realised n^3")
    CPU_SAMPLE = {32: 96, 64: 48, 128: 16}  # single-core sample (and per pool worker per round: POOL_SAMPLE)
    POOL_SAMPLE = {32: 24, 64: 12, 128: 4}
    VERIFY_PER_CLASS = 256
    e2e_per_class = 8192

    def __init__(self):
        from paper_2502_03000_b200.datagen import batch_sizes
        from paper_2502_03000_b200.shard import class_ranges, partition_by_cost
        self.ws, self.rank = _ws()
        self.sizes = batch_sizes(self.BATCH, self.SIZES)
        self.lo, self.hi = partition_by_cost(self.sizes.astype(np.float64) ** 3, self.ws)[self.rank]
        self.ranges = class_ranges(self.sizes, self.lo, self.hi, self.SIZES)

    @property
    def width(self):
        return 8 if self.dtype == "f64" else 4

    def counts(self):
        return {n: int((self.sizes == n).sum()) for n in self.SIZES}

    def _bytes(self, counts):
        w = self.width
        return sum(c * (5 * n * n * w + w) for n, c in counts.items())

    def _flops(self, counts):
        return sum(c * (2 * n ** 3 + 4 * n * n) for n, c in counts.items())

    def work_per_step(self):  # the whole batch (all ranks)
        return self._bytes(self.counts())

    def flops_per_step(self):
        return self._flops(self.counts())

    def rank_counts(self):
        return {n: c for n, (f, c) in self.ranges.items()}

    def _tdt(self):
        import torch
        return torch.float64 if self.dtype == "f64" else torch.float32

    def _host_instance(self, k, n, idx):
        from paper_2502_03000_b200.datagen import host_batch_instance
        x = host_batch_instance(k, n, idx)
        return x if self.dtype == "f64" else np.asfortranarray(x.astype(np.float32).astype(np.float64))

    def host_inputs(self):
        # bounded single-core CPU sample: the first CPU_SAMPLE[n] instances of each class
        return {n: [[self._host_instance(k, n, i) for k in range(4)] for i in range(self.CPU_SAMPLE[n])]
                for n in self.SIZES}

    def setup(self, lm, host):
        from paper_2502_03000_b200.batch import empty_batch
        from paper_2502_03000_b200.datagen import fill_batch_class
        ctx = {}
        for n, (first, count) in self.ranges.items():
            ctx[n] = [fill_batch_class(empty_batch(count, n, n, self._tdt()), k, n, first) for k in range(4)]
        return ctx

    def step_fn(self, lm, ctx):
        from paper_2502_03000_b200.batch import atb_schur_trace
        return lambda: [atb_schur_trace(*ctx[n]) for n in self.SIZES]

    def verify(self, lm, ctx, h, outs, O):
        """VERIFY_PER_CLASS instances per size class, spread over the rank's
        class range (both ends: the persistent loops' tail), inputs
        regenerated on the host with numpy (so the device generator is
        checked too), E normwise and s against the oracle."""
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 x1 x2 * +")
        tol = 1e-12 if self.dtype == "f64" else 1e-5
        worst_e = worst_s = 0.0
        checked, bad = 0, []
        for ci, n in enumerate(self.SIZES):
            first, count = self.ranges[n]
            E, s = outs[ci]
            idx = _spread(first, count, self.VERIFY_PER_CLASS)
            Ed = E[idx].double().cpu().numpy()
            sd = s[idx].double().cpu().numpy()
            for t, i in enumerate(idx):
                A, B, C, D = (self._host_instance(k, n, first + i) for k in range(4))
                g = np.zeros((n, n), order="F")
                O.gemm(A.T, B, g)
                Er = np.zeros((n, n), order="F")
                O.program(ops.numpy(), args.numpy(), [], [g, C, D], Er)
                tr = O.trace_of_product(A, B)
                ee = _normwise(Ed[t], Er)
                se = abs(sd[t] - tr) / max(abs(tr), np.sum(np.abs(A * B.T)) * 1e-2)
                worst_e, worst_s = max(worst_e, ee), max(worst_s, se)
                if ee > tol or se > tol:
                    bad.append((n, first + i))
                checked += 1
        return not bad, {"instances_checked": checked, "per_class": self.VERIFY_PER_CLASS,
                         "E_normwise_err_max": worst_e, "s_rel_err_max": worst_s, "tol": tol,
                         "inputs": "regenerated on the host with numpy (checks the device generator)",
                         "mismatches": bad[:8]}

    def kernels_for_roofline(self, lm, ctx):
        from paper_2502_03000_b200.batch import atb_schur_trace
        out = []
        for n, c in self.rank_counts().items():
            if c:
                out.append((f"atb_schur_trace n={n}", self._bytes({n: c}),
                            lambda n=n: atb_schur_trace(*ctx[n]), self._flops({n: c})))
        return out

    cpu_sample_desc = "160 instances (96 of n=32, 48 of n=64, 16 of n=128), oracle gemm + program + trace each"

    def _cpu_instance(self, O, n, A, B, C, D, ops, args):
        g = np.zeros((n, n), order="F")
        O.gemm(A.T, B, g)
        E = np.zeros((n, n), order="F")
        O.program(ops, args, [], [g, C, D], E)
        O.trace_of_product(A, B)

    def cpu_step(self, O, h):
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 x1 x2 * +")
        ops, args = ops.numpy(), args.numpy()
        for n in self.SIZES:
            for A, B, C, D in h[n]:
                self._cpu_instance(O, n, A, B, C, D, ops, args)

    def cpu_work_per_step(self):
        return self._bytes(self.CPU_SAMPLE)

    def pool_prepare(self, O, wid):
        from paper_2502_03000_b200.datagen import host_matrix
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 x1 x2 * +")
        rng_seed = [1000003 * 42 + 101 * 5 + 77, wid]
        inst = {n: [[host_matrix(rng_seed + [n, i, k], n, n) for k in range(4)] for i in range(self.POOL_SAMPLE[n])]
                for n in self.SIZES}
        return inst, ops.numpy(), args.numpy()

    def pool_round(self, O, state):
        inst, ops, args = state
        for n in self.SIZES:
            for A, B, C, D in inst[n]:
                self._cpu_instance(O, n, A, B, C, D, ops, args)

    def pool_work_round(self):
        return self._bytes(self.POOL_SAMPLE)

    def e2e_fn(self, lm, ctx):
        """Through the batch API from pinned host buffers, pipelined over
        chunks of 1024 instances: chunk j's inputs upload on one copy stream
        while chunk j-1 computes and chunk j-2's results download on
        another (PCIe carries both directions at once).  A bounded sample
        (e2e_per_class instances of each class, copied from the resident
        seeded batch) keeps the pinned host footprint to a few GB."""
        import torch
        from paper_2502_03000_b200.batch import atb_schur_trace, empty_batch
        tdt, w = self._tdt(), self.width
        # a rate: the per-rank sample shrinks with the world size so N ranks pin
        # about as much host memory as one
        per = max(1024, self.e2e_per_class // max(self.ws, 1))
        k = {n: min(per, c) for n, c in self.rank_counts().items()}
        host_in, dev_in, host_out, dev_out = {}, {}, {}, {}
        for n in self.SIZES:
            if not k[n]:
                continue
            host_in[n] = [torch.empty((k[n], n, n), dtype=tdt).pin_memory().transpose(1, 2) for _ in range(4)]
            for t, src in zip(host_in[n], ctx[n]):
                t.copy_(src[:k[n]])
            dev_in[n] = [empty_batch(k[n], n, n, tdt) for _ in range(4)]
            dev_out[n] = (empty_batch(k[n], n, n, tdt), torch.empty(k[n], dtype=tdt, device="cuda"))
            host_out[n] = (torch.empty((k[n], n, n), dtype=tdt).pin_memory().transpose(1, 2),
                           torch.empty(k[n], dtype=tdt).pin_memory())
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        CH = 1024
        comp = torch.cuda.current_stream()

        def run():
            h2d.wait_stream(comp)
            d2h.wait_stream(comp)
            for n in host_in:
                for lo in range(0, k[n], CH):
                    hi = min(k[n], lo + CH)
                    with torch.cuda.stream(h2d):
                        for t, hsrc in zip(dev_in[n], host_in[n]):
                            t[lo:hi].copy_(hsrc[lo:hi], non_blocking=True)
                    comp.wait_stream(h2d)
                    E, s = dev_out[n]
                    atb_schur_trace(*(t[lo:hi] for t in dev_in[n]), out=(E[lo:hi], s[lo:hi]))
                    d2h.wait_stream(comp)
                    with torch.cuda.stream(d2h):
                        host_out[n][0][lo:hi].copy_(E[lo:hi], non_blocking=True)
                        host_out[n][1][lo:hi].copy_(s[lo:hi], non_blocking=True)
            torch.cuda.synchronize()
            return [v for n in host_out for v in host_out[n]]
        self.e2e_work = self._bytes(k)
        self.e2e_sample = f"{per} instances of each size class per rank, chunks of {CH}"
        return run, sum(4 * c * n * n * w for n, c in k.items()), sum(c * (n * n + 1) * w for n, c in k.items())


class Config5b(Workload):
    """Row-sharded 32768^2: config-1 expression on row blocks + trace(A*B) + one all-reduce."""

    config = "5b"
    N = 32768
    graphable = False
    scaling = "strong"
    workload = ("row-sharded float64 32768x32768 A,B,C U(-1,1): D = 2*A + B % C - A / (1 + abs(B)) on each rank's "
                "row block (no communication) and trace(A*B) from the rank's A rows / B columns + one NCCL "
                "all-reduce of one float64")
    cpu_rows = 256
    cpu_sample_desc = "a 256-row block (config-1 program on 256 x 32768 + its trace partial)"
    e2e_rows = 1024

    @staticmethod
    def seed(name):
        from paper_2502_03000_b200.datagen import seed_for
        return seed_for(5, 50 + "ABC".index(name))

    def work_per_step(self):
        n = self.N
        return 4 * n * n * 8 + 2 * n * n * 8  # total over all ranks (strong scaling)

    def host_inputs(self):
        rng = np.random.default_rng(1000003 * 42 + 101 * 5 + 60)
        r, n = self.cpu_rows, self.N
        return {"A": np.asfortranarray(rng.uniform(-1, 1, (r, n))), "B": np.asfortranarray(rng.uniform(-1, 1, (r, n))),
                "C": np.asfortranarray(rng.uniform(-1, 1, (r, n))), "Bc": np.asfortranarray(rng.uniform(-1, 1, (n, r)))}

    def setup(self, lm, host):
        import torch
        from paper_2502_03000_b200.datagen import fill_seeded
        from paper_2502_03000_b200.matrix import fortran_empty
        from paper_2502_03000_b200.shard import ShardedTrace, row_range
        ws, rank = _ws()
        n = self.N
        lo, hi = row_range(n, rank, ws)
        self.lo, self.hi = lo, hi
        blk = {}
        for k in "ABC":  # rows [lo, hi) of the row-major draw stream of an n x n matrix
            blk[k] = fill_seeded(fortran_empty(hi - lo, n), self.seed(k), skip=lo * n, row_stream=n)
        blk["Bc"] = blk["B"] if ws == 1 else fill_seeded(fortran_empty(n, hi - lo), self.seed("B"), skip=lo,
                                                         row_stream=n)
        mats = {k: lm.DenseMatrix(blk[k]) for k in "ABC"}
        plan = lm.rewrite(2 * mats["A"] + mats["B"] % mats["C"] - mats["A"] / (1 + abs(mats["B"])))
        return {"blk": blk, "plan": plan, "trace": ShardedTrace(),
                "s": torch.empty(1, dtype=torch.float64, device="cuda")}

    def step_fn(self, lm, ctx):
        def step():
            d = lm.execute(ctx["plan"])
            s = ctx["trace"](ctx["blk"]["A"], ctx["blk"]["Bc"], ctx["s"])
            return [d, s]
        return step

    def verify(self, lm, ctx, h, outs, O):
        """Sampled rows of D bitwise vs the oracle program on the same rows
        regenerated on the host with numpy; a 64-row block's trace partial
        (device kernel on the resident block) vs the oracle on its host
        copy."""
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.datagen import host_draws
        from paper_2502_03000_b200.kernels import parse_program
        import torch
        ops, args, *_ = parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
        n, lo, hi = self.N, self.lo, self.hi
        D = outs[0].data
        rows = sorted({0, 1, (hi - lo) // 2, hi - lo - 1})
        rows_ok = True
        for r in rows:
            src = [np.asfortranarray(host_draws(self.seed(k), (lo + r) * n, n).reshape(1, n)) for k in "ABC"]
            ref = np.empty((1, n), order="F")
            O.program(ops.numpy(), args.numpy(), [2.0, 1.0], src, ref)
            rows_ok &= _bitwise(D[r:r + 1, :].cpu().numpy(), ref)
        b = ctx["blk"]
        r0 = (hi - lo) // 3
        part = torch.empty(1, dtype=torch.float64, device="cuda")
        K.trace_of_product(b["A"][r0:r0 + 64, :], b["Bc"][:, r0:r0 + 64], out=part)
        Ah = b["A"][r0:r0 + 64, :].cpu().numpy()
        Bh = b["Bc"][:, r0:r0 + 64].cpu().numpy()
        tr = O.trace_of_product(np.asfortranarray(Ah), np.asfortranarray(Bh))
        rel = abs(float(part.item()) - tr) / abs(tr)
        return rows_ok and rel <= 1e-12, {"D_rows_bitwise": len(rows), "rows_ok": bool(rows_ok),
                                          "trace_block_rel_err": rel, "tol": 1e-12,
                                          "size": f"full 32768-wide rows, rank block [{lo}, {hi})"}

    def kernels_for_roofline(self, lm, ctx):
        from paper_2502_03000_b200 import kernels as K
        from paper_2502_03000_b200.matrix import fortran_empty
        b = ctx["blk"]
        r, n = b["A"].shape
        out = fortran_empty(r, n)
        return [("fused_expr (row block)", 4 * r * n * 8,
                 lambda: K.fused_expr("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -", (2.0, 1.0), [b["A"], b["B"], b["C"]],
                                      out)),
                ("trace_of_product (row block)", 2 * r * n * 8, lambda: K.trace_of_product(b["A"], b["Bc"],
                                                                                            out=ctx["s"]))]

    def cpu_step(self, O, h):
        from paper_2502_03000_b200.kernels import parse_program
        ops, args, *_ = parse_program("x0 c0 * x1 x2 * + x0 x1 abs c1 + / -")
        out = np.empty(h["A"].shape, order="F")
        O.program(ops.numpy(), args.numpy(), [2.0, 1.0], [h["A"], h["B"], h["C"]], out)
        O.trace_of_product(h["A"], h["Bc"])

    def cpu_work_per_step(self):
        r, n = self.cpu_rows, self.N
        return 4 * r * n * 8 + 2 * r * n * 8

    def e2e_fn(self, lm, h):
        import torch
        from paper_2502_03000_b200.shard import ShardedTrace
        r, n = self.e2e_rows, self.N
        rng = np.random.default_rng(7)
        pinned = {k: torch.from_numpy(np.ascontiguousarray(rng.uniform(-1, 1, (n, r)))).pin_memory().t()
                  for k in "ABC"}
        pinned["Bc"] = torch.from_numpy(np.ascontiguousarray(rng.uniform(-1, 1, (r, n)))).pin_memory().t()
        out = torch.empty((n, r), dtype=torch.float64).pin_memory().t()
        st = ShardedTrace()

        def run():
            m = {k: lm.DenseMatrix(t) for k, t in pinned.items()}
            d = lm.evaluate(2 * m["A"] + m["B"] % m["C"] - m["A"] / (1 + abs(m["B"])))
            s = st(m["A"].data, m["Bc"].data)
            out.copy_(d.data)
            val = float(s.item())
            torch.cuda.synchronize()
            return [out, val]
        self.e2e_work = 6 * r * n * 8
        self.e2e_sample = f"{r}-row block"
        return run, 4 * r * n * 8, r * n * 8 + 8


class Config5a32(Config5a):
    config = "5a-f32"
    dtype = "f32"
    workload = Config5a.workload.replace("U(-1,1) float64", "U(-1,1) float32 (float64 draws rounded)")


WORKLOADS = {"1": Config1, "2": Config2, "3a": Config3a, "3b": Config3b, "3c": Config3c, "4a": Config4a,
             "4b": Config4b, "5a": Config5a, "5a-f32": Config5a32, "5b": Config5b}


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


def _all_true(ok, ws: int) -> bool:
    if ws == 1:
        return bool(ok)
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def time_cpu(O, wl, host, budget_s: float = 10.0, min_steps: int = 1, max_steps: int = 1000):
    """Run the C restatement of the reference loops for ~budget_s."""
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps and (steps < min_steps or time.perf_counter() - t0 < budget_s):
        wl.cpu_step(O, host)
        steps += 1
    el = time.perf_counter() - t0
    return steps, el


def cpu_pool_rate(wl, budget_s: float, workers: int) -> dict:
    """All-core rate of the oracle over independent instances (process pool)."""
    pool = CpuPool(wl.config, workers)
    try:
        one = pool.step(1)  # warm-up round (page-in, caches)
        rounds = max(1, int(budget_s / max(one, 1e-3)))
        el = pool.step(rounds)
    finally:
        pool.close()
    work = wl.pool_work_round() * workers * rounds
    return {"value": work / el / wl.scale(), "unit": wl.unit, "cores": workers, "kind": "port",
            "sample": f"{rounds} rounds x {workers} processes ({el:.1f} s); per process per round "
                      f"{getattr(wl, 'POOL_SAMPLE', None) or getattr(wl, 'POOL_SYSTEMS', '')} instances, "
                      f"oracle/lm_oracle.c"}


def _default_setup(wl, lm, host):
    return {k: lm.DenseMatrix(v) for k, v in host.items()}


def _default_step(wl, lm, ctx):
    exprs = wl.expressions(lm, ctx)
    if wl.graphable:
        plans = [lm.rewrite(e) for e in exprs]
        return lambda: [lm.execute(p, host_scalar=False) for p in plans]
    # steps with host synchronisation (structure scans, pivot checks):
    # evaluate() per step, rewrite included, like the reference's timed region
    return lambda: [lm.evaluate(e, host_scalar=False) for e in wl.expressions(lm, ctx)]


def _default_e2e(wl, lm, host):
    import torch
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory().t() for k, v in host.items()}
    outs = {}

    def run():
        m = {k: lm.DenseMatrix(t) for k, t in pinned.items()}
        res = []
        for e in wl.expressions(lm, m):
            r = lm.evaluate(e)
            if isinstance(r, float):
                res.append(r)
                continue
            key = len(res)
            if key not in outs or outs[key].shape != r.data.shape:
                outs[key] = torch.empty(r.data.shape[::-1], dtype=r.data.dtype).pin_memory().t()
            outs[key].copy_(r.data)
            res.append(outs[key])
        torch.cuda.synchronize()
        return res

    h2d = sum(t.numel() * t.element_size() for t in pinned.values())
    res = run()
    d2h = sum(8 if isinstance(r, float) else r.numel() * r.element_size() for r in res)
    return run, h2d, d2h


def _time_device(fn, steps):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _cpu_baseline(args, wl, host):
    from oracle import lm_oracle as O
    cores = _host_cores()
    steps, el = time_cpu(O, wl, host, budget_s=args.cpu_budget)
    cpu = {"value": wl.cpu_work_per_step() * steps / el / wl.scale(), "unit": wl.unit, "cores": 1,
           "host_cores": cores, "kind": "port",
           "sample": f"{steps} steps ({el:.1f} s) of {getattr(wl, 'cpu_sample_desc', 'the same workload')}, "
                     f"oracle/lm_oracle.c (the reference loops restated in C), single thread: 1 of {cores} cores "
                     f"(the reference is single-threaded, SPEC.md:317)"}
    if wl.pool and not args.no_pool:
        cpu["all_cores"] = cpu_pool_rate(wl, args.cpu_budget, cores)
    return cpu


def run_ours(args, wl, ws, rank, local):
    # the CPU baseline runs first: its process pool forks before this
    # process creates a CUDA context
    host = wl.host_inputs()
    cpu = None
    if not args.no_cpu and ws == 1 and rank == 0:
        cpu = _cpu_baseline(args, wl, host)

    import torch

    import paper_2502_03000_b200 as lm
    from paper_2502_03000_b200 import _native

    torch.cuda.set_device(local)
    ctx = wl.setup(lm, host) if hasattr(wl, "setup") else _default_setup(wl, lm, host)
    step = wl.step_fn(lm, ctx) if hasattr(wl, "step_fn") else _default_step(wl, lm, ctx)

    # verify before timing: the step's own outputs against the oracle
    verified, vinfo = None, None
    if not args.no_verify:
        from oracle import lm_oracle as O
        outs = step()
        torch.cuda.synchronize()
        ok, vinfo = wl.verify(lm, ctx, host, outs, O)
        del outs
        verified = _all_true(ok, ws) if ok is not None else None

    sampler = ClockSampler(local, enabled=not args.no_clocks)
    with sampler:
        for _ in range(args.warmup):  # JIT compiles, allocator pools, clocks up
            step()
        torch.cuda.synchronize()
        c0 = _native.launch_count()
        step()
        torch.cuda.synchronize()
        launches_per_step = _native.launch_count() - c0
        timed = step
        if wl.graphable:  # capture the static step as one CUDA graph
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()
            torch.cuda.current_stream().wait_stream(s)
            with torch.cuda.graph(g):
                step()
            timed = g.replay
            for _ in range(args.warmup):
                timed()
        torch.cuda.synchronize()
        _barrier(ws)
        torch.cuda.synchronize()
        ms = _time_device(timed, args.steps)
        _barrier(ws)

        # per-kernel durations for the roofline (CUDA events on the launching stream)
        kern = []
        for entry in wl.kernels_for_roofline(lm, ctx):
            name, work, thunk = entry[:3]
            flops = entry[3] if len(entry) > 3 else None
            thunk()
            torch.cuda.synchronize()
            if getattr(wl, "roofline_graphable", True):
                # 10 back-to-back launches per graph: per-launch device time
                # without the graph-launch gap of a one-kernel graph
                reps = 10
                gk = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gk):
                    for _ in range(reps):
                        thunk()
                gk.replay()
                torch.cuda.synchronize()
                t = _time_device(gk.replay, max(args.steps, 5)) / reps
            else:  # multi-stream / host-synchronising step: plain events
                t = _time_device(thunk, max(args.steps, 3))
            kern.append((name, work, t, flops))
    ms_max = _max_over_ranks(ms, ws)

    e2e = None
    if not args.no_e2e:
        run, h2d, d2h = (wl.e2e_fn(lm, ctx if wl.config in ("5a", "5a-f32") else host) if hasattr(wl, "e2e_fn")
                         else _default_e2e(wl, lm, host))
        for _ in range(2):
            run()
        _barrier(ws)
        k_e2e = max(5, min(args.steps, 10))
        per = []
        for _ in range(k_e2e):  # run() ends with the results on the host (synchronised)
            t0 = time.perf_counter()
            run()
            per.append(time.perf_counter() - t0)
        # median step: host-side hiccups (a stray page-in or GC pause can triple
        # one pipelined step) do not decide the number; the mean is reported too
        el = _max_over_ranks(statistics.median(per), ws)
        el_mean = _max_over_ranks(sum(per) / len(per), ws)
        work = getattr(wl, "e2e_work", None)
        if work is None:
            work = wl.work_per_step() if wl.scaling == "weak" else wl.work_per_step() / ws
        e2e = {"value": work * ws / el / wl.scale(), "unit": wl.unit, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": el * 1e3, "ms_per_step_mean": el_mean * 1e3,
               "steps": k_e2e, "statistic": "median of per-step wall times (host clock, synchronised)",
               "includes": "pinned-host inputs H2D, evaluate / batch API (rewrite + device scans + kernels), "
                           "results D2H"}
        if hasattr(wl, "e2e_sample"):
            e2e["sample"] = f"{wl.e2e_sample} through the API per step (bounded pinned host memory)"

    roof = None
    if kern:
        name, work, kms, kflops = max(kern, key=lambda x: x[2])
        if wl.bound == "fp64":
            peak, peak_kind = _fp64_peak()
            if getattr(wl, "exact_fp64", False):
                # exact-order arithmetic: separately rounded mul and sub, 2
                # FP64-pipe instructions per multiply-add (1 flop each)
                peak, peak_kind = peak / 2, peak_kind + "; /2 for exact mul+sub (no FMA)"
            achieved, unit = work / (kms * 1e-3) / 1e12, "TFLOP/s"
        else:
            peak, peak_kind = _peaks()
            achieved, unit = work / (kms * 1e-3) / 1e9, "GB/s"
            if kflops is not None:
                fpeak, fkind = _fp64_peak() if wl.dtype == "f64" else _tf32x3_peak()
                if getattr(wl, "exact_fp64", False):
                    fpeak, fkind = fpeak / 2, fkind + "; /2 for exact mul+sub (no FMA)"
                fach = kflops / (kms * 1e-3) / 1e12
                if fach / fpeak > achieved / peak:  # the kernel is compute-bound: report that roofline
                    work, achieved, peak, peak_kind, unit = kflops, fach, fpeak, fkind, "TFLOP/s"
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(f"config{wl.config}", {}).get(name)
        roof = {"bound": "tensor" if unit == "TFLOP/s" else "hbm", "kernel": name, "achieved": achieved,
                "peak": peak, "peak_kind": peak_kind, "unit": unit, "frac": achieved / peak, "traffic": traffic,
                "work_per_launch": work, "ms_per_launch": kms,
                "all": {n: dict({"ms": t, wl.unit: w / (t * 1e-3) / wl.scale()},
                                **({"TFLOP/s": f / (t * 1e-3) / 1e12} if f is not None else {}))
                        for n, w, t, f in kern}}
        if unit == "TFLOP/s":
            roof["note"] = ("FP64 (DMMA/DFMA) ceiling; sm_100a has no tcgen05 f64 kind" if wl.dtype == "f64" else
                            "f32 products on TF32 tensor cores (3xTF32, FFMA-level accuracy)")

    strong = wl.scaling == "strong"
    total_work = wl.work_per_step() * (1 if strong else ws)
    parallelism = "single GPU" if ws == 1 else (
        f"{ws} ranks, " + ("instance partition balanced by realised n^3, no collective" if wl.config in
                           ("4b", "5a", "5a-f32") else "row shards + one NCCL scalar all-reduce" if strong
                           else "independent replicas"))
    out = {"metric": METRIC, "value": total_work / (ms_max * 1e-3) / wl.scale(), "unit": wl.unit,
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
           "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
           "dtype": wl.dtype,
           "data": "synthetic: seeded U(-1,1) (SURVEY.md 8(d)), numpy-identical draws generated on the device; "
                   "no public dataset",
           "config": {"workload": wl.workload, "baseline_config": wl.config, "work_per_step": wl.work_per_step(),
                      "l2": "working set per step > 126 MB L2; no flush needed",
                      "parallelism": parallelism,
                      "timing": ("CUDA events around CUDA-graph replays of the compiled plans" if wl.graphable
                                 else "CUDA events around evaluate() calls (host syncs inside)")},
           "impl": "ours", "verified": verified, "verify": vinfo, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
           "clocks": sampler.summary(), "gpu_launches": launches_per_step * args.steps}
    if hasattr(wl, "flops_per_step"):
        out["config"]["flops_per_step"] = wl.flops_per_step()
        out["tflops"] = wl.flops_per_step() * (1 if strong else ws) / (ms_max * 1e-3) / 1e12
    return out


def run_reference(args, wl, ws, rank):
    """Reference arm: the reference's loops (C restatement, oracle/) on the
    host cores -- every core for the batched configs (independent
    instances, one process each), one core otherwise (the reference
    algorithm is single-threaded)."""
    if rank != 0:
        return None
    cores = _host_cores()
    if wl.pool:
        pool = CpuPool(wl.config, cores)
        try:
            for _ in range(args.warmup):
                pool.step(1)
            el = sum(pool.step(1) for _ in range(args.steps)) / args.steps
        finally:
            pool.close()
        v = wl.pool_work_round() * cores / el / wl.scale()
        used = cores
        sample = (f"{args.steps} steps; each step one round on {cores} processes, per process "
                  f"{getattr(wl, 'POOL_SAMPLE', None) or getattr(wl, 'POOL_SYSTEMS', '')} instances; "
                  f"oracle/lm_oracle.c (the reference's numba loops restated in C)")
    else:
        from oracle import lm_oracle as O
        host = wl.host_inputs()
        for _ in range(args.warmup):
            wl.cpu_step(O, host)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wl.cpu_step(O, host)
        el = (time.perf_counter() - t0) / args.steps
        v = wl.cpu_work_per_step() / el / wl.scale()
        used = 1
        sample = (f"{args.steps} steps of {getattr(wl, 'cpu_sample_desc', 'the full workload')}, oracle/lm_oracle.c "
                  f"(the reference's numba loops restated in C), single thread like the reference: 1 of {cores} cores")
    return {"metric": METRIC, "value": v, "unit": wl.unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el * 1e3, "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
            "dtype": wl.dtype, "data": "synthetic: seeded U(-1,1) (SURVEY.md 8(d))",
            "config": {"workload": wl.workload, "baseline_config": wl.config, "work_per_step": wl.work_per_step()},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": wl.unit, "cores": used, "host_cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(args, argv) -> int:
    """`--gpus N` without torchrun: launch N ranks (one per GPU) ourselves."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(pathlib.Path(__file__).resolve()),
           *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pool", action="store_true", help="skip the all-core CPU pool")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-clocks", action="store_true", help="skip the NVML clock sampler thread")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args, argv))
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
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = run_ours(args, wl, ws, rank, local)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if out.get("verified") is False:
        sys.exit(3)  # a wrong result is not a benchmark number


if __name__ == "__main__":
    main()
