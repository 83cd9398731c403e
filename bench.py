#!/usr/bin/env python
"""POAS co-executed GEMM benchmark on B200 (driver contract: one JSON line).

Metric (BASELINE.json): co-executed GEMM TFLOP/s at N=16384 on 1/2/4/8 B200,
plus speedup vs the best single unit.

Per rank (one process per GPU; `--gpus N` launches the N ranks itself; weak scaling):
  units      gpu<r>.tc   tensor cores (tcgen05 bf16 -> fp32) on TC_SMS SMs
             gpu<r>.simt CUDA cores (fp32 FFMA) on SIMT_SMS whole SMs
  predict    the POAS profiler probes both units on this box (C++, real
             kernels) -> "poas-profile v1"
  optimize/adapt/schedule   the reference-identical planner -> schedule JSON
  step       one co-executed GEMM of this rank's M=16384 rows x N=K=16384:
             every unit's share concurrently through the executor (C ABI);
             at N > 1 rank 0's B (bf16; fp32 too if the CUDA-core unit has
             rows) is delivered by the library's communicator inside the
             step, in column panels (copy-engine chain over CUDA IPC by
             default, NCCL optional); the tensor unit consumes them in ONE
             launch whose producers wait per panel on a device flag
             written after that panel landed
  value      whole-job TFLOP/s = 2*M_total*N*K / max-over-ranks device time
  e2e        the same GEMM through poas_b200_execute with HOST pinned buffers
             (bf16 A/B for the tensor unit, fp32 for the others, fp32 C):
             H2D copy-in, compute, D2H copy-out inside the timed step;
             e2e.fp32_host: the same with fp32 A/B converted on the GPU

`--impl reference` times the reference's own CPU path for this workload on
the host cores (the reference planner from oracle/_ref planning a CPU-only
run, executed tile by tile by the oracle port) and prints the same line.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = 20261017
N_DEFAULT = 16384
TC_SMS = 146
TC_SMS_MULTI = 144  # N > 1: 4 SMs (with the idle CUDA-core unit's 2) stay free for NCCL's broadcast kernels
SIMT_SMS = 2
PROFILING = "probes=9,repetitions=3,bandwidth_payload=268435456"
# the tensor unit re-probed on the budget the partition decision gives it:
# the bottom and top of its range, 5 repetitions each, so the fitted line
# passes through the measured top (the size the steps run); in between the
# time is a staircase of whole waves of tiles (tools/sweep.py PROF_TC)
PROFILING_TC = "probes=2,repetitions=5,bandwidth_payload=268435456"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", 0) or 0), "measured"
        except Exception:
            pass
    return 1590.0, 1400.0, "fallback"  # B200_PROFILING.md: 1.59 burst, ~1.4 sustained


def concurrent_link_ms(torch, h2d_bytes: int, d2h_bytes: int) -> float | None:
    """Best of 3: `h2d_bytes` host->device and `d2h_bytes` device->host at
    the same time (pinned host memory, 64 MiB copies, one stream each), ms."""
    try:
        chunk = 64 << 20
        hs = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
        hd = torch.empty(d2h_bytes, dtype=torch.uint8).pin_memory()
        ds = torch.empty(d2h_bytes, dtype=torch.uint8, device="cuda")
        dd = torch.empty(h2d_bytes, dtype=torch.uint8, device="cuda")
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(True) for _ in range(3))
            e0.record()
            s_in.wait_event(e0)
            s_out.wait_event(e0)
            with torch.cuda.stream(s_in):
                for a in range(0, h2d_bytes, chunk):
                    dd[a:a + chunk].copy_(hs[a:a + chunk], non_blocking=True)
            with torch.cuda.stream(s_out):
                for a in range(0, d2h_bytes, chunk):
                    hd[a:a + chunk].copy_(ds[a:a + chunk], non_blocking=True)
            e1.record(s_in)
            e2.record(s_out)
            torch.cuda.synchronize()
            t = max(e0.elapsed_time(e1), e0.elapsed_time(e2))
            best = t if best is None else min(best, t)
        del hs, hd, ds, dd
        return best
    except Exception:
        return None


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s, MEASURED_PEAKS.json) or None."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return None


class ClockSampler:
    """SM clock + clock-event (throttle) reasons DURING the timed region.

    NVML (the library nvidia-smi reads) polled every 10 ms from a thread, so
    even a sub-second timed region gets real samples; nvidia-smi -lms 100 is
    the fallback when pynvml is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[int, int, int]] = []  # (sm_mhz, max_mhz, reason bits)
        self._stop = threading.Event()
        self._nv = None
        self._max = None
        self.error = None

    _nvml = {}  # gpu -> (pynvml, handle): initialised once (nvmlInit can take
    # ~100 ms; right before a timed region that idle gap lets the power cap
    # recover and the region run at boost clocks)

    @classmethod
    def prepare(cls, gpu: int) -> None:
        """NVML up front, outside any timed region."""
        if gpu in cls._nvml:
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            cls._nvml[gpu] = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(gpu))
        except Exception:
            cls._nvml[gpu] = None

    def __enter__(self):
        try:
            self.prepare(self.gpu)
            if self._nvml[self.gpu] is None:
                raise RuntimeError("NVML unavailable")
            self._nv = self._nvml[self.gpu]
            self._sample()  # one synchronous sample: fails here, not silently in the thread
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception as exc:
            self.error = repr(exc)
            self._nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _sample(self):
        nv, h = self._nv
        if self._max is None:
            self._max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:  # older bindings: the pre-rename entry point
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), self._max, bits))

    def _poll(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception as exc:  # keep the reason; the summary reports it
                self.error = repr(exc)
                break
            self._stop.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self._nv is not None:
            try:
                self._sample()  # the region's last moment
            except Exception as e:
                self.error = repr(e)
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for clk, cmax, bits in self.samples:
            sm.append(float(clk))
            mx = max(mx, float(cmax))
            for bit, nm in self.REASONS.items():
                if bits & bit:
                    reasons.add(nm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "error": self.error}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# ----------------------------------------------------------------- reference
class ReferenceCPUPath:
    """The reference's CPU path for an N^3 GEMM on this host: the reference
    planner (oracle/_ref/libpoasref.so, compiled from /root/reference) plans
    a CPU-only machine; the oracle port executes a bounded sample of that
    plan's work (the first `rows` rows of A against every k'-strip of B,
    split-K, as the plan's tiles do) on all host cores. B and the largest A
    sample are generated once."""

    def __init__(self, n: int, max_rows: int):
        import oracle

        self.oracle, self.n = oracle, n
        self.cores = os.cpu_count() or 1
        # CPU-only machine, reference ProfilingConfig defaults (cpu sides 1000-2000).
        cfg = ("poas-machine v1\n\nbus true\n\ndevice cpu0\nkind cpu\ntrue_slope 2e-12\n"
               "true_intercept 0.0005\nelem_size 4\nnoise 0\ndrift 0\ncache_bytes 33554432\n")
        profile = oracle.ref.exact_profile(cfg)
        t0 = time.perf_counter()
        sched = json.loads(oracle.ref.plan(profile, n, n, n))
        self.plan_s = time.perf_counter() - t0
        tiles = sched["devices"][0]["tiles"]
        self.kp = tiles[0]["k"]
        self.strips = n // self.kp
        self.parts = len(tiles) // self.strips
        self.ntiles = len(tiles)
        self.A = oracle.fill_uniform(min(max_rows, n), n, oracle.stream_seed(SEED, "A"), total_cols=n)
        self.B = oracle.fill_uniform(n, n, oracle.stream_seed(SEED, "B"))
        oracle.exec_tiles_f32(self.A[:8], self.B, [8] * self.strips, self.kp)  # page-in, thread spin-up

    def run(self, rows: int) -> float:
        """Seconds for `rows` rows x full K (split-K over the plan's strips)."""
        t0 = time.perf_counter()
        self.oracle.exec_tiles_f32(self.A[:rows], self.B, [rows] * self.strips, self.kp)
        return time.perf_counter() - t0

    def rows_for(self, seconds: float) -> int:
        """Rows whose sample takes about `seconds` (multiples of 64)."""
        t = self.run(64)
        rows = int(64 * seconds / max(t, 1e-6)) // 64 * 64
        return max(64, min(rows, self.A.shape[0]))

    def sample(self, rows: int) -> str:
        return (f"reference CPU-only plan of {self.n}^3 ({self.ntiles} tiles {self.parts}x{self.strips}, "
                f"k'={self.kp}) planned by oracle/_ref in {self.plan_s * 1e6:.0f} us; timed: {rows} rows x "
                f"full K ({self.strips} split-K tiles of {rows}x{self.kp}x{self.n}) by the oracle port, "
                f"fp32, {self.cores} threads")


def reference_cpu_path(n: int, sample_rows: int | None = None, reps: int = 1, seconds: float = 10.0):
    """(TFLOP/s, seconds per rep, sample description, cores) of the
    reference CPU path on a bounded sample: `sample_rows` rows, or as many
    as take about `seconds`."""
    ref = ReferenceCPUPath(n, sample_rows or 8192)
    rows = sample_rows or ref.rows_for(seconds)
    sec = sum(ref.run(rows) for _ in range(reps)) / reps
    return 2.0 * rows * n * n / sec / 1e12, sec, ref.sample(rows), ref.cores


def run_reference(args):
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    if rank != 0:
        return 0
    n = args.n
    reps_w, reps_k = max(0, args.warmup), max(1, args.steps)
    # each step a bounded sample: ~10 s, and the whole run under ~3 minutes
    ref = ReferenceCPUPath(n, args.ref_rows or 8192)
    rows = args.ref_rows or ref.rows_for(min(10.0, 150.0 / (reps_w + reps_k)))
    for _ in range(reps_w):
        ref.run(rows)
    sec = sum(ref.run(rows) for _ in range(reps_k)) / reps_k
    tfl, sample, cores = 2.0 * rows * n * n / sec / 1e12, ref.sample(rows), ref.cores
    line = {
        "metric": "co-executed GEMM TFLOP/s at N=16384 (1/2/4/8 B200); speedup vs best single unit",
        "value": round(tfl, 4), "unit": "TFLOP/s", "n_gpus": world, "steps": reps_k,
        "warmup": reps_w, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C3 GEMM N={n} (reference CPU path: reference planner + oracle port "
                               f"executing its CPU-only plan, bounded sample)", "m": n, "n": n, "k": n},
        "cpu_baseline": {"value": round(tfl, 4), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(tfl, 4), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"unknown ({os.cpu_count()} logical CPUs)"


def host_unit_baseline(poas, n: int) -> dict:
    """This repo's own host-CPU unit (host_gemm: AVX-512 packed panels +
    OpenMP, every host core) on the same host: config C1 (2048^3 fp32 through
    predict -> plan -> execute on a CPU-only machine) and a bounded sample of
    the N^3 workload -- the competent CPU path beside the oracle port."""
    import numpy as np

    out = {"cores": os.cpu_count()}
    # C1: the POAS pipeline on the host cores only
    units = "cpu0=cpu:threads=0"
    prof = poas.profile_machine(units, "probes=5,repetitions=2,cpu_min_side=1000,cpu_max_side=2000", bus=True, retries=2)
    c1 = 2048
    sched = poas.plan(prof, c1, c1, c1)
    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")
    A = np.empty((c1, c1), np.float32)
    B = np.empty((c1, c1), np.float32)
    Cm = np.empty((c1, c1), np.float32)
    poas.fill_uniform_host(A.ctypes.data, c1, c1, c1, 0, 0, c1, sa)
    poas.fill_uniform_host(B.ctypes.data, c1, c1, c1, 0, 0, c1, sb)
    ex = poas.Executor(units)
    io = poas.GemmIO(m=c1, n=c1, k=c1, a_host=A.ctypes.data, lda_host=c1, b_host=B.ctypes.data, ldb_host=c1,
                     c_host=Cm.ctypes.data, ldc_host=c1, resident=0)
    ex.execute(sched, io, 1)
    # the median of three 5-repeat runs (the host's clock wanders after the
    # reference path's 10 s of all-core load just before)
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        r_ = ex.execute(sched, io, 5)
        runs.append(((time.perf_counter() - t0) / 5, r_))
    runs.sort(key=lambda x: x[0])
    sec, rep = runs[1]
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = float(np.linalg.norm(Cm - ref) / np.linalg.norm(ref))
    out["c1"] = {"workload": "C1: 2048^3 fp32, POAS predict/plan/execute on a CPU-only machine (host_gemm)",
                 "tflops": round(2.0 * c1 ** 3 / sec / 1e12, 4), "ms": round(sec * 1e3, 3),
                 "plan_tiles": len(json.loads(sched)["devices"][0]["tiles"]),
                 "makespan_error_pct": round(rep["makespan_error_pct"], 3), "c_rel_err": float(f"{err:.3e}"),
                 "c_ok": err <= 2e-5}
    # the N^3 workload, a bounded sample of rows (all of K and N)
    rows = 512
    A2 = np.empty((rows, n), np.float32)
    B2 = np.empty((n, n), np.float32)
    C2 = np.empty((rows, n), np.float32)
    poas.fill_uniform_host(A2.ctypes.data, n, rows, n, 0, 0, n, sa)
    poas.fill_uniform_host(B2.ctypes.data, n, n, n, 0, 0, n, sb)
    poas.host_gemm(64, n, n, A2.ctypes.data, n, B2.ctypes.data, n, C2.ctypes.data, n)
    t0 = time.perf_counter()
    poas.host_gemm(rows, n, n, A2.ctypes.data, n, B2.ctypes.data, n, C2.ctypes.data, n)
    sec = time.perf_counter() - t0
    out["sample"] = {"rows": rows, "n": n, "k": n, "tflops": round(2.0 * rows * n * n / sec / 1e12, 4),
                     "seconds": round(sec, 3)}
    return out


def reference_planner_cost(profile: str, m: int, n: int, k: int) -> dict:
    """the reference planner (oracle/_ref, compiled from
    /root/reference) -- us per plan, one thread -- on this run's profile and
    on the reference's mach2 machine, and its exhaustive oracle_grid_search
    at resolution 2000 over mach2's 3 units on all host threads."""
    import oracle

    out = {}
    sec = oracle.ref.time_plan(profile, m, n, k, 200)
    out["plan_us_this_profile"] = round(sec * 1e6, 2)
    mach2 = (ROOT / "tests" / "golden" / "mach2.cfg")
    if mach2.exists():
        prof2 = oracle.ref.exact_profile(mach2.read_text())
        out["plan_us_mach2"] = {f"{a}x{b}x{c}": round(oracle.ref.time_plan(prof2, a, b, c, 200) * 1e6, 2)
                                for a, b, c in ((2048, 2048, 2048), (8192, 8192, 8192), (16384, 16384, 16384),
                                                (65536, 8192, 8192))}
        t0 = time.perf_counter()
        oracle.ref.oracle_grid_search(prof2, 16384, 16384, 16384, 2000, parallel=True)
        out["oracle_grid_search_res2000_s"] = round(time.perf_counter() - t0, 4)
        out["threads"] = os.cpu_count()
    return out


# ----------------------------------------------------------------------- ours
def warm_sustained(poas, torch, dev, seconds: float) -> None:
    """Back-to-back 8192^3 tensor GEMMs for `seconds` (scratch operands)."""
    n = 8192
    a = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    b = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    c = torch.empty(n, n, device=dev)
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 3)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 4)
    s = torch.cuda.current_stream().cuda_stream
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end:
        for _ in range(20):  # ~15 ms of queued work per check
            poas.tc_gemm(poas.DTYPE_BF16, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=s)
        torch.cuda.synchronize()
    del a, b, c


def _static_summary(dyn):
    """The first dynamic iteration ran the profile-only (static) plan."""
    it = dyn["iterations"][0]
    return {"rows": it["rows"], "predicted_ms": round(it["predicted_makespan"] * 1e3, 4),
            "measured_ms": round(it["measured_makespan"] * 1e3, 4),
            "makespan_error_pct": round(it["makespan_error_pct"], 3)}


class Group:
    """The job's ranks for the bench's own bookkeeping (barrier, max over
    ranks, all-gather): the library communicator (poas_b200_comm_*), or a
    no-op at N = 1."""

    def __init__(self, comm):
        self.comm = comm

    def barrier(self):
        if self.comm:
            self.comm.barrier()

    def max(self, v: float) -> float:
        return self.comm.max(v) if self.comm else float(v)

    def allgather(self, text: str) -> list[str]:
        return self.comm.allgather(text) if self.comm else [text]


def relaunch(args) -> int:
    """`bench.py --gpus N` without a launcher: re-run under torchrun with N
    ranks (one process per GPU) and pass its output through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    log("launching", " ".join(cmd[2:6]), "...")
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # (--size: "--n" is ambiguous on a torchrun command line)
    ap.add_argument("--n", "--size", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--m-total", type=int, default=None,
                    help="strong scaling (config C4: --m-total 65536 --size 8192): the job's M rows "
                         "split over the ranks instead of --size rows per rank")
    ap.add_argument("--tc-sms", type=int, default=None,
                    help=f"tensor unit SM budget (default {TC_SMS}; {TC_SMS_MULTI} with --b-transport nccl "
                         "at N > 1)")
    ap.add_argument("--simt-sms", type=int, default=SIMT_SMS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-cpu", action="store_true", help="e2e without the host-CPU unit")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 strong-scaling measurement")
    ap.add_argument("--c4-steps", type=int, default=10)
    ap.add_argument("--b-panels", type=int, default=16,
                    help="N > 1: B column panels broadcast separately (overlap with compute)")
    ap.add_argument("--b-transport", default="ce", choices=["ce", "nccl"],
                    help="N > 1: how B reaches the ranks -- copy-engine chain over CUDA IPC (no SMs) "
                         "or NCCL broadcasts (kernels beside the GEMM)")
    ap.add_argument("--policy", default="best-subset", choices=["reference", "best-subset"],
                    help="planner policy: the reference algorithm (byte-identical plans) or the "
                         "opt-in best-subset B200 extension")
    ap.add_argument("--alpha", type=float, default=1.0,
                    help="dynamic scheduling: weight of the newest measurement in the model re-fit")
    ap.add_argument("--replan-threshold", type=float, default=2.0,
                    help="dynamic scheduling: re-plan when |makespan error| exceeds this (%%)")
    ap.add_argument("--profile", default=None,
                    help="reuse a poas-profile v1 file for the resident units instead of probing "
                         "('{rank}' is replaced by the rank); probes timed under a profiler are "
                         "meaningless")
    ap.add_argument("--alpha-resident", type=float, default=0.2,
                    help="dynamic scheduling of the resident run: EWMA weight of the newest round")
    ap.add_argument("--warmup-seconds", type=float, default=1.0,
                    help="minimum length of the dynamic warm-up (steady power-capped state)")
    # The resident steps run the tensor pipe continuously, in the deepest
    # power-capped state: their probes follow 1.5 s of warm-up GEMMs and a
    # 60 ms pre-roll each (C3 static error +5.1% -> +0.9%, C4 +8.1% -> +3.6%,
    # two alternating runs each, profiles/r02_probe_regime). The e2e step is
    # link-bound (the tensor unit idles between parts) and the C2/C5 sweep
    # keeps the regime its errors were validated in: 20 ms.
    ap.add_argument("--preroll", type=int, default=60,
                    help="ms of back-to-back launches before each timed GPU-unit probe of the resident "
                         "run (0: cold probes)")
    ap.add_argument("--preroll-e2e", type=int, default=20,
                    help="pre-roll of the e2e run's probes and of the C2/C5 sweep (ms)")
    ap.add_argument("--probe-warmup", type=float, default=1.5,
                    help="seconds of tensor-core GEMMs before profiling (0: probe a cool GPU)")
    ap.add_argument("--no-adapt", action="store_true",
                    help="warm-up runs the static plan (no model re-fit / re-plan)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip BASELINE configs C2 and C5 (rank 0 at N=1; ~30 s)")
    ap.add_argument("--ref-rows", type=int, default=None)
    ap.add_argument("--save", default=None, help="directory for profile/schedule/report artefacts")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    from paper_2209_10245_b200 import poas, shard

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    # One process per GPU (ranks beyond the visible GPUs share them: the
    # multi-rank path exercised on a one-GPU box -- the measured
    # configuration is one GPU per rank).
    local = env_int("LOCAL_RANK", 0) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    transport = args.b_transport
    comm = poas.Comm(shard.comm_name(), rank, world, local) if world > 1 else None
    grp = Group(comm)
    if comm and transport == "nccl":
        # NCCL's broadcast kernels run beside the persistent GEMM on the SMs
        # its budget leaves free (TC_SMS_MULTI): every one of its CTAs must
        # fit there, or the GEMM spins on flags only NCCL can release
        for var in ("NCCL_MAX_NCHANNELS", "NCCL_MAX_CTAS"):
            os.environ.setdefault(var, str(148 - TC_SMS_MULTI))
        comm.init_nccl()
    if args.tc_sms is None:
        args.tc_sms = TC_SMS_MULTI if (world > 1 and transport == "nccl") else TC_SMS
    ClockSampler.prepare(local)
    n = k = args.n
    m_total = args.m_total or args.n * world
    save = Path(args.save) if args.save else None
    if save and rank == 0:
        save.mkdir(parents=True, exist_ok=True)

    g = local  # CUDA ordinal inside this process (CUDA_VISIBLE_DEVICES respected)
    tc_id, simt_id = f"gpu{rank}.tc", f"gpu{rank}.simt"
    # probes pre-rolled (preroll=<ms>: each timed probe follows back-to-back
    # launches of the same GEMM): the sustained, power-capped regime the
    # timed steps run in, not the boost clock of a launch after an idle gap
    units_res = (f"{tc_id}=xpu:dev={g}:sms={args.tc_sms}:dtype=bf16:elem=2:link=fused:probe=8192-16384:"
                 f"preroll={args.preroll};"
                 f"{simt_id}=gpu:dev={g}:sms={args.simt_sms}:exclusive=1:elem=4:link=hbm:probe=512-2048:"
                 f"preroll={args.preroll}")
    # NCCL's kernels need the idle units' SMs: no lending with that transport
    units_exec = units_res + (";lend=0" if (world > 1 and transport == "nccl") else "")

    # ---- predict (this GPU's units, real kernels) + the level-1 link probe
    # Ranks that share a GPU (the multi-rank path exercised on a one-GPU
    # box) probe in turn: concurrent probes would time each other's kernels
    # and skew the level-1 split (one rank was left no rows).
    shared_gpu = world > 1 and torch.cuda.device_count() < env_int("LOCAL_WORLD_SIZE", world)

    def in_turn(fn):
        if not shared_gpu:
            return fn()
        out_ = None
        for r_ in range(world):
            grp.barrier()
            if r_ == rank:
                out_ = fn()
        grp.barrier()
        return out_

    def probe_units():
        # Bring the GPU to the power-capped steady state the timed region
        # runs in before probing (the probes are short GEMMs; on a cool GPU
        # they see burst clocks the sustained run never gets).
        if args.probe_warmup > 0:
            warm_sustained(poas, torch, dev, args.probe_warmup)
        return poas.profile_machine(units_res, PROFILING, bus=True, retries=2)

    t0 = time.perf_counter()
    if args.profile:  # a profile measured earlier on this box (e.g. for an ncu pass)
        profile = Path(args.profile.replace("{rank}", str(rank))).read_text()
    else:
        profile = in_turn(probe_units)
    t_prof = time.perf_counter() - t0
    link_bw = None
    if comm:
        # DeviceBackend::time_transfer of each GPU's level-1 link: B (16-bit)
        # delivered to every rank by the transport the steps use
        b_bytes = k * n * 2
        link_bw = b_bytes / comm.time_broadcast(b_bytes, transport, 3)
    # The Optimize stage's SM-partition decision (B200 extension,
    # poas_b200_plan_partitions): the CUDA-core unit's budget among
    # candidates, from this profile scaled by SM counts. Budget 0 = the unit
    # left out and its SMs lent to the tensor unit, which is what the
    # executor does whenever the plan gives the unit no rows.
    sm_partition = None
    try:
        cand = [0, 2, 4, 8, 16, 32]
        pp = poas.plan_partitions(profile, m_total // world, n, k, tc_id, args.tc_sms, simt_id,
                                  args.simt_sms, cand, args.policy)
        sm_partition = {"candidates": [{"simt_sms": c["simt_sms"], "tc_sms": c["tc_sms"],
                                        "predicted_ms": round(c["makespan"] * 1e3, 4), "rows": c["rows"]}
                                       for c in pp["candidates"]],
                        "chosen_simt_sms": pp["candidates"][pp["best"]]["simt_sms"],
                        "model": "each GPU unit's compute slope scaled inversely with its SM count, the "
                                 "CUDA-core unit's resident-operand bandwidth with its SM count; planned "
                                 f"with policy {args.policy}"}
    except Exception as exc:  # reported, never fatal
        sm_partition = {"error": f"{type(exc).__name__}: {exc}"}
    # Predict again after Optimize: with the CUDA-core unit left out, the
    # executor lends its SMs to the tensor unit, so the tensor unit is probed
    # on that budget and its model spliced into the profile (same machine,
    # same hash). The static prediction then describes the grid that runs:
    # at 8192^3 the 146- and 148-SM grids differ by a whole wave of tiles
    # (8 vs 7), at 16384^3 by 29 vs 28.
    if (not args.profile and isinstance(sm_partition, dict) and sm_partition.get("chosen_simt_sms") == 0
            and not (world > 1 and transport == "nccl")):
        lent_sms = args.tc_sms + args.simt_sms
        units_lent = (f"{tc_id}=xpu:dev={g}:sms={lent_sms}:dtype=bf16:elem=2:link=fused:probe=8192-16384:"
                      f"preroll={args.preroll}")
        def reprobe():
            try:
                return poas.splice_unit(profile, poas.profile_machine(units_lent, PROFILING_TC, bus=True,
                                                                      retries=2), tc_id), None
            except Exception as exc:  # reported; the first profile stands
                return profile, f"{type(exc).__name__}: {exc}"

        profile, err = in_turn(reprobe)
        if err:
            sm_partition["tensor_unit_reprobe_error"] = err
        else:
            sm_partition["tensor_unit_reprobed_on_sms"] = lent_sms
    t_prof = time.perf_counter() - t0
    if save and rank == 0:
        (save / "profile_resident.txt").write_text(profile)
    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")

    def resident_run(label, m_all, n, k, steps, panels_req, adapt=True, full=True):
        """Plan (two-level at N > 1), place the operands, warm up through the
        dynamic scheduler and time `steps` executor steps of the row-sharded
        GEMM (B broadcast by the library inside every step at N > 1)."""
        if world > 1:
            plan = shard.plan(grp.allgather(profile), [link_bw] * world, m_all, n, k, args.policy)
            rows_l1, row0 = plan["rows"], plan["row0"][rank]
            m = rows_l1[rank]
            if m == 0:
                raise SystemExit(f"rank {rank}: the level-1 plan left this GPU no rows ({rows_l1})")
            schedule = json.dumps(plan["plans"][rank])
            schedule = poas.schedule_roundtrip(schedule)
        else:
            rows_l1, row0, m = [m_all], 0, m_all
            schedule = poas.plan_policy(profile, m, n, k, args.policy)
        ref_policy_makespan = json.loads(poas.plan(profile, m, n, k))["makespan"]
        sched = json.loads(schedule)
        rows = {d["id"]: d["rows"] for d in sched["devices"]}
        log(f"rank {rank} {label}: level-1 rows {rows_l1}; plan rows {rows}; "
            f"predicted {sched['makespan']*1e3:.3f} ms")
        if save and rank == 0:
            (save / f"schedule_{label}.json").write_text(schedule)
        P = panels_req if world > 1 else 1
        while P > 1 and (n % P or (n // P) % 256):  # panels of whole pair tiles (one-launch path)
            P //= 2
        np_ = n // P
        A32 = torch.empty(m, k, device=dev, dtype=torch.float32)
        A16 = torch.empty(m, k, device=dev, dtype=torch.bfloat16)
        C = torch.empty(m, n, device=dev, dtype=torch.float32)
        # B panel-major ([P][K][N/P]): each column panel is one contiguous
        # chunk of the broadcast; only rank 0 holds it
        B32 = torch.zeros(P, k, np_, device=dev, dtype=torch.float32)
        B16 = torch.zeros(P, k, np_, device=dev, dtype=torch.bfloat16)
        poas.fill_uniform(poas.DTYPE_F32, A32.data_ptr(), k, m, k, row0, 0, k, sa)
        poas.fill_uniform(poas.DTYPE_BF16, A16.data_ptr(), k, m, k, row0, 0, k, sa)

        def fill_b():
            for p in range(P):
                poas.fill_uniform(poas.DTYPE_F32, B32[p].data_ptr(), np_, k, np_, 0, p * np_, n, sb)
                poas.fill_uniform(poas.DTYPE_BF16, B16[p].data_ptr(), np_, k, np_, 0, p * np_, n, sb)

        if rank == 0:
            fill_b()
        torch.cuda.synchronize()
        wcomm = None
        if world > 1:
            # one communicator per workload (its B registration)
            wcomm = comm if label == "main" else poas.Comm(shard.comm_name() + "_" + label, rank, world, local)
            if transport == "nccl" and wcomm is not comm:
                wcomm.init_nccl()
            wcomm.register_b(B16.data_ptr(), B32.data_ptr(), k, n, P)
        ex = poas.Executor(units_exec)
        io = poas.GemmIO(m=m, n=n, k=k, a_dev=A32.data_ptr(), lda_dev=k, b_dev=B32.data_ptr(), ldb_dev=np_,
                         a16_dev=A16.data_ptr(), lda16_dev=k, b16_dev=B16.data_ptr(), ldb16_dev=np_,
                         c_dev=C.data_ptr(), ldc_dev=n, resident=1, b_panels=P,
                         comm=wcomm.handle if wcomm else None, b_transport=poas.TRANSPORTS[transport])

        # Warm-up = dynamic scheduling (paper §3.4.2, poas_b200_run_dynamic):
        # the probes are short bursts, the timed region runs at the sustained
        # power-capped clock; each warm-up execution re-fits the unit models
        # from its measured phases and re-plans. The first one runs the
        # static plan, so its error is the static model's prediction error.
        # Rounds of 5 back-to-back steps (single steps with host gaps run
        # cooler), for >= --warmup-seconds in all; EWMA re-fit (alpha 0.2:
        # under the power cap a 60 ms block wanders +-8%,
        # profiles/r01_warmup). At N > 1 every rank runs the same number of
        # executions (each one is a collective broadcast).
        ex.execute(schedule, io, 1)
        warm_reps = 5
        warm_iters = min(400, max(args.warmup, int(args.warmup_seconds / max(sched["makespan"] * warm_reps,
                                                                             1e-6)) + 1))
        if args.no_adapt or not adapt:
            warm_iters, warm_reps = args.warmup, 1
        warm_iters = int(grp.max(warm_iters))
        with ClockSampler(g) as warm_clk:  # the clocks the re-fit saw (last half of the warm-up)
            dyn = ex.run_dynamic(profile, m, n, k, io, iterations=warm_iters, policy=args.policy,
                                 alpha=args.alpha_resident, repeats=warm_reps,
                                 replan_threshold_pct=1e9 if (args.no_adapt or not adapt) else args.replan_threshold)
        warm_mhz = [x[0] for x in warm_clk.samples[len(warm_clk.samples) // 2:]]
        warm_sm_mhz = float(statistics.median(warm_mhz)) if warm_mhz else None
        schedule = poas.schedule_roundtrip(json.dumps(dyn["schedule"]))
        sched = json.loads(schedule)
        rows = {d["id"]: d["rows"] for d in sched["devices"]}
        log(f"rank {rank} {label}: dynamic warm-up {[round(i['makespan_error_pct'], 2) for i in dyn['iterations']]} % "
            f"-> rows {rows}, predicted {sched['makespan']*1e3:.3f} ms")
        if save and rank == 0:
            (save / f"dynamic_{label}.json").write_text(json.dumps(dyn, indent=1))

        # ---- the timed region: `steps` executor steps back to back (at N > 1
        # each one broadcasts B), bracketed by a barrier + synchronize, CUDA
        # events around them on the current stream (the executor's units
        # start behind an event recorded on it), SM clocks sampled during.
        # the run's one-time costs, untimed: a one-unit resident plan replays
        # its steps as one CUDA graph, captured for this schedule, operands
        # and step count on first use
        ex.execute(schedule, io, steps)
        grp.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # Keep the GPU at the steps' duty cycle across the host work before
        # the timed region (clock sampler start, enqueueing the first step):
        # an idle gap of a few ms lets the power cap's controller recover,
        # and a short timed region then runs up to 14% faster than the
        # steady state the model was fit in (profiles/r01_warmup).
        s_cur = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            poas.tc_gemm(poas.DTYPE_BF16, m, np_, k, A16.data_ptr(), k, B16[0].data_ptr(), np_,
                         C.data_ptr(), n, stream=s_cur)
        with ClockSampler(g) as clk:
            e0.record()
            rep = ex.execute(schedule, io, steps)
            e1.record()
            torch.cuda.synchronize()
        grp.barrier()
        ms_total = grp.max(e0.elapsed_time(e1))
        ms_step = ms_total / steps

        # ---- check C (every rank, full size, outside the timed region):
        # (1) C.x = A_u.(B_u.x) in fp64 over all of C; (2) 64 sampled full
        # rows (first/last, tile boundaries, random) against fp64 products
        # of the same rounded operands -- the arithmetic of the tests' CPU
        # oracle (tests/test_gpu_fullsize.py), here with torch in fp64. The
        # ranks that received B regenerate it locally for the reference.
        if rank != 0:
            fill_b()
        x = torch.randn(n, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(7))
        xs = x.view(P, np_)
        y = C.double() @ x
        y_ref = torch.empty_like(y)
        gen = torch.Generator().manual_seed(5 + rank)
        picks = {0, m - 1}
        for t in range(0, max(1, m // 256), max(1, m // 256 // 12)):
            picks.update(r for r in (t * 256, t * 256 + 127, t * 256 + 128, t * 256 + 255) if r < m)
        while len(picks) < min(64, m):
            picks.add(int(torch.randint(0, m, (1,), generator=gen)))
        rows_s = sorted(picks)[:64]
        num = den = num_x = den_x = 0.0
        r0 = 0
        for d_ in sched["devices"]:
            r = d_["rows"]
            if r == 0:
                continue
            Bu, Au = (B16, A16) if d_["id"] == tc_id else (B32, A32)
            bx = sum(Bu[p].double() @ xs[p] for p in range(P))
            y_ref[r0:r0 + r] = Au[r0:r0 + r].double() @ bx
            sel = [i for i in rows_s if r0 <= i < r0 + r]
            if sel:
                idx = torch.tensor(sel, device=dev)
                Ar = Au.index_select(0, idx).double()
                ref_rows = torch.cat([Ar @ Bu[p].double() for p in range(P)], dim=1)
                num += float((C.index_select(0, idx).double() - ref_rows).norm() ** 2)
                den += float(ref_rows.norm() ** 2)
                # the same rows from the UNROUNDED fp32 operands (BASELINE.md
                # section 3: bf16 <= 8e-3, fp16 <= 2e-3; reported, not gated)
                A32r = A32.index_select(0, idx).double()
                exact = torch.cat([A32r @ B32[p].double() for p in range(P)], dim=1)
                num_x += float((C.index_select(0, idx).double() - exact).norm() ** 2)
                den_x += float(exact.norm() ** 2)
            r0 += r
        c_prop = grp.max(float((y - y_ref).norm() / y_ref.norm()))
        c_rows = grp.max((num / den) ** 0.5 if den > 0 else 0.0)
        # relative Frobenius bound for fp32 accumulation over K (SURVEY.md
        # 8d): 2e-5 up to K = 16384 (1.79e-5 measured
        # there, as cuBLAS), growing linearly with K beyond
        tol = 2e-5 * max(1.0, k / 16384)
        if not (c_prop <= tol and c_rows <= tol):
            raise SystemExit(f"{label}: C check failed: rel err {c_prop:.3e} / sampled rows {c_rows:.3e} > {tol}")
        c_check = {"property": "C.x = A.(B.x), fp64, each unit's own operand precision, every rank",
                   "max_rel_err": float(f"{c_prop:.3e}"), "tol": tol,
                   "sampled_rows": {"rows": len(rows_s), "rel_frobenius": float(f"{c_rows:.3e}"),
                                    "reference": "fp64 product of the same rounded operands (first/last, "
                                                 "128/256-row tile boundaries, random rows; every rank)",
                                    "vs_unrounded_inputs": float(f"{grp.max((num_x / den_x) ** 0.5 if den_x > 0 else 0.0):.3e}"),
                                    "vs_unrounded_bound": "bf16 8e-3 (BASELINE.md 3)"}}
        meas_make = rep["measured_makespan"]
        pred_make = rep["predicted_makespan"]
        it0 = dyn["iterations"][0]
        static_same = it0["rows"] == rows
        static_pred = it0["predicted_makespan"]
        # makespan error of the profile-only (static) prediction, job-wide:
        # the slowest rank's measured step against the slowest predicted
        meas_job = grp.max(meas_make)
        pred_job = grp.max(static_pred if static_same else pred_make)
        pred_adapt_job = grp.max(pred_make)
        out = {
            "label": label, "m": m, "rows_l1": rows_l1, "row0": row0, "P": P, "ms_step": ms_step,
            "value": 2.0 * m_all * n * k / (ms_step * 1e-3) / 1e12, "clocks": clk.summary(),
            "schedule": schedule, "sched": sched, "rows": rows, "dyn": dyn, "rep": rep,
            "c_check": c_check, "ref_policy_makespan": ref_policy_makespan, "warm_sm_mhz": warm_sm_mhz,
            "static_same": static_same, "meas_job": meas_job, "pred_job": pred_job,
            "pred_adapt_job": pred_adapt_job, "warm_reps": warm_reps, "ex": ex, "io": io,
            "A16": A16, "B16": B16, "C": C, "comm": wcomm, "np": np_,
        }
        if save and rank == 0:
            (save / f"report_{label}.json").write_text(json.dumps(rep, indent=1))
        return out

    main_res = resident_run("main", m_total, n, k, args.steps, args.b_panels)
    m, row0 = main_res["m"], main_res["row0"]
    sched, rows, schedule = main_res["sched"], main_res["rows"], main_res["schedule"]
    ex, io, A16, B16, C = main_res["ex"], main_res["io"], main_res["A16"], main_res["B16"], main_res["C"]
    P, np_, dyn, rep_last = main_res["P"], main_res["np"], main_res["dyn"], main_res["rep"]
    ms_step, value, clocks = main_res["ms_step"], main_res["value"], main_res["clocks"]

    # roofline: the tensor kernel's launch inside the timed steps
    tc_compute = rep_last["devices"][[d["id"] for d in rep_last["devices"]].index(tc_id)]["compute"]["measured"] \
        if tc_id in [d["id"] for d in rep_last["devices"]] else 0.0
    tc_rows = rows.get(tc_id, 0)
    peak_burst, peak_sust, peak_kind = measured_peaks()
    achieved = 2.0 * tc_rows * n * k / tc_compute / 1e12 if tc_compute > 0 else 0.0
    traffic = None
    tp = ROOT / "profiles" / "tc_gemm_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(str(args.n))
        except Exception:
            traffic = None

    # ---- speedup vs best single unit (the tensor unit; the 2-SM CUDA-core
    # unit alone is predicted ~3 orders of magnitude slower). Co-executed and
    # standalone steps alternate so both see the same power/thermal state
    # (sw_power_cap drifts over a run); medians of the per-step makespans.
    s_sched = poas.plan_standalone(profile, tc_id, m, n, k)
    for _ in range(2):
        ex.execute(s_sched, io, 1)
    pair_co, pair_alone = [], []
    for _ in range(max(3, args.steps // 2)):
        pair_co.append(ex.execute(schedule, io, 1)["measured_makespan"])
        pair_alone.append(ex.execute(s_sched, io, 1)["measured_makespan"])
    best_single = statistics.median(pair_alone)
    simt_alone_pred = json.loads(poas.plan_standalone(profile, simt_id, m, n, k))["makespan"]
    co_median = statistics.median(pair_co)
    speedup = best_single / co_median if co_median > 0 else None

    # tensor-core-only on every SM (what a non-POAS caller would run)
    sms_all = poas.sm_count()
    tc_all_ms = cublas_ms = cublas_rel = None
    if world == 1:
        # Our tensor kernel on every SM beside cuBLAS (torch.mm bf16 -> fp32
        # out, the library the measured peak comes from) on the same operands,
        # alternating launches so both see the same power-cap state. cuBLAS is
        # a timing reference only; nothing on the POAS path calls it.
        s = torch.cuda.current_stream().cuda_stream
        B16m = B16[0]
        C_lib = torch.empty(m, n, device=dev, dtype=torch.float32)

        def ours():
            poas.tc_gemm(poas.DTYPE_BF16, m, n, k, A16.data_ptr(), k, B16.data_ptr(), n, C.data_ptr(), n,
                         stream=s)

        def lib():
            torch.mm(A16, B16m, out_dtype=torch.float32, out=C_lib)

        for _ in range(3):
            ours()
            lib()
        torch.cuda.synchronize()
        t_ours, t_lib = [], []
        for _ in range(5):
            for fn, acc in ((ours, t_ours), (lib, t_lib)):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                fn()
                a1.record()
                torch.cuda.synchronize()
                acc.append(a0.elapsed_time(a1))
        tc_all_ms = statistics.median(t_ours)
        cublas_ms = statistics.median(t_lib)
        # cuBLAS's C under the same property check, for scale
        xg = torch.randn(n, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(7))
        yr = A16.double() @ (B16m.double() @ xg)
        cublas_rel = float((C_lib.double() @ xg - yr).norm() / yr.norm())
        del C_lib, yr

    # ---- C4 (BASELINE config 4): 65536 x 8192 x 8192 row-sharded over the
    # ranks -- strong scaling (total work fixed), measured in the same run
    c4 = None
    if not args.no_c4 and not args.m_total:
        r4 = resident_run("c4", 65536, 8192, 8192, args.c4_steps, args.b_panels, adapt=True)
        c4 = {"workload": f"C4: M=65536 x N=K=8192 row-sharded over {world} GPU(s), B broadcast from rank 0",
              "scaling": "strong", "value": round(r4["value"], 3), "unit": "TFLOP/s",
              "ms_per_step": round(r4["ms_step"], 4), "steps": args.c4_steps,
              "level1_rows_per_gpu": r4["rows_l1"], "plan_rows": r4["rows"],
              "b_panels": r4["P"], "b_transport": transport if world > 1 else None,
              "predicted_makespan_ms": round(r4["pred_job"] * 1e3, 4),
              "measured_makespan_ms": round(r4["meas_job"] * 1e3, 4),
              "makespan_error_pct": round(100.0 * (r4["meas_job"] - r4["pred_job"]) / r4["meas_job"], 3),
              "adapted_makespan_error_pct": round(100.0 * (r4["meas_job"] - r4["pred_adapt_job"])
                                                  / r4["meas_job"], 3),
              "c_check": r4["c_check"], "clocks": r4["clocks"]}
        del r4

    # ---- e2e through the C ABI with host buffers over PCIe. Headline: the
    # tensor unit's link carries 16-bit A/B (the reference's XPU link model,
    # elem_size 2; the workload's operand precision, as in the resident run)
    # with overlapped copies (planner policy "overlap" + executor
    # "overlap=1": A row parts and B column panels host->device while
    # earlier blocks compute and their C goes device->host)
    # and consecutive steps pipelined ("pipeline=1"). Alongside: every step
    # isolated, fp32 host A/B converted on the GPU, and the paper's
    # synchronous copies (copy-in, compute, copy-out per unit). CPU-side
    # units (host cores, the CUDA-core unit's fp32 operands) read the fp32
    # host copies.
    e2e = None
    if not args.no_e2e:
        hA = torch.empty(m, k, dtype=torch.float32, pin_memory=True)
        hB = torch.empty(k, n, dtype=torch.float32, pin_memory=True)
        hC = torch.empty(m, n, dtype=torch.float32, pin_memory=True)
        poas.fill_uniform_host(hA.data_ptr(), k, m, k, row0, 0, k, sa)
        poas.fill_uniform_host(hB.data_ptr(), n, k, n, 0, 0, n, sb)
        hA16 = hA.bfloat16().pin_memory()  # RNE, bit-identical to the device conversion
        hB16 = hB.bfloat16().pin_memory()
        local_world = env_int("LOCAL_WORLD_SIZE", world)
        e2e_profiles = {}

        def run_e2e(tc_elem, overlap, pipeline=False):
            units_e2e = units_res.replace("elem=2:link=fused", f"elem={tc_elem}:link=pcie").replace(
                "elem=4:link=hbm", "elem=4:link=pcie").replace(f"preroll={args.preroll}",
                                                               f"preroll={args.preroll_e2e}")
            if not args.no_e2e_cpu:
                # With host-resident operands the host cores are a unit too:
                # they compute rows in place while the GPU units' copies hold
                # the link (the box's cores shared by the ranks on this node).
                threads = max(1, ((os.cpu_count() or 2) - 2) // max(1, local_world))
                units_e2e += f";cpu{rank}=cpu:threads={threads}"
            policy = "overlap" if overlap else args.policy
            if tc_elem not in e2e_profiles:  # same units either way: probe once
                e2e_profiles[tc_elem] = poas.profile_machine(
                    units_e2e, PROFILING + ",cpu_min_side=1024,cpu_max_side=2048", bus=True, retries=2)
            prof_e2e = e2e_profiles[tc_elem]
            ref_e2e = json.loads(poas.plan(prof_e2e, m, n, k))
            ex_e2e = poas.Executor(units_e2e + (";overlap=1" if overlap else "")
                                   + (";pipeline=1" if pipeline else ""))
            io_h = poas.GemmIO(m=m, n=n, k=k, a_host=hA.data_ptr(), lda_host=k, b_host=hB.data_ptr(),
                               ldb_host=n, c_host=hC.data_ptr(), ldc_host=n, resident=0)
            if tc_elem == 2:
                io_h.a16_host, io_h.lda16_host = hA16.data_ptr(), k
                io_h.b16_host, io_h.ldb16_host = hB16.data_ptr(), n
            # dynamic scheduling warm-up (as for the resident run): the host
            # unit's probes (sides <= 2048, cache-resident B) cannot see the
            # 1 GiB B stream of the real share; measured runs re-fit it.
            dyn_e2e = ex_e2e.run_dynamic(prof_e2e, m, n, k, io_h, iterations=max(args.warmup, 6),
                                         policy=policy, alpha=args.alpha,
                                         replan_threshold_pct=args.replan_threshold)
            sched_e2e = poas.schedule_roundtrip(json.dumps(dyn_e2e["schedule"]))
            se = json.loads(sched_e2e)
            ex_e2e.execute(sched_e2e, io_h, 3)  # a multi-step run's one-time costs, untimed
            # probe (before, and apart from, the timed steps): 3 steps back to
            # back -- decides between pipelined and isolated steps below
            t_probe = time.perf_counter()
            ex_e2e.execute(sched_e2e, io_h, 3)
            probe_ms = (time.perf_counter() - t_probe) / 3 * 1e3
            grp.barrier()
            steps_e2e = max(3, args.steps)
            t0 = time.perf_counter()
            r_e2e = ex_e2e.execute(sched_e2e, io_h, steps_e2e)
            wall = grp.max(time.perf_counter() - t0)
            linked = [d for d in se["devices"] if d["rows"] > 0 and not d["id"].startswith("cpu")]
            # bytes crossing the link per step: each GPU unit's A rows and all
            # of B in its link element size, its C rows in fp32
            esz = {d["id"]: (tc_elem if d["id"] == tc_id else 4) for d in linked}
            h2d = sum(esz[d["id"]] * (d["rows"] * k + k * n) for d in linked)
            d2h = sum(4 * d["rows"] * n for d in linked)
            ms = wall / steps_e2e * 1e3
            out = {"value": round(2.0 * m_total * n * k / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                   "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                   "ms_per_step": round(ms, 3), "steps": steps_e2e, "probe_ms_per_step": round(probe_ms, 3),
                   # link roofline: the busiest direction's bytes at the
                   # profiled link bandwidth (full duplex when overlapped)
                   "link_bound_ms": None,
                   "plan_rows": {d["id"]: d["rows"] for d in se["devices"]},
                   "row_parts": {d["id"]: len(d["tiles"]) for d in linked} if overlap else None,
                   "policy": policy,
                   "reference_policy_plan_rows": {d["id"]: d["rows"] for d in ref_e2e["devices"]},
                   "reference_policy_predicted_ms": round(ref_e2e["makespan"] * 1e3, 4),
                   "predicted_makespan_ms": round(r_e2e["predicted_makespan"] * 1e3, 4),
                   "measured_makespan_ms": round(r_e2e["measured_makespan"] * 1e3, 4),
                   "makespan_error_pct": round(r_e2e["makespan_error_pct"], 3),
                   "static_plan": _static_summary(dyn_e2e),
                   "dynamic_replans": dyn_e2e["replans"],
                   "units": units_e2e + (";overlap=1" if overlap else "") + (";pipeline=1" if pipeline else ""),
                   "gemm_latency_ms": round(r_e2e["measured_makespan"] * 1e3, 3),
                   "path": "poas_b200_execute (C ABI), pinned host "
                           + ("bf16 A/B for the tensor unit (fp32 for the others)" if tc_elem == 2
                              else "fp32 A/B converted on the GPU")
                           + ", fp32 C; H2D + compute + D2H in every step"
                           + ("; copies overlapped with compute (row parts x column panels)" if overlap
                              else "; synchronous copies (the paper's scheme)")
                           + ("; consecutive steps pipelined (step i+1's copies start beside step i's "
                              "copy-out tail)" if pipeline else "")}
            bw = [float(ln.split()[1]) for ln in prof_e2e.splitlines() if ln.startswith("bandwidth ")]
            bw = max(bw) if bw else 0.0
            if bw > 0:
                link_s = max(h2d, d2h) / bw if overlap else (h2d + d2h) / bw
                out["link_bound_ms"] = round(link_s * 1e3, 3)
                out["link_bandwidth_gbs"] = round(bw / 1e9, 2)
            if overlap and rank == 0:
                # the link measured as the overlapped step uses it: this
                # step's H2D and D2H bytes at once, contiguous 64 MiB copies
                # (one stream per direction; more streams do not help,
                # profiles/r02_pcie) -- the practical floor of the step
                cl = concurrent_link_ms(torch, h2d, d2h)
                if cl:
                    out["link_concurrent_ms"] = round(cl, 3)
                    out["link_frac"] = round(cl / out["ms_per_step"], 3)
            if save and rank == 0:
                tag = ("e2e" if tc_elem == 2 else "e2e_fp32") + ("" if overlap else "_sync") + (
                    "_pipelined" if pipeline else "")
                (save / f"profile_{tag}.txt").write_text(prof_e2e)
                (save / f"dynamic_{tag}.json").write_text(json.dumps(dyn_e2e, indent=1))
                (save / f"report_{tag}.json").write_text(json.dumps(r_e2e, indent=1))
                (save / f"schedule_{tag}.json").write_text(sched_e2e)
            return out

        # headline: a stream of GEMMs, each step's copies and GEMM overlapped
        # and consecutive steps pipelined; beside it the same with every step
        # isolated (its latency is the per-GEMM makespan), fp32 host operands,
        # and the paper's synchronous copies. Pipelining is an executor mode
        # the adapt stage picks per box: each mode's 3-step probe (measured
        # before either's timed steps) decides the headline (on most boxes it
        # wins, 23.5 vs 29-30 ms; on a box with a weak host side the two
        # directions' DMA contend and it lost, profiles/r01_overlap).
        piped = run_e2e(2, overlap=True, pipeline=True)
        single = run_e2e(2, overlap=True)
        choose_piped = grp.max(1.0 if piped["probe_ms_per_step"] <= single["probe_ms_per_step"] else 0.0) > 0
        if choose_piped:
            e2e, e2e["single_step"] = piped, single
            # The planner predicts one GEMM's makespan (its overlap
            # timeline). The isolated steps measure exactly that. A
            # pipelined step's latency also holds its neighbours' copies
            # (step i+1's copy-in shares the link with step i's copy-out),
            # so it is reported beside the prediction error, not as it.
            e2e["pipelined_latency"] = {key: e2e[key] for key in
                                        ("predicted_makespan_ms", "measured_makespan_ms", "makespan_error_pct")}
            for key in ("predicted_makespan_ms", "measured_makespan_ms", "makespan_error_pct"):
                e2e[key] = single[key]
            e2e["makespan_error_basis"] = ("predicted one-GEMM makespan vs the isolated-step run "
                                           "(single_step); the pipelined latency beside it")
        else:
            e2e, e2e["pipelined"] = single, piped
        e2e["mode_choice"] = ("pipelined" if e2e is piped else "single_step") + \
            f" (probe {piped['probe_ms_per_step']} vs {single['probe_ms_per_step']} ms per step)"
        e2e["fp32_host"] = run_e2e(4, overlap=True)
        e2e["synchronous"] = run_e2e(2, overlap=False)

    # ---- CPU baselines (rank 0 at N=1 only): the reference's CPU path (the
    # oracle port executing the reference planner's CPU-only plan) and,
    # beside it, this repo's own host-CPU unit (AVX-512 host_gemm) on the
    # same host cores, so the GPU/CPU ratio has a competent CPU path next
    # to it; plus the reference planner's own cost
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            tfl, sec, sample, cores = reference_cpu_path(args.n, sample_rows=args.ref_rows, reps=1)
            cpu_baseline = {"value": round(tfl, 4), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                            "sample": sample, "cpu_model": cpu_model()}
            # each extra reported on its own: a noisy host probe fit (the
            # reference's fit_linear rejects a non-positive slope) must not
            # take the reference CPU path's number with it
            for key, fn in (("host_unit", lambda: host_unit_baseline(poas, args.n)),
                            ("reference_planner", lambda: reference_planner_cost(profile, m, n, k))):
                try:
                    cpu_baseline[key] = fn()
                except Exception as exc:
                    cpu_baseline[key] = {"error": f"{type(exc).__name__}: {exc}"}
        except Exception as exc:  # reported, never fatal
            cpu_baseline = {"value": None, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
                            "sample": f"unavailable: {exc}"}

    # ---- BASELINE configs C2 and C5 (rank 0 at N=1 only; tools/sweep.py):
    # C2 = 8192^3 co-executed by host CPU + fp32 CUDA cores + fp16 tensor
    # cores; C5 = square sizes 1024..32768, the POAS plan (static prediction
    # error, then the dynamic re-plan) vs tensor cores alone on every SM vs
    # the cuBLAS timing reference vs the host-CPU unit. Reported, never fatal.
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        try:
            sys.path.insert(0, str(ROOT / "tools"))
            import sweep as sw

            t_sw = time.perf_counter()
            c5 = sw.c5([1024, 2048, 4096, 8192, 16384, 32768], args.preroll_e2e)
            c2 = sw.c2()
            sv = sw.simt_vs_cublas_fp32()
            keep = ("n", "plan_rows", "static_error_pct", "poas_tflops", "adapted_error_pct",
                    "tc_only_148sm_tflops", "cublas_bf16_fp32out_tflops", "host_cpu_tflops", "host_cores")
            sweep = {
                "c5": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if k in keep}
                       for r in c5["rows"]],
                "c5_note": "POAS = the plan after the dynamic warm-up (static_error_pct: the profile-only "
                           "plan against its own timed steps); tc_only = our tensor kernel on every SM; "
                           "cublas = torch.mm bf16->fp32 (timing reference only); resident operands, "
                           "sustained regime (graph-replayed steps lasting >= 0.25 s)",
                "c2": {"n": c2["n"], "tflops": round(c2["tflops"], 3), "plan_rows": c2["plan_rows"],
                       "static_plan_rows": c2["static_plan"]["rows"],
                       "static_error_pct": round(c2["static_plan"]["makespan_error_pct"], 3),
                       "makespan_error_pct": round(c2["makespan_error_pct"], 3),
                       "units": "host CPU (AVX-512) + fp32 CUDA cores (2 SMs) + fp16 tensor cores (146 SMs)"},
                "simt_vs_cublas_fp32": dict(
                    {k: (round(v, 3) if isinstance(v, float) else v) for k, v in sv.items()},
                    # FP32 pipe: 148 SMs x 128 lanes x 2 flop x 1965 MHz
                    fp32_peak_tflops=round(148 * 128 * 2 * 1.965e9 / 1e12, 1),
                    frac_of_fp32_peak=round(sv["simt_all_sms_tflops"] / (148 * 128 * 2 * 1.965e9 / 1e12), 3)),
                "seconds": round(time.perf_counter() - t_sw, 1)}
        except Exception as exc:  # reported, never fatal
            sweep = {"error": f"{type(exc).__name__}: {exc}"}

    # per step: one GEMM launch per busy unit (the tensor unit consumes all
    # B panels in one launch; a CUDA-core unit launches once per panel),
    # plus the executor's start-gate kernel on this GPU -- except when the
    # executor replays the steps as one CUDA graph (resident operands, one
    # busy GPU unit, one panel, no communicator, <= 256 repeats: executor.cpp
    # graph_mode), which has no gate
    busy = [d for d in sched["devices"] if d["rows"] > 0]
    graph_replay = (world == 1 and P <= 1 and len(busy) == 1 and args.steps <= 256
                    and os.environ.get("POAS_EXEC_GRAPH") != "0")
    launches_per_step = sum((1 if d["id"] == tc_id else P) for d in busy) + (0 if graph_replay else 1)
    meas_make, pred_job, pred_adapt = main_res["meas_job"], main_res["pred_job"], main_res["pred_adapt_job"]
    static_same = main_res["static_same"]
    if rank == 0:
        line = {
            "metric": "co-executed GEMM TFLOP/s at N=16384 (1/2/4/8 B200); speedup vs best single unit",
            "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong" if args.m_total else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": (f"C4: M={m_total} x N=K={args.n} row-sharded over {world} GPU(s)" if args.m_total
                             else f"C3: square GEMM N={args.n} per GPU (M={args.n}*{world})")
                            + ", bf16 tensor-core + fp32 CUDA-core co-execution planned by POAS; at N>1 B "
                              "broadcast from rank 0 by the library inside every step",
                "m": m_total, "n": n, "k": k, "parallelism": f"POAS row split x {world} GPU(s)",
                "level1_rows_per_gpu": main_res["rows_l1"],
                "units": {tc_id: f"tcgen05 bf16->fp32 on {args.tc_sms} SMs",
                          simt_id: f"fp32 SIMT on {args.simt_sms} SMs"},
                "planner_policy": args.policy,
                "reference_policy_predicted_ms": round(main_res["ref_policy_makespan"] * 1e3, 4),
                "plan_rows": rows, "l2": (f"inputs larger than L2 (per rank: A {m * k * 2 / 2**20:.0f} MiB + B "
                                          f"{k * n * 2 / 2**20:.0f} MiB bf16, fp32 copies twice that; L2 126 MB)"
                                          if (m * k + k * n) * 2 > 126e6 else "inputs fit in L2 (small size)"),
                # the paper's scheduler is static: its prediction is the
                # profile's, for the plan that ran (same rows); the dynamic
                # re-fit's prediction is reported beside it. Job-wide: the
                # slowest rank's step against the slowest prediction.
                "predicted_makespan_ms": round(pred_job * 1e3, 4),
                "measured_makespan_ms": round(meas_make * 1e3, 4),
                "makespan_error_pct": round(100.0 * (meas_make - pred_job) / meas_make, 3),
                "prediction": ("profile-only (static POAS, the paper's scheduler) for the plan that ran, "
                               "against the timed steps" if static_same else
                               "adapted (the profile-only plan differed from the plan that ran)"),
                "adapted": {"predicted_makespan_ms": round(pred_adapt * 1e3, 4),
                            "makespan_error_pct": round(100.0 * (meas_make - pred_adapt) / meas_make, 3),
                            "warmup_sm_mhz": main_res["warm_sm_mhz"],
                            "note": "dynamic scheduling: warm-up runs re-fit the profile (EWMA); under "
                                    "the power cap a short timed region can run in a boost phase the "
                                    "re-fit did not see (profiles/r01_warmup)"},
                "static_plan": _static_summary(dyn),
                "dynamic_replans": dyn["replans"],
                "dynamic_warmup_iterations": len(dyn["iterations"]),
                "dynamic_warmup_steps_per_iteration": main_res["warm_reps"],
                "speedup_vs_best_single_unit": round(speedup, 4) if speedup else None,
                "best_single_unit": {"id": tc_id, "measured_makespan_ms": round(best_single * 1e3, 4),
                                     "coexec_paired_makespan_ms": round(co_median * 1e3, 4),
                                     "pairs": len(pair_co)},
                "simt_standalone_predicted_ms": round(simt_alone_pred * 1e3, 2),
                "tc_only_all_sms_tflops": round(2.0 * m * n * k / (tc_all_ms * 1e-3) / 1e12, 2)
                if tc_all_ms else None,
                "cublas_bf16_fp32out_tflops": round(2.0 * m * n * k / (cublas_ms * 1e-3) / 1e12, 2)
                if cublas_ms else None,
                "sm_count": sms_all, "profile_seconds": round(t_prof, 2),
                "c_check": dict(main_res["c_check"], **({"cublas_rel_err": float(f"{cublas_rel:.3e}")}
                                                         if cublas_rel is not None else {})),
                "b_transport": (f"{transport}: " + ("copy-engine chain over CUDA IPC (rank r pulls each "
                                                    "panel from rank r-1), no SMs" if transport == "ce"
                                                    else "ncclBroadcast per panel")) if world > 1 else None,
                "level1_link_gbs": round(link_bw / 1e9, 2) if link_bw else None,
                "b_panels": P,
                "c4": c4,
                "sm_partition": sm_partition,
                "sweep": sweep,
            },
            # the tensor kernel is timed inside a long back-to-back run under
            # the power cap: the measured SUSTAINED cuBLAS figure is its
            # denominator (B200_PROFILING.md); the burst one is kept beside it
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2),
                         "peak": peak_sust or peak_burst, "unit": "TFLOP/s",
                         "frac": round(achieved / (peak_sust or peak_burst), 4),
                         "peak_burst": peak_burst, "frac_burst": round(achieved / peak_burst, 4),
                         "traffic": traffic,
                         # the ncu DRAM bytes per launch over this run's
                         # launch time: the kernel's achieved HBM bandwidth
                         "hbm_achieved_gbs": (round(traffic / tc_compute / 1e9, 1)
                                              if traffic and tc_compute > 0 else None),
                         "hbm_peak_gbs": hbm_peak(),
                         "kernel": f"{poas.tc_kernel_name(tc_rows, n, k)} "
                                   f"({poas.tc_scheduler_name(tc_rows, n, k)} tile scheduler)",
                         "peak_kind": (f"of {peak_kind}: bf16 sustained (cuBLAS seconds-long loop under the "
                                       f"power cap), the kernel being timed inside {args.steps} back-to-back "
                                       f"steps" if peak_sust else f"of {peak_kind}: bf16 burst")},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    grp.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
