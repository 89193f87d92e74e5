"""Benchmark engine: timing protocol, verification, target registry.

Drop-in for the reference's ``csrk.bench`` (pkg/src/csrk/bench.py).  The
protocol is unchanged -- ``warmups`` untimed runs, then ``reps`` timed runs,
arithmetic mean, only the multiply inside the window, reorder / pack timed
separately (bench.py:85-105, 212-326) -- but every target executes on the
device with x and y resident in HBM, as the paper times GPU kernels
(PAPER.md:643-644).  Each step synchronises the device before returning, so
wall clocks stay valid; :class:`CudaEventClock` swaps in device-event time.

Targets (TARGETS, the registration point of reference bench.py:58, 169-178):

  ref        plain CSR kernel (bits of spmv_csr_ref)
  cpu2/cpu3  CSR-2 / CSR-3 streaming kernel (bits of spmv_csr2 / spmv_csr3)
  gpu3-emu   PAPER Listing 3 kernel (bits of emulate_gpu_spmv3)
  gpu35-emu  PAPER Listing 4 kernel (bits of emulate_gpu_spmv35)
  cuda3      B200 streaming kernel, serial rows   (== cpu3 bits)
  cuda35     B200 streaming kernel, strided rows  (== gpu35-emu bits)
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import asdict, dataclass

import numpy as np

from . import _native as nat
from .format import CsrMatrix, pack_csrk, permute_vector, unpermute_vector
from .kernels import STRIDED_NX, BlockDims, host_row_sums, spmv_csr_ref
from .reorder import band_k
from .tuning import (
    VOLTA,
    DeviceProfile,
    compute_stats,
    cpu_candidate_srs,
    cpu_fallback_srs,
    gpu_candidate_grid,
    grid_search,
    tune_gpu,
)

__all__ = [
    "SCHEMA_VERSION",
    "DEFAULT_WARMUPS",
    "DEFAULT_REPS",
    "DEFAULT_TOLERANCE",
    "TARGETS",
    "BenchRecord",
    "CudaEventClock",
    "default_threads",
    "max_rel_error",
    "scaled_error",
    "time_kernel",
    "empirical_search",
    "run_benchmark",
    "spmv_bytes",
]

SCHEMA_VERSION = 1
DEFAULT_WARMUPS = 5
DEFAULT_REPS = 20
DEFAULT_TOLERANCE = 1e-10

TARGETS = ("ref", "cpu2", "cpu3", "gpu3-emu", "gpu35-emu", "cuda3", "cuda35")


def default_threads() -> int:
    """OMP_NUM_THREADS when set to a positive integer, else the CPU count
    (bench.py:61-66); recorded as the host core count of CPU baselines."""
    env = os.environ.get("OMP_NUM_THREADS", "").strip()
    if env.isdigit() and int(env) > 0:
        return int(env)
    return os.cpu_count() or 1


def max_rel_error(y, ref) -> float:
    """max |y - ref| / max(|ref|, 1e-300) (bench.py:69-82)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.shape != ref.shape:
        raise ValueError("shape mismatch between result and reference")
    if y.size == 0:
        return 0.0
    return float((np.abs(y - ref) / np.maximum(np.abs(ref), 1e-300)).max())


def scaled_error(y, ref, abs_row_dot) -> float:
    """max_i |y_i - ref_i| / (|A||x|)_i -- the cancellation-free parity
    metric of SURVEY.md §8(c)(3); rows with (|A||x|)_i = 0 must match
    exactly."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.asarray(abs_row_dot, dtype=np.float64)
    diff = np.abs(y - ref)
    if y.size == 0:
        return 0.0
    zero = d == 0
    if np.any(diff[zero] != 0):
        return float("inf")
    return float((diff[~zero] / d[~zero]).max()) if np.any(~zero) else 0.0


NOMINAL_HBM_GBS = 8000.0


def measured_hbm_gbs():
    """The measured HBM copy bandwidth of this machine, GB/s: $CSRK_HBM_GBS,
    else MEASURED_PEAKS.json next to the package (the repo root), else None."""
    env = os.environ.get("CSRK_HBM_GBS", "").strip()
    if env:
        try:
            return float(env)
        except ValueError:
            return None
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError, TypeError):
        return None


def spmv_bytes(n_rows: int, n_cols: int, nnz: int, value_bytes: int = 8) -> int:
    """Algorithmic HBM bytes of one SpMV: vals + col_idx
    + row_ptr + x + y, each touched once."""
    return nnz * (value_bytes + 4) + 4 * (n_rows + 1) + (n_cols + n_rows) * value_bytes


def time_kernel(step, warmups: int = DEFAULT_WARMUPS, reps: int = DEFAULT_REPS,
                clock=time.perf_counter):
    """``warmups + reps`` calls of ``step``, each bracketed by ``clock()``;
    returns (durations of the last ``reps``, result of the final call)
    (bench.py:85-105)."""
    if warmups < 0:
        raise ValueError("warmups must be non-negative")
    if reps < 1:
        raise ValueError("reps must be at least 1")
    durations = []
    result = None
    for i in range(warmups + reps):
        t0 = clock()
        result = step()
        t1 = clock()
        if i >= warmups:
            durations.append(t1 - t0)
    return durations, result


class CudaEventClock:
    """A ``clock`` for time_kernel reading device time: each call records a
    CUDA event on the legacy default stream, waits for it, and returns
    seconds since the first call."""

    def __init__(self):
        import torch

        self._torch = torch
        self._origin = None

    def __call__(self) -> float:
        torch = self._torch
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.default_stream())
        ev.synchronize()
        if self._origin is None:
            self._origin = ev
            return 0.0
        return self._origin.elapsed_time(ev) / 1e3


@dataclass(frozen=True)
class BenchRecord:
    """One measurement, reproducible from its fields (bench.py:108-127)."""

    schema_version: int
    matrix_id: str
    kernel: str
    tuning: dict
    warmups: int
    reps: int
    mean_seconds: float
    gflops: float
    max_rel_error: float
    tolerance: float
    passed: bool
    reorder_seconds: float
    pack_seconds: float
    # B200 extensions: algorithmic HBM bytes per
    # multiply (spmv_bytes) over the mean time, its fraction of the nominal
    # 8 TB/s and of the measured copy bandwidth (when known), the scaled
    # error max |y - ref| / (|A||x|) of SURVEY.md §8(c)(3), and what the
    # result was verified against
    gbs: float = 0.0
    frac_of_nominal: float = 0.0
    frac_of_measured: float | None = None
    scaled_error: float = 0.0
    verified_against: str = "spmv_csr_ref (host, sequential row sums)"

    def to_dict(self) -> dict:
        return asdict(self)


class _DeviceStep:
    """One device-resident multiply of a packed matrix: x uploaded once,
    y kept in HBM; calling it launches the kernel and waits."""

    def __init__(self, target: str, m, xp: np.ndarray, dims: BlockDims | None):
        self.target = target
        self.m = m
        self.dev = m.device()
        n_out = self.dev.n_rows
        self.n_out = n_out
        self.x = nat.DeviceBuffer.from_array(np.ascontiguousarray(xp, dtype=np.float64))
        self.y = nat.DeviceBuffer(max(8, n_out * 8))
        self.dims = dims
        if target == "cuda35" and (dims is None or dims.x not in STRIDED_NX):
            # strided orders outside the instantiated lane counts use Listing 4
            self.target = "gpu35-emu"

    def __call__(self):
        t, d = self.target, self.dims
        if self.n_out:
            if t in ("ref", "cpu2", "cpu3", "cuda3"):
                self.dev.spmv_ptr(self.x.address, self.y.address, 0)
            elif t == "cuda35":
                self.dev.spmv_ptr(self.x.address, self.y.address, 0,
                                  variant=nat.CSRK_STRIDED, nx=d.x)
            elif t == "gpu3-emu":
                nat.call("csrk_spmv_listing3", self.dev.ptr, d.x, d.y, self.x.ptr,
                         self.y.ptr, None, None)
            elif t == "gpu35-emu":
                nat.call("csrk_spmv_listing4", self.dev.ptr, d.x, d.y, d.z, self.x.ptr,
                         self.y.ptr, None, None)
            else:
                raise ValueError(f"unknown kernel target {t!r}")
        nat.call("csrk_stream_sync", None)
        return self

    def result(self) -> np.ndarray:
        return self.y.to_array(np.float64, self.n_out)


def _tuning_dict(k, ssrs, srs, dims, variant: str) -> dict:
    return {"k": k, "ssrs": ssrs, "srs": srs,
            "block_dims": None if dims is None else [dims.x, dims.y, dims.z],
            "kernel_variant": variant}


def _k_for_target(target: str):
    return {"ref": None, "cpu2": 2}.get(target, 3)


def _validate_dims(target: str, dims):
    if target in ("gpu3-emu",) and dims is not None and dims.z != 1:
        raise ValueError("the 2D mapping does not use the z dimension")


def _make_step(target: str, packed, xp, threads: int, dims):
    if target not in TARGETS or target == "ref":
        raise ValueError(f"unknown kernel target {target!r}")
    _validate_dims(target, dims)
    return _DeviceStep(target, packed, xp, dims)


def _resolve_sizes(a: CsrMatrix, target, k, profile, tune_mode, x, threads, grid_reps):
    stats = compute_stats(a)
    if k == 2:
        if tune_mode == "grid":
            return None, empirical_search(a, target, 2, x, threads, grid_reps).best, None
        return None, cpu_fallback_srs(), None
    params = tune_gpu(stats, profile)
    ssrs, srs, dims = params.ssrs, params.srs, params.block_dims
    if tune_mode == "grid":
        ssrs, srs = empirical_search(a, target, 3, x, threads, grid_reps, dims).best
    return ssrs, srs, dims


def empirical_search(a: CsrMatrix, target: str, k: int, x, threads: int, reps: int = 3,
                     dims: BlockDims | None = None, candidates=None):
    """Per-matrix grid search (bench.py:181-209): each candidate is reordered
    and packed once, outside timing; a runner call times exactly one
    device multiply with CUDA events.  ``candidates`` defaults to the
    reference's grids (CPU ladder for k = 2, the 64 GPU pairs for k = 3)."""
    cache = {}
    clock = CudaEventClock()

    def prepare(cand):
        if cand not in cache:
            targets = [cand] if k == 2 else [cand[1], cand[0]]
            res = band_k(a, k, targets)
            packed = pack_csrk(a, res.perm, res.level_group_sizes, download=False)
            cache[cand] = _make_step(target, packed, permute_vector(res.perm, x),
                                     threads, dims)
        return cache[cand]

    def runner(_a, cand):
        step = prepare(cand)
        t0 = clock()
        step()
        return clock() - t0

    if candidates is None:
        candidates = cpu_candidate_srs() if k == 2 else gpu_candidate_grid()
    return grid_search(a, candidates, runner, reps=reps)


def run_benchmark(a: CsrMatrix, matrix_id: str, target: str, *, ssrs=None, srs=None,
                  block_dims: BlockDims | None = None, profile: DeviceProfile = VOLTA,
                  tune_mode: str = "auto", warmups: int = DEFAULT_WARMUPS,
                  reps: int = DEFAULT_REPS, threads: int | None = None,
                  tolerance: float = DEFAULT_TOLERANCE, seed: int = 0,
                  clock=time.perf_counter, step_wrapper=None) -> BenchRecord:
    """Stats -> tuning -> Band-k -> pack -> timed multiplies -> verification
    against the plain-CSR kernel, as reference bench.py:212-326."""
    if target not in TARGETS:
        raise ValueError(f"unknown kernel target {target!r}")
    if tune_mode not in ("auto", "grid"):
        raise ValueError(f"unknown tuning mode {tune_mode!r}")
    threads = threads or default_threads()
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, a.n_cols)
    ref_y = spmv_csr_ref(a, x)
    k = _k_for_target(target)
    reorder_s = pack_s = 0.0
    perm = None
    if target == "ref":
        step = _DeviceStep("ref", a, x, None)
        tuning = _tuning_dict(None, None, None, None, "ref")
    else:
        t_ssrs, t_srs, t_dims = _resolve_sizes(a, target, k, profile, tune_mode, x,
                                               threads, 3)
        t_ssrs = t_ssrs if ssrs is None else ssrs
        t_srs = t_srs if srs is None else srs
        t_dims = t_dims if block_dims is None else block_dims
        t0 = time.perf_counter()
        res = band_k(a, k, [t_srs] if k == 2 else [t_srs, t_ssrs])
        reorder_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        packed = pack_csrk(a, res.perm, res.level_group_sizes, download=False)
        pack_s = time.perf_counter() - t0
        perm = res.perm
        step = _make_step(target, packed, permute_vector(perm, x), threads, t_dims)
        shows_dims = target.startswith("gpu") or target.startswith("cuda")
        tuning = _tuning_dict(k, t_ssrs, t_srs, t_dims if shows_dims else None, target)
    if step_wrapper is not None:
        step = step_wrapper(step)
    durations, last = time_kernel(step, warmups, reps, clock)
    mean = sum(durations) / len(durations)
    y = last.result() if isinstance(last, _DeviceStep) else np.asarray(last)
    if perm is not None:
        y = unpermute_vector(perm, y)
    err = max_rel_error(y, ref_y)
    scale = host_row_sums(a.row_ptr, a.col_idx, np.abs(a.vals), np.abs(x))
    gbs = spmv_bytes(a.n_rows, a.n_cols, a.nnz, 8) / mean / 1e9 if mean > 0 else float("inf")
    peak = measured_hbm_gbs()
    return BenchRecord(
        schema_version=SCHEMA_VERSION, matrix_id=matrix_id, kernel=target,
        tuning=tuning, warmups=warmups, reps=reps, mean_seconds=mean,
        gflops=2.0 * a.nnz / mean / 1e9 if mean > 0 else float("inf"),
        max_rel_error=err, tolerance=tolerance, passed=bool(err <= tolerance),
        reorder_seconds=reorder_s, pack_seconds=pack_s,
        gbs=gbs, frac_of_nominal=gbs / NOMINAL_HBM_GBS,
        frac_of_measured=(gbs / peak) if peak else None,
        scaled_error=scaled_error(y, ref_y, scale))
