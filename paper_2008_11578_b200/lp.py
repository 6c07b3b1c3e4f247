"""Batched closest-point LP on the GPU: the device twin of the reference's
lp.solve_batch / _kernels.solve_range (pkg/src/orcasim/lp.py:263-291,
pkg/src/orcasim/_kernels.py:306-336).

    solve_range(coff, cpts, cnrm, tgt, caps, seeds) -> (out_v, status, failed_at)
        flat CSR arrays exactly as _kernels.solve_range takes them
    solve_batch(problems)  -> list[LpResult]
        object-level API with the reference's validation messages
    LpBatch(...)            resident batch for repeated solves (benchmarks)

No CPU fallback: all three launch liborca_b200.so kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np

from ._lib import ORCA_CERT32, ORCA_F64, ORCA_MIXED, check, load, precision_code, ptr

__all__ = ["HalfPlaneConstraint", "LpProblem", "LpResult", "LpStatus", "LpBatch",
           "shuffle_order", "solve_range", "solve_batch", "solve_closest_point",
           "solve_least_penetration", "DEFAULT_WORK_UNIT_STEPS"]

DEFAULT_WORK_UNIT_STEPS = 64        # lp.py:28 (accepted and ignored: results do not depend on it)

MASK64 = (1 << 64) - 1


class LpStatus(Enum):
    FEASIBLE = "feasible"
    FALLBACK_USED = "fallback_used"


_STATUS_OF_CODE = (LpStatus.FEASIBLE, LpStatus.FALLBACK_USED)     # _kernels.py: FEASIBLE = 0, FALLBACK_USED = 1


@dataclass
class HalfPlaneConstraint:
    """One half-plane of permitted velocities: `point` on the boundary line, `normal` the unit
    normal into the permitted side -- v is allowed iff dot(v - point, normal) >= 0 (lp.py:47-64)."""

    point: np.ndarray
    normal: np.ndarray

    def __post_init__(self):
        self.point = np.asarray(self.point, dtype=float)
        self.normal = np.asarray(self.normal, dtype=float)

    def satisfies(self, velocity, slack: float = 0.0) -> bool:
        v = np.asarray(velocity, dtype=float)
        return float(np.dot(v - self.point, self.normal)) >= -slack


@dataclass
class LpProblem:
    """Closest-point problem: constraints, desired velocity, speed cap and the seed that fixes
    the constraint insertion order (lp.py:67-80)."""

    constraints: list
    target: np.ndarray
    speed_cap: float
    shuffle_seed: int = 0

    def __post_init__(self):
        self.target = np.asarray(self.target, dtype=float)
        self.speed_cap = float(self.speed_cap)
        self.shuffle_seed = int(self.shuffle_seed) & MASK64


@dataclass
class LpResult:
    velocity: np.ndarray
    status: LpStatus
    failed_at: int | None = None

    @property
    def feasible(self) -> bool:
        return self.status is LpStatus.FEASIBLE


def _mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return (z ^ (z >> 31)) & MASK64


def shuffle_order(count: int, seed: int) -> list[int]:
    """Constraint insertion order for a shuffle seed (lp.py:101-112); host-side
    twin of the in-kernel shuffle, kept in lockstep by tests/test_gpu_kat.py."""
    perm = list(range(count))
    state = seed & MASK64
    for i in range(count - 1, 0, -1):
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        j = _mix64(state) % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def _lp_precision(precision) -> int:
    """The LP entry points take arbitrary float64 problems: 'f64' (default, bit-identical
    to the reference) or 'f32'. 'mixed' has no separate meaning here and maps to 'f64'."""
    code = precision_code(precision)
    return ORCA_F64 if code in (ORCA_MIXED, ORCA_CERT32) else code


def _prep(coff, cpts, cnrm, tgt, caps, seeds):
    coff = np.ascontiguousarray(coff, dtype=np.int64)
    n = coff.shape[0] - 1
    cpts = np.ascontiguousarray(cpts, dtype=np.float64).reshape(-1, 2)
    cnrm = np.ascontiguousarray(cnrm, dtype=np.float64).reshape(-1, 2)
    tgt = np.ascontiguousarray(tgt, dtype=np.float64).reshape(-1, 2)
    caps = np.ascontiguousarray(caps, dtype=np.float64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    if n < 0 or tgt.shape[0] != n or caps.shape[0] != n or seeds.shape[0] != n:
        raise ValueError("inconsistent batch arrays")
    if cpts.shape[0] != int(coff[-1]) or cnrm.shape[0] != int(coff[-1]):
        raise ValueError("constraint arrays do not match coff[-1]")
    return n, coff, cpts, cnrm, tgt, caps, seeds


def solve_range(coff, cpts, cnrm, tgt, caps, seeds, precision="f64", device: int = 0):
    """_kernels.solve_range over the whole batch on the GPU.
    Returns (out_v f64[n,2], status i64[n], failed_at i64[n])."""
    n, coff, cpts, cnrm, tgt, caps, seeds = _prep(coff, cpts, cnrm, tgt, caps, seeds)
    from .engine import _host_empty          # pinned (pooled) result buffers when torch is there
    out_v = _host_empty((n, 2))
    status = _host_empty(n, np.int64)
    failed = _host_empty(n, np.int64)
    check(load().orca_lp_solve_batch(device, _lp_precision(precision), n, ptr(coff), ptr(cpts),
                                     ptr(cnrm), ptr(tgt), ptr(caps), ptr(seeds), ptr(out_v),
                                     ptr(status), ptr(failed)))
    return out_v, status, failed


class LpBatch:
    """A batch resident on the device: build once, solve repeatedly."""

    def __init__(self, coff, cpts, cnrm, tgt, caps, seeds, precision="f64", device: int = 0,
                 stream=None):
        self._L = load()
        self.n, coff, cpts, cnrm, tgt, caps, seeds = _prep(coff, cpts, cnrm, tgt, caps, seeds)
        self.m = int(coff[-1])
        self._h = C.c_void_p()
        check(self._L.orca_lp_batch_create(C.byref(self._h), device, _lp_precision(precision),
                                           self.n, ptr(coff), ptr(cpts), ptr(cnrm), ptr(tgt),
                                           ptr(caps), ptr(seeds)))
        if stream is not None:
            handle = getattr(stream, "cuda_stream", stream)
            check(self._L.orca_lp_batch_set_stream(
                self._h, C.c_void_p(int(handle) if handle else None)))

    def solve(self):
        check(self._L.orca_lp_batch_solve(self._h))

    def results(self):
        out_v = np.empty((self.n, 2))
        status = np.empty(self.n, dtype=np.int64)
        failed = np.empty(self.n, dtype=np.int64)
        check(self._L.orca_lp_batch_download(self._h, ptr(out_v), ptr(status), ptr(failed)))
        return out_v, status, failed

    def close(self):
        if getattr(self, "_h", None) is not None and self._h:
            self._L.orca_lp_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- object-level API (validation text follows lp.py:115-140) -----------------

def _validate_constraints(constraints, label=""):
    pts = np.empty((len(constraints), 2), dtype=np.float64)
    nrm = np.empty((len(constraints), 2), dtype=np.float64)
    for idx, c in enumerate(constraints):
        p = np.asarray(c.point, dtype=float).reshape(2)
        n = np.asarray(c.normal, dtype=float).reshape(2)
        if not np.all(np.isfinite(p)) or not np.all(np.isfinite(n)):
            raise ValueError(f"{label}constraint {idx}: non-finite point or normal")
        nn = float(n[0] * n[0] + n[1] * n[1])
        if abs(nn - 1.0) > 2.1e-9:
            raise ValueError(
                f"{label}constraint {idx}: normal must be unit length, got |n|={np.sqrt(nn)!r}")
        pts[idx] = p
        nrm[idx] = n
    return pts, nrm


def _validate_problem(problem, label=""):
    target = np.asarray(problem.target, dtype=float).reshape(2)
    if not np.all(np.isfinite(target)):
        raise ValueError(f"{label}target is non-finite")
    cap = float(problem.speed_cap)
    if not np.isfinite(cap) or cap <= 0.0:
        raise ValueError(f"{label}speed_cap must be positive and finite, got {cap!r}")
    pts, nrm = _validate_constraints(problem.constraints, label)
    return pts, nrm, target, cap


def solve_batch(problems, worker_count: int = 1, work_unit_steps: int = 64, *,
                precision="f64", device: int = 0):
    """lp.solve_batch (lp.py:263-291): validate, pack to CSR, solve on the GPU. The output is
    index-aligned with the input; worker_count / work_unit_steps are validated like the
    reference's and otherwise ignored (its results are independent of both)."""
    if worker_count < 1:
        raise ValueError(f"worker_count must be >= 1, got {worker_count}")
    del work_unit_steps
    n = len(problems)
    if n == 0:
        return []
    coff = np.zeros(n + 1, dtype=np.int64)
    parts = []
    for i, p in enumerate(problems):
        parts.append(_validate_problem(p, label=f"problem {i}: "))
        coff[i + 1] = coff[i] + len(p.constraints)
    m = int(coff[n])
    cpts, cnrm = np.empty((m, 2)), np.empty((m, 2))
    tgt, caps = np.empty((n, 2)), np.empty(n)
    seeds = np.empty(n, dtype=np.uint64)
    for i, (pts, nrm, target, cap) in enumerate(parts):
        cpts[coff[i]:coff[i + 1]] = pts
        cnrm[coff[i]:coff[i + 1]] = nrm
        tgt[i], caps[i] = target, cap
        seeds[i] = np.uint64(problems[i].shuffle_seed & MASK64)
    out_v, status, failed = solve_range(coff, cpts, cnrm, tgt, caps, seeds, precision, device)
    return [LpResult(out_v[i].copy(), _STATUS_OF_CODE[int(status[i])],
                     None if status[i] == 0 else int(failed[i])) for i in range(n)]


def solve_closest_point(problem, *, precision="f64", device: int = 0) -> LpResult:
    """lp.solve_closest_point (lp.py:152-165) for one problem."""
    return solve_batch([problem], precision=precision, device=device)[0]


def solve_least_penetration(constraints, speed_cap, start_index=0, warm_start=(0.0, 0.0), *,
                            precision="f64", device: int = 0) -> np.ndarray:
    """Velocity minimising the worst signed constraint violation (clamped at zero) within the
    speed disc; ties broken by proximity to warm_start (lp.py:168-190 -> _kernels.py:254-283,
    constraints in the given order). warm_start is assumed to satisfy constraints[:start_index]."""
    cap = float(speed_cap)
    if not np.isfinite(cap) or cap <= 0.0:
        raise ValueError(f"speed_cap must be positive and finite, got {cap!r}")
    warm = np.asarray(warm_start, dtype=float).reshape(2)
    if not np.all(np.isfinite(warm)):
        raise ValueError("warm_start is non-finite")
    pts, nrm = _validate_constraints(constraints)
    k = len(constraints)
    if not 0 <= start_index <= k:
        raise ValueError(f"start_index {start_index} out of range for {k} constraints")
    out = np.empty(2)
    check(load().orca_least_penetration(device, _lp_precision(precision), k, ptr(pts), ptr(nrm), cap,
                                        int(start_index), float(warm[0]), float(warm[1]), ptr(out)))
    return out
