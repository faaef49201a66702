"""Thin ctypes binding of include/asyflexa.h (argument marshalling only).

Every function below has the name of the C entry point it wraps; all
arithmetic happens in ``lib/libasyflexa.so`` (sm_100a kernels).  There is no
CPU fallback: importing this module fails loudly when the library is absent.

``Solver`` is a convenience wrapper that builds an ``asy_problem`` from a
``paper_1701_04900_b200.inputs.Problem`` (numpy host arrays, or device arrays
uploaded with torch -- torch is used only for device memory).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libasyflexa.so")
if os.environ.get("ASY_LIB_VARIANT"):  # developer builds with other compile-time geometry (tools/)
    LIB_PATH = os.path.join(_HERE, "lib", "libasyflexa_%s.so" % os.environ["ASY_LIB_VARIANT"])
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1701_04900_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ---- constants (include/asyflexa.h) ----------------------------------------
ASY_OK, ASY_ERR_INVALID, ASY_ERR_CUDA, ASY_ERR_NOMEM, ASY_ERR_STATE, ASY_ERR_UNSUPPORTED = range(6)
ASY_MEM_HOST, ASY_MEM_DEVICE = 0, 1
ASY_DENSE_COLMAJOR, ASY_CSC = 0, 1
ASY_LOSS_LS, ASY_LOSS_LOGISTIC = 0, 1
ASY_REG_L1, ASY_REG_EXP, ASY_REG_LOG = 0, 1, 2
ASY_MODE_ASYNC, ASY_MODE_SYNC_JACOBI = 0, 1
ASY_SCHED_CYCLIC, ASY_SCHED_RANDOM = 0, 1
ASY_KERNEL_JACOBI, ASY_KERNEL_DENSE_PANEL, ASY_KERNEL_DENSE_SLAB, ASY_KERNEL_SPARSE = 0, 1, 2, 3
ASY_KERNEL_DENSE_SLAB_TMEM = 4
KERNEL_NAMES = {0: "jacobi (asy::dense_gemvT/gemvN)", 1: "asy::dense_async_kernel",
                2: "asy::dense_slab_kernel", 3: "asy::sparse_async_kernel",
                4: "asy::dense_slabt_kernel"}

_vp, _dp = C.c_void_p, C.POINTER(C.c_double)


class asy_problem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mem", C.c_int32), ("m", C.c_int64), ("n", C.c_int64),
                ("A", _vp), ("lda", C.c_int64),
                ("colptr", _vp), ("rowidx", _vp), ("vals", _vp), ("nnz", C.c_int64),
                ("loss", C.c_int32), ("reg", C.c_int32),
                ("loss_scale", C.c_double), ("c_nonconvex", C.c_double), ("lambda_", C.c_double),
                ("theta", C.c_double), ("b", _vp), ("tau", _vp), ("lo", _vp), ("hi", _vp),
                ("lo_all", C.c_double), ("hi_all", C.c_double), ("block_size", C.c_int64)]


class asy_tuning(C.Structure):
    _fields_ = [("dense_kernel", C.c_int32), ("panel_park", C.c_int32), ("slab_hold", C.c_int32),
                ("slab_chunk_rows", C.c_int32), ("slab_ring", C.c_int32), ("measure_delay", C.c_int32),
                ("reserved", C.c_int32 * 2)]


class asy_solve_params(C.Structure):
    _fields_ = [("mode", C.c_int32), ("schedule", C.c_int32), ("seed", C.c_uint64),
                ("gamma", C.c_double), ("sweeps", C.c_int64), ("max_delay", C.c_int64),
                ("reset", C.c_int32), ("x_mem", C.c_int32), ("x0", _vp), ("x_out", _vp),
                ("f_hist", _vp), ("workers", C.c_int32), ("panel_rows", C.c_int32),
                ("stages", C.c_int32), ("tuning", C.POINTER(asy_tuning))]


class asy_solve_stats(C.Structure):
    _fields_ = [("block_updates", C.c_int64), ("launches", C.c_int64), ("kernel_ms", C.c_double),
                ("total_ms", C.c_double), ("objective", C.c_double), ("epochs", C.c_int64),
                ("kernel", C.c_int32), ("delay", C.c_int32), ("delay_observed", C.c_int32)]


class asy_stationarity_out(C.Structure):
    _fields_ = [("objective", C.c_double), ("smooth", C.c_double), ("mf_norm2", C.c_double),
                ("mf_norminf", C.c_double), ("merit_inf", C.c_double)]


_H = C.c_void_p
_lib.asy_create.argtypes = [C.c_int, _vp, C.POINTER(_H)]
_lib.asy_destroy.argtypes = [_H]
_lib.asy_set_problem.argtypes = [_H, C.POINTER(asy_problem)]
_lib.asy_solve.argtypes = [_H, C.POINTER(asy_solve_params), C.POINTER(asy_solve_stats)]
_lib.asy_stationarity.argtypes = [_H, _vp, C.c_int32, C.POINTER(asy_stationarity_out)]
_lib.asy_get_x.argtypes = [_H, _vp, C.c_int32]
_lib.asy_objective.argtypes = [_H, _dp]
if hasattr(_lib, "asy_get_residual") or not os.environ.get("ASY_LIB_VARIANT"):  # (older developer builds lack it)
    _lib.asy_get_residual.argtypes = [_H, _vp, C.c_int32]
_lib.asy_last_error.argtypes = [_H]
_lib.asy_last_error.restype = C.c_char_p
_lib.asy_version.restype = C.c_char_p
_lib.asy_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
_lib.asy_philox4x32_10.restype = None
_lib.asy_schedule_block.argtypes = [C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]
_lib.asy_schedule_prev.argtypes = [C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]
_lib.asy_schedule_device.argtypes = [_H, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _vp]
for _f in ("asy_create", "asy_destroy", "asy_set_problem", "asy_solve", "asy_stationarity",
           "asy_get_x", "asy_objective", "asy_schedule_block", "asy_schedule_prev", "asy_schedule_device"):
    getattr(_lib, _f).restype = C.c_int


class AsyError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[asyflexa error {code}] {msg}")
        self.code = code


def _check(code, h):
    if code != ASY_OK:
        raise AsyError(code, (_lib.asy_last_error(h) or b"").decode())


# ---- the C entry points, same names --------------------------------------
def asy_version() -> str:
    return _lib.asy_version().decode()


def asy_create(device: int = 0, stream: int = 0):
    h = _H()
    code = _lib.asy_create(device, _vp(stream or None), C.byref(h))
    _check(code, None)
    return h


def asy_destroy(h) -> None:
    _check(_lib.asy_destroy(h), h)


def asy_set_problem(h, p: asy_problem) -> None:
    _check(_lib.asy_set_problem(h, C.byref(p)), h)


def asy_solve(h, sp: asy_solve_params) -> asy_solve_stats:
    st = asy_solve_stats()
    _check(_lib.asy_solve(h, C.byref(sp), C.byref(st)), h)
    return st


def asy_stationarity(h, x_ptr=None, x_mem=ASY_MEM_DEVICE) -> asy_stationarity_out:
    out = asy_stationarity_out()
    _check(_lib.asy_stationarity(h, _vp(x_ptr), x_mem, C.byref(out)), h)
    return out


def asy_get_x(h, x_ptr, x_mem) -> None:
    _check(_lib.asy_get_x(h, _vp(x_ptr), x_mem), h)


def asy_get_residual(h, r_ptr, r_mem) -> None:
    _check(_lib.asy_get_residual(h, r_ptr, r_mem), h)


def asy_objective(h) -> float:
    F = C.c_double()
    _check(_lib.asy_objective(h, C.byref(F)), h)
    return F.value


def asy_last_error(h=None) -> str:
    return (_lib.asy_last_error(h) or b"").decode()


def asy_philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    _lib.asy_philox4x32_10(c, k, o)
    return list(o)


def asy_schedule_block(schedule: int, seed: int, nblocks: int, k: int) -> int:
    out = C.c_int64()
    code = _lib.asy_schedule_block(schedule, seed, nblocks, k, C.byref(out))
    if code != ASY_OK:
        raise AsyError(code, "asy_schedule_block: invalid arguments")
    return out.value


def asy_schedule_prev(schedule: int, seed: int, nblocks: int, k: int) -> int:
    out = C.c_int64()
    code = _lib.asy_schedule_prev(schedule, seed, nblocks, k, C.byref(out))
    if code != ASY_OK:
        raise AsyError(code, "asy_schedule_prev: invalid arguments")
    return out.value


def asy_schedule_device(h, schedule: int, seed: int, nblocks: int, k0: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.int64)
    _check(_lib.asy_schedule_device(h, schedule, seed, nblocks, k0, count, out.ctypes.data), h)
    return out


# ---- convenience wrapper ----------------------------------------------------
def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class Solver:
    """One handle + one installed problem.

    mem="device": arrays are uploaded once with torch (borrowed by the library);
    mem="host":   numpy arrays are handed to the library, which copies them."""

    def __init__(self, P, device: int = 0, mem: str = "device", stream: int = 0, pinned: bool = False):
        self.P = P
        self.h = asy_create(device, stream)
        self.device = device
        self._keep = []
        self.mem = ASY_MEM_DEVICE if mem == "device" else ASY_MEM_HOST
        self.set_problem(P, pinned=pinned)

    # arrays as the library will see them
    def _arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        if self.mem == ASY_MEM_HOST:
            if getattr(self, "_pinned", False) and a.nbytes > 0:
                # page-lock the array in place (no second host copy of a 32 GB matrix)
                import torch
                rt = torch.cuda.cudart()
                if int(rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)) == 0:
                    self._registered.append(a.ctypes.data)
            self._keep.append(a)
            return a.ctypes.data
        import torch
        t = torch.from_numpy(a).to(f"cuda:{self.device}")
        self._keep.append(t)
        return t.data_ptr()

    def problem_struct(self, P) -> asy_problem:
        p = asy_problem()
        p.mem = self.mem
        p.m, p.n = P.m, P.n
        if P.kind == "dense":
            p.kind = ASY_DENSE_COLMAJOR
            At = np.ascontiguousarray(P.A.T)  # rows of A^T = columns of A
            p.A = self._arr(At, np.float64)
            p.lda = P.m
        else:
            p.kind = ASY_CSC
            p.colptr = self._arr(P.colptr, np.int64)
            p.rowidx = self._arr(P.rowidx, np.int32)
            p.vals = self._arr(P.vals, np.float64)
            p.nnz = int(P.vals.size)
        p.loss = ASY_LOSS_LS if P.loss == "ls" else ASY_LOSS_LOGISTIC
        p.reg = {"l1": ASY_REG_L1, "exp": ASY_REG_EXP, "log": ASY_REG_LOG}[P.reg]
        p.loss_scale = P.scale
        p.c_nonconvex = P.c
        p.lambda_ = P.lam
        p.theta = P.theta
        p.b = self._arr(P.b, np.float64)
        p.tau = self._arr(P.tau, np.float64)
        if np.ndim(P.lo) == 0:
            p.lo_all, p.hi_all = float(P.lo), float(P.hi)
        else:
            p.lo = self._arr(P.lo, np.float64)
            p.hi = self._arr(P.hi, np.float64)
        p.block_size = P.block
        return p

    def set_problem(self, P, pinned: bool = False):
        self._unregister()
        self._keep = []
        self.P = P
        self._pinned = pinned
        self.pstruct = self.problem_struct(P)  # host / device arrays kept alive by _keep
        asy_set_problem(self.h, self.pstruct)  # device A / CSC stay borrowed via _keep

    def _unregister(self):
        regs = getattr(self, "_registered", [])
        if regs:
            import torch
            rt = torch.cuda.cudart()
            for ptr in regs:
                rt.cudaHostUnregister(ptr)
        self._registered = []

    def solve(self, *, mode=ASY_MODE_ASYNC, sweeps=1, gamma=None, schedule=ASY_SCHED_CYCLIC, seed=0,
              max_delay=-1, reset=False, x0=None, f_hist=False, workers=0, panel_rows=0, stages=0,
              tuning=None):
        """tuning: None or a dict of asy_tuning fields (kernel choice / geometry overrides)."""
        sp = asy_solve_params()
        sp.mode, sp.schedule, sp.seed = mode, schedule, seed
        sp.gamma = self.P.gamma if gamma is None else gamma
        sp.sweeps, sp.max_delay, sp.reset = sweeps, max_delay, int(reset)
        sp.x_mem = ASY_MEM_HOST
        x0a = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            sp.x0 = x0a.ctypes.data
        hist = np.zeros(sweeps) if f_hist else None
        if f_hist:
            sp.f_hist = hist.ctypes.data
        sp.workers, sp.panel_rows, sp.stages = workers, panel_rows, stages
        tu = None
        if tuning:
            tu = asy_tuning(**tuning)
            sp.tuning = C.pointer(tu)
        st = asy_solve(self.h, sp)
        return (st, hist) if f_hist else st

    def x(self) -> np.ndarray:
        out = np.zeros(self.P.n)
        asy_get_x(self.h, out.ctypes.data, ASY_MEM_HOST)
        return out

    def objective(self) -> float:
        return asy_objective(self.h)

    def residual(self) -> np.ndarray:
        out = np.zeros(self.P.m)
        asy_get_residual(self.h, out.ctypes.data, ASY_MEM_HOST)
        return out

    def stationarity(self, x=None) -> asy_stationarity_out:
        if x is None:
            return asy_stationarity(self.h, None, ASY_MEM_DEVICE)
        xa = np.ascontiguousarray(x, np.float64)
        return asy_stationarity(self.h, xa.ctypes.data, ASY_MEM_HOST)

    def close(self):
        if self.h is not None:
            asy_destroy(self.h)
            self.h = None
        self._unregister()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
