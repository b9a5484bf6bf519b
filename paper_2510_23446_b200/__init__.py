"""paper_2510_23446_b200 — B200-native tree-cotree IETI-DP time stepper (arXiv 2510.23446).

Thin ctypes binding over the C ABI declared in include/tcg_ietidp.h (argument
marshalling only: topology/tree/partition run in the library's C++ host code, every
arithmetic step of the method runs in its sm_100a CUDA kernels). There is no CPU
fallback: if libtcg_ietidp.so is missing or cannot be loaded, importing `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.environ.get("TCG_LIBPATH") or os.path.join(HERE, "libtcg_ietidp.so")  # (env: A/B experiments only)

TCG_OK, TCG_EINVAL, TCG_ESTATE, TCG_ENOTSPD, TCG_ENOCONV, TCG_ECUDA, TCG_ENCCL, TCG_ENOMEM = 0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "TCG_OK", -1: "TCG_EINVAL", -2: "TCG_ESTATE", -3: "TCG_ENOTSPD", -4: "TCG_ENOCONV",
                -5: "TCG_ECUDA", -6: "TCG_ENCCL", -7: "TCG_ENOMEM"}
PLAN_EDGE_CLASS, PLAN_EDGE_REGION, PLAN_TREE, PLAN_PART, PLAN_PATCH_COUNTS, PLAN_LAMBDA, PLAN_PRIMAL, PLAN_RANK_OF_PATCH = range(8)

EXPORTS = ["tcg_create", "tcg_set_patches", "tcg_set_materials", "tcg_set_source", "tcg_set_time", "tcg_set_solver", "tcg_set_warm_start",
           "tcg_plan", "tcg_get_plan", "tcg_setup", "tcg_refactor", "tcg_step", "tcg_get_coefficients", "tcg_get_history",
           "tcg_get_info", "tcg_fapply", "tcg_bench_fapply", "tcg_set_profile", "tcg_set_virtual_ranks", "tcg_nccl_unique_id", "tcg_last_error",
           "tcg_destroy", "tcg_set_error_tracking", "tcg_get_errors", "tcg_set_nonlinear", "tcg_get_newton"]


class TcgInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_patches", "n_local", "n_edges", "n_verts", "m", "n_c", "n_gauge", "n_dirichlet", "n_primal_local_total",
        "nr_min", "nr_max", "nb_min", "nb_max", "np_min", "np_max", "steps_done", "total_iters", "device_bytes",
        "kernel_launches")] + [(n, C.c_double) for n in (
        "bytes_fapply", "bytes_precond", "bytes_step_fixed", "flops_factor", "ms_plan", "ms_assembly", "ms_factor",
        "ms_coarse", "ms_steps", "ms_pcg_last_step", "prof_ms")] + [("prof_launches", C.c_int64),
        ("prof_bytes_per_launch", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("rank", C.c_int32), ("world", C.c_int32), ("pad_", C.c_int32),
        ("coarse_sparse", C.c_int32), ("coarse_nodes", C.c_int64), ("coarse_levels", C.c_int64), ("coarse_factor_bytes", C.c_double),
        ("n_nonlinear", C.c_int64), ("newton_iters", C.c_int64), ("linear_solves", C.c_int64), ("hist_len", C.c_int64),
        ("ms_newton_numeric", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "pad_"}


class TcgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_LIB = None


def lib():
    """Load the in-tree C-ABI library (raises if it is missing: no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIBPATH):
        raise ImportError(f"{LIBPATH} not built: run `python -m paper_2510_23446_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIBPATH)
    vp, dp, ip, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64)
    L.tcg_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.c_char_p, vp]
    L.tcg_set_patches.argtypes = [vp, ip, dp, dp, C.c_int, ip]
    L.tcg_set_materials.argtypes = [vp, dp, dp, C.c_size_t]
    L.tcg_set_source.argtypes = [vp, C.c_int, dp, C.c_size_t]
    L.tcg_set_time.argtypes = [vp, C.c_double, C.c_int]
    L.tcg_set_solver.argtypes = [vp, C.c_double, C.c_int, C.c_int, C.c_int]
    L.tcg_set_warm_start.argtypes = [vp, C.c_int]
    L.tcg_plan.argtypes = [vp]
    L.tcg_get_plan.argtypes = [vp, C.c_int, i64p, C.c_size_t]
    L.tcg_setup.argtypes = [vp]
    L.tcg_refactor.argtypes = [vp]
    L.tcg_step.argtypes = [vp, C.c_int]
    L.tcg_get_coefficients.argtypes = [vp, C.c_int, dp, C.c_size_t]
    L.tcg_get_history.argtypes = [vp, ip, dp, C.c_size_t, dp, C.c_size_t]
    L.tcg_get_info.argtypes = [vp, C.POINTER(TcgInfo)]
    L.tcg_fapply.argtypes = [vp, dp, dp, C.c_size_t]
    L.tcg_bench_fapply.argtypes = [vp, C.c_int, dp]
    L.tcg_set_profile.argtypes = [vp, C.c_int]
    L.tcg_set_virtual_ranks.argtypes = [vp, C.c_int]
    L.tcg_nccl_unique_id.argtypes = [C.c_char_p]
    L.tcg_last_error.argtypes = [vp]
    L.tcg_last_error.restype = C.c_char_p
    if hasattr(L, "tcg_get_errors") or not os.environ.get("TCG_LIBPATH"):  # (older A/B builds lack them)
        L.tcg_set_error_tracking.argtypes = [vp, C.c_int]
        L.tcg_get_errors.argtypes = [vp, dp, dp, dp, C.c_size_t]
    if hasattr(L, "tcg_set_nonlinear") or not os.environ.get("TCG_LIBPATH"):
        L.tcg_set_nonlinear.argtypes = [vp, dp, C.c_size_t, C.c_double, C.c_int]
        L.tcg_get_newton.argtypes = [vp, ip, C.c_size_t, ip, dp, C.c_size_t]
    L.tcg_destroy.argtypes = [vp]
    L.tcg_destroy.restype = None
    for n in EXPORTS:
        if n not in ("tcg_last_error", "tcg_destroy") and (hasattr(L, n) or not os.environ.get("TCG_LIBPATH")):
            getattr(L, n).restype = C.c_int
    _LIB = L
    return L


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a multi-GPU handle (rank 0 creates, all ranks pass it)."""
    buf = C.create_string_buffer(128)
    st = lib().tcg_nccl_unique_id(buf)
    if st != TCG_OK:
        raise TcgError(st, "ncclGetUniqueId failed")
    return buf.raw


class Solver:
    """One handle of the C ABI. Arguments mirror include/tcg_ietidp.h."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None, stream=None):
        self.L = lib()
        self.h = C.c_void_p()
        st = self.L.tcg_create(C.byref(self.h), device, rank, world, nccl_id, stream)
        if st != TCG_OK:
            msg = self.L.tcg_last_error(self.h).decode() if self.h else "tcg_create failed"
            raise TcgError(st, msg)

    def _ck(self, st):
        if st != TCG_OK:
            raise TcgError(st, self.L.tcg_last_error(self.h).decode())

    def set_patches(self, npatch, lo, hi, p, elems):
        self._ck(self.L.tcg_set_patches(self.h, (C.c_int * 3)(*npatch), (C.c_double * 3)(*lo),
                                        (C.c_double * 3)(*hi), int(p), (C.c_int * 3)(*elems)))

    def set_materials(self, sigma, nu):
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        n = np.ascontiguousarray(nu, dtype=np.float64)
        self._ck(self.L.tcg_set_materials(self.h, _dptr(s), _dptr(n), len(s)))

    def set_source(self, kind, params=()):
        """J = amp * phi(t) * S(x): kind 1 params (amp, freq), kind 2 (amp,), kind 0 ()."""
        p = np.ascontiguousarray(params, dtype=np.float64)
        self._ck(self.L.tcg_set_source(self.h, int(kind), _dptr(p) if p.size else None, p.size))

    def set_time(self, T, n_steps):
        self._ck(self.L.tcg_set_time(self.h, float(T), int(n_steps)))

    def set_solver(self, rtol=1e-10, max_iter=5000, scaling=1, tree_order=0):
        self._ck(self.L.tcg_set_solver(self.h, float(rtol), int(max_iter), int(scaling), int(tree_order)))

    def set_warm_start(self, k=4):
        """PCG of every step after the first starts from the Galerkin projection on the
        previous k solutions (R20); 0 = the paper's lambda0 = 0."""
        self._ck(self.L.tcg_set_warm_start(self.h, int(k)))
        return self

    def set_error_tracking(self, on=True):
        """Accumulate the paper's eps_B, eps_E every step (source 3 only)."""
        self._ck(self.L.tcg_set_error_tracking(self.h, int(bool(on))))
        return self

    def errors(self, per_step=False):
        """(eps_B, eps_E) and, with per_step, the (e_B, e_E) pairs of every step done."""
        eb, ee = C.c_double(), C.c_double()
        ns = self.info()["steps_done"] if per_step else 0
        ps = np.zeros(2 * max(ns, 1))
        self._ck(self.L.tcg_get_errors(self.h, C.byref(eb), C.byref(ee), _dptr(ps) if per_step else None, ns))
        return (eb.value, ee.value, ps[:2 * ns].reshape(-1, 2)) if per_step else (eb.value, ee.value)

    def set_nonlinear(self, k, newton_tol=1e-8, newton_max=20):
        """Brauer reluctivity nu = k1 exp(k2 |B|^2) + k3 per patch (k: (P, 3); zero rows linear)
        with Newton's method per step (R25)."""
        k = np.ascontiguousarray(k, dtype=np.float64).reshape(-1)
        self._ck(self.L.tcg_set_nonlinear(self.h, _dptr(k) if k.size else None, k.size // 3, float(newton_tol),
                                          int(newton_max)))
        return self

    def newton(self):
        """(Newton iterations per step, PCG iterations per linear solve, increments per solve)."""
        inf = self.info()
        ns, nv = inf["steps_done"] if inf["n_nonlinear"] else 0, inf["linear_solves"]
        ni = np.zeros(max(ns, 1), dtype=np.int32)
        si = np.zeros(max(nv, 1), dtype=np.int32)
        inc = np.zeros(max(nv, 1))
        self._ck(self.L.tcg_get_newton(self.h, ni.ctypes.data_as(C.POINTER(C.c_int)), ns,
                                       si.ctypes.data_as(C.POINTER(C.c_int)), _dptr(inc), nv))
        return ni[:ns], si[:nv], inc[:nv]

    def configure(self, prob):
        """Set everything from a problem description with the fields of workloads.Problem."""
        self.set_patches(prob.npatch, prob.lo, prob.hi, prob.p, prob.elems)
        self.set_materials(prob.sigma, prob.nu)
        self.set_source(prob.source, getattr(prob, "source_params", ()))
        self.set_time(prob.T, prob.n_steps)
        self.set_solver(prob.rtol, prob.max_iter, prob.scaling, prob.tree_order)
        self.set_warm_start(getattr(prob, "warm_start", 0))
        if getattr(prob, "nl", None) is not None:
            self.set_nonlinear(prob.nl, getattr(prob, "newton_tol", 1e-8), getattr(prob, "newton_max", 20))
        if getattr(prob, "track_errors", False):
            self.set_error_tracking(True)
        return self

    def plan(self):
        self._ck(self.L.tcg_plan(self.h))

    def plan_array(self, what, n):
        out = np.zeros(n, dtype=np.int64)
        self._ck(self.L.tcg_get_plan(self.h, int(what), out.ctypes.data_as(C.POINTER(C.c_int64)), n))
        return out

    def setup(self):
        self._ck(self.L.tcg_setup(self.h))

    def refactor(self):
        self._ck(self.L.tcg_refactor(self.h))

    def step(self, n=1):
        self._ck(self.L.tcg_step(self.h, int(n)))

    def info(self):
        inf = TcgInfo()
        self._ck(self.L.tcg_get_info(self.h, C.byref(inf)))
        return inf.as_dict()

    def coefficients(self, layout=1, out=None):
        inf = self.info()
        n = inf["n_edges"] if layout == 1 else inf["n_patches"] * inf["n_local"]
        if out is None:
            out = np.zeros(n)
        self._ck(self.L.tcg_get_coefficients(self.h, int(layout), _dptr(out), n))
        return out

    def history(self):
        inf = self.info()
        ns = inf["steps_done"]
        it = np.zeros(ns, dtype=np.int32)
        fr = np.zeros(ns)
        self._ck(self.L.tcg_get_history(self.h, it.ctypes.data_as(C.POINTER(C.c_int)), _dptr(fr), ns, None, 0))
        hl = int(inf["hist_len"])
        hist = np.zeros(max(hl, 1))
        self._ck(self.L.tcg_get_history(self.h, None, None, ns, _dptr(hist), hl))
        return it, fr, hist[:hl]

    def set_virtual_ranks(self, n):
        self._ck(self.L.tcg_set_virtual_ranks(self.h, int(n)))

    def set_profile(self, kernel_id):
        self._ck(self.L.tcg_set_profile(self.h, int(kernel_id)))

    def apply_F(self, lam):
        """q = F lam (the dual operator, through the C ABI; lam of length m)."""
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        q = np.empty_like(lam)
        self._ck(self.L.tcg_fapply(self.h, _dptr(lam), _dptr(q), lam.size))
        return q

    def bench_fapply(self, n):
        ms = C.c_double()
        self._ck(self.L.tcg_bench_fapply(self.h, int(n), C.byref(ms)))
        return ms.value

    def close(self):
        if self.h:
            self.L.tcg_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
