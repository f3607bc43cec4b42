"""ctypes binding of libbbot.so (include/bbot.h).  Argument marshalling only:
every arithmetic step runs in the library's CUDA kernels.  There is no CPU
fallback -- if the shared library is missing, importing this module raises.

Vectors may be numpy arrays (host, float64, C-contiguous) or torch CUDA
tensors (device, float64, contiguous); the memory kind is passed to the C-ABI.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BBOT_LIB") or os.path.join(_HERE, "libbbot.so")   # BBOT_LIB: A/B builds

BBOT_MEM_HOST, BBOT_MEM_DEVICE = 0, 1
STATUS = {0: "OK", 1: "E_INPUT", 2: "E_GEOMETRY", 3: "E_STATE", 4: "E_NOCONV", 5: "E_CUDA",
          6: "E_NCCL", 7: "E_NOMEM", 8: "E_INTERNAL", 9: "E_ORDER"}


class SolverOpts(C.Structure):
    _fields_ = [("eps_out", C.c_double), ("eps_T", C.c_double), ("eps_A", C.c_double),
                ("restart", C.c_int), ("maxit", C.c_int), ("restart_T", C.c_int),
                ("maxit_inner", C.c_int), ("omega_A", C.c_double), ("omega_T", C.c_double),
                ("coarse_max_A", C.c_int), ("coarse_max_T", C.c_int),
                ("precond", C.c_int), ("coarse_max_S", C.c_int),   # 0 = BB, 1 = SIMPLE (NEXT f1), 2 = HSS (f2)
                ("alpha_hss", C.c_double), ("eps_in_hss", C.c_double),
                ("recon", C.c_int)]                                # 0 = arithmetic, 1 = harmonic (f4)


class SolveStats(C.Structure):
    _fields_ = [("outer_its", C.c_int), ("inner_T_its", C.c_int), ("inner_A_its_max", C.c_int),
                ("inner_A_its_total", C.c_longlong), ("converged", C.c_int), ("rel_res", C.c_double),
                ("scale", C.c_double), ("t_assemble_ms", C.c_double), ("t_setup_ms", C.c_double),
                ("t_krylov_ms", C.c_double), ("t_recover_ms", C.c_double),
                ("amg_levels_A", C.c_int), ("amg_levels_T", C.c_int), ("t_graph_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class IpmOpts(C.Structure):
    _fields_ = [("mu0", C.c_double), ("mu_factor", C.c_double), ("mu_min", C.c_double),
                ("newton_rel_tol", C.c_double), ("newton_abs_floor", C.c_double),
                ("frac_to_boundary", C.c_double), ("newton_max", C.c_int), ("max_mu_steps", C.c_int),
                ("mu_tight", C.c_double), ("eps_A_tight", C.c_double),
                ("simple_below_mu", C.c_double)]   # A34 hybrid


class IpmRecord(C.Structure):
    _fields_ = [("mu", C.c_double), ("newton", C.c_int), ("alpha", C.c_double), ("res_norm", C.c_double),
                ("solve", SolveStats)]


class IpmStats(C.Structure):
    _fields_ = [("n_systems", C.c_int), ("total_outer", C.c_longlong), ("total_inner_T", C.c_longlong),
                ("n_unconverged", C.c_int), ("final_mu", C.c_double), ("kinetic_energy", C.c_double),
                ("wall_ms", C.c_double), ("n_simple_fallback", C.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


IPM_CB = C.CFUNCTYPE(None, C.POINTER(IpmRecord), C.c_void_p)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbbot.so not built ({LIB_PATH}); run python -m paper_2209_00315_b200._build")
lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_sigs = {
    "bbot_default_solver_opts": (None, [C.POINTER(SolverOpts)]),
    "bbot_default_ipm_opts": (None, [C.POINTER(IpmOpts)]),
    "bbot_create": (C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int, _P, _P, C.POINTER(SolverOpts), _P,
                              C.POINTER(C.c_void_p)]),
    "bbot_destroy": (None, [_P]),
    "bbot_last_error": (C.c_char_p, [_P]),
    "bbot_sizes": (C.c_int, [_P] + [C.POINTER(C.c_longlong)] * 3 + [C.POINTER(C.c_int)]
                   + [C.POINTER(C.c_longlong)] * 2),
    "bbot_set_opts": (C.c_int, [_P, C.POINTER(SolverOpts)]),
    "bbot_T_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    "bbot_set_state": (C.c_int, [_P, _P, _P, _P, C.c_double, C.c_int]),
    "bbot_get_state": (C.c_int, [_P, _P, _P, _P, _D, C.c_int]),
    "bbot_init_state": (C.c_int, [_P, C.c_double]),
    "bbot_residual": (C.c_int, [_P, _P, _P, _P, _D, C.c_int]),
    "bbot_assemble": (C.c_int, [_P]),
    "bbot_jp_matvec": (C.c_int, [_P, _P, _P, C.c_int]),
    "bbot_bb_apply": (C.c_int, [_P, _P, _P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bbot_solve": (C.c_int, [_P, _P, _P, _P, C.POINTER(SolveStats), C.c_int]),
    "bbot_solve_rhs": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, C.POINTER(SolveStats), C.c_int]),
    "bbot_newton_update": (C.c_int, [_P, C.c_double, _D]),
    "bbot_ipm_run": (C.c_int, [_P, C.POINTER(IpmOpts), C.POINTER(IpmStats), IPM_CB, C.c_void_p]),
    "bbot_kinetic_energy": (C.c_int, [_P, _D]),
    "bbot_get_T": (C.c_int, [_P, C.POINTER(C.c_longlong), _P, _P, _P]),
    "bbot_amg_info": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    "bbot_amg_agg": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "bbot_amg_level_info": (C.c_int, [_P, C.c_int, C.c_int] + [C.POINTER(C.c_longlong)] * 3 + [C.POINTER(C.c_int)]),
    "bbot_amg_vcycle": (C.c_int, [_P, C.c_int, _P, _P, C.c_int]),
    "bbot_launch_count": (C.c_longlong, [_P]),
    "bbot_mem_usage": (C.c_int, [_P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "bbot_set_exec_mode": (C.c_int, [_P, C.c_int]),
    "bbot_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "bbot_set_dist": (C.c_int, [_P, C.c_int, C.c_int, C.c_char_p]),
    "bbot_set_dist_virtual": (C.c_int, [_P, C.c_int, C.c_int, C.c_longlong]),
    "bbot_get_slab": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bbot_slab_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bbot_time_blocks": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "bbot_prof_start": (C.c_int, [_P]),
    "bbot_prof_stop": (C.c_int, [_P, C.c_char_p, C.c_longlong, C.POINTER(C.c_longlong)]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


class BbotError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib.bbot_nccl_unique_id(buf)
    if st != 0:
        raise BbotError(st, "bbot_nccl_unique_id failed (see stderr)")
    return buf.raw


def slab_plan(Kp1: int, nranks: int, rank: int, S: int):
    """(lo, hi): the slices of an S-slice vector that `rank` owns (bbot_slab_plan)."""
    lo, hi = C.c_int(), C.c_int()
    st = lib.bbot_slab_plan(int(Kp1), int(nranks), int(rank), int(S), C.byref(lo), C.byref(hi))
    if st != 0:
        raise BbotError(st, "bbot_slab_plan: bad arguments")
    return lo.value, hi.value


def time_blocks(K: int):
    """(B, nb): the AMG(T) time blocks of a K-slice problem (bbot_time_blocks, A42)."""
    b, nb = C.c_int(), C.c_int()
    st = lib.bbot_time_blocks(int(K), C.byref(b), C.byref(nb))
    if st != 0:
        raise BbotError(st, "bbot_time_blocks: bad arguments")
    return b.value, nb.value


def default_solver_opts(**kw) -> SolverOpts:
    o = SolverOpts()
    lib.bbot_default_solver_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def default_ipm_opts(**kw) -> IpmOpts:
    o = IpmOpts()
    lib.bbot_default_ipm_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _ptr(a, n=None, writable=False):
    """(pointer, memkind) of a numpy array or torch tensor."""
    if a is None:
        return None, BBOT_MEM_HOST
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous or (writable and not a.flags.writeable):
            raise TypeError("expected a C-contiguous float64 numpy array")
        if n is not None and a.size != n:
            raise ValueError(f"expected {n} values, got {a.size}")
        return a.ctypes.data_as(C.c_void_p), BBOT_MEM_HOST
    # torch tensor
    if getattr(a, "dtype", None) is not None and str(a.dtype) == "torch.float64" and a.is_contiguous():
        if n is not None and a.numel() != n:
            raise ValueError(f"expected {n} values, got {a.numel()}")
        return C.c_void_p(a.data_ptr()), (BBOT_MEM_DEVICE if a.is_cuda else BBOT_MEM_HOST)
    raise TypeError("expected numpy float64 array or contiguous torch float64 tensor")


class Context:
    """One bbot_ctx (one GPU)."""

    def __init__(self, verts, tris, K, rho_in, rho_f, opts: SolverOpts | None = None, stream=None):
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        tris = np.ascontiguousarray(tris, dtype=np.int32)
        rho_in = np.ascontiguousarray(rho_in, dtype=np.float64)
        rho_f = np.ascontiguousarray(rho_f, dtype=np.float64)
        self._h = C.c_void_p()
        st = lib.bbot_create(verts.ctypes.data_as(C.c_void_p), verts.shape[0], tris.ctypes.data_as(C.c_void_p),
                             tris.shape[0], int(K), rho_in.ctypes.data_as(C.c_void_p),
                             rho_f.ctypes.data_as(C.c_void_p), C.byref(opts) if opts is not None else None,
                             C.c_void_p(stream) if stream else None, C.byref(self._h))
        if st != 0:
            raise BbotError(st, "bbot_create failed (see stderr)")
        nbar, N, NE, n, m = (C.c_longlong() for _ in range(5))
        Kc = C.c_int()
        lib.bbot_sizes(self._h, C.byref(nbar), C.byref(N), C.byref(NE), C.byref(Kc), C.byref(n), C.byref(m))
        self.nbar, self.N, self.NE, self.K, self.n, self.m = (nbar.value, N.value, NE.value, Kc.value,
                                                              n.value, m.value)

    def _check(self, st):
        if st != 0:
            raise BbotError(st, lib.bbot_last_error(self._h).decode())

    def close(self):
        if self._h:
            lib.bbot_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def T_width(self):
        return self.T_nnz()[1]

    def T_nnz(self):
        W, nnz = C.c_int(), C.c_longlong()
        self._check(lib.bbot_T_info(self._h, C.byref(W), C.byref(nnz)))
        return nnz.value, W.value

    # ---- state
    def set_opts(self, opts: SolverOpts):
        self._check(lib.bbot_set_opts(self._h, C.byref(opts)))

    def set_state(self, phi, rho, s, mu):
        pp, mem = _ptr(phi, self.n)
        pr, _ = _ptr(rho, self.m)
        ps, _ = _ptr(s, self.m)
        self._check(lib.bbot_set_state(self._h, pp, pr, ps, float(mu), mem))

    def get_state(self, phi=None, rho=None, s=None):
        if phi is None:
            phi, rho, s = np.empty(self.n), np.empty(self.m), np.empty(self.m)
        mu = C.c_double()
        pp, mem = _ptr(phi, self.n, True)
        self._check(lib.bbot_get_state(self._h, pp, _ptr(rho, self.m, True)[0], _ptr(s, self.m, True)[0],
                                       C.byref(mu), mem))
        return phi, rho, s, mu.value

    def init_state(self, mu0=1.0):
        self._check(lib.bbot_init_state(self._h, float(mu0)))

    def residual(self):
        F_phi, F_rho, F_s = np.empty(self.n), np.empty(self.m), np.empty(self.m)
        nrm = C.c_double()
        self._check(lib.bbot_residual(self._h, _ptr(F_phi)[0], _ptr(F_rho)[0], _ptr(F_s)[0], C.byref(nrm),
                                      BBOT_MEM_HOST))
        return F_phi, F_rho, F_s, nrm.value

    # ---- hot path
    def assemble(self):
        self._check(lib.bbot_assemble(self._h))

    def jp_matvec(self, x, y=None):
        y = np.empty(self.n + self.m) if y is None else y
        px, mem = _ptr(x, self.n + self.m)
        self._check(lib.bbot_jp_matvec(self._h, px, _ptr(y, self.n + self.m, True)[0], mem))
        return y

    def bb_apply(self, r, z=None):
        z = np.empty(self.n + self.m) if z is None else z
        pr, mem = _ptr(r, self.n + self.m)
        it_t, it_a = C.c_int(), C.c_int()
        self._check(lib.bbot_bb_apply(self._h, pr, _ptr(z, self.n + self.m, True)[0], mem, C.byref(it_t),
                                      C.byref(it_a)))
        return z, it_t.value, it_a.value

    def solve(self, dphi=None, drho=None, ds=None):
        """FGMRES + recovery; returns (dphi, drho, ds, stats).  Pass torch device
        tensors to keep the direction on the GPU; None -> host numpy."""
        host = dphi is None
        if host:
            dphi, drho, ds = np.empty(self.n), np.empty(self.m), np.empty(self.m)
        st = SolveStats()
        pp, mem = _ptr(dphi, self.n, True)
        self._check(lib.bbot_solve(self._h, pp, _ptr(drho, self.m, True)[0], _ptr(ds, self.m, True)[0],
                                   C.byref(st), mem))
        return dphi, drho, ds, st.as_dict()

    def solve_rhs(self, f, g, h, dphi=None, drho=None, ds=None):
        """solve(rhs) -> direction: the Newton system (3.1) of the last assembly with a
        caller-given (f; g; h) (bbot_solve_rhs).  numpy inputs -> numpy outputs; torch
        device tensors (outputs must be given) -> the direction stays on the GPU."""
        host = isinstance(f, np.ndarray)
        if host:
            f, g, h = (np.ascontiguousarray(a, dtype=np.float64) for a in (f, g, h))
            dphi, drho, ds = np.empty(self.n), np.empty(self.m), np.empty(self.m)
        st = SolveStats()
        fp, mem = _ptr(f, self.n)
        self._check(lib.bbot_solve_rhs(self._h, fp, _ptr(g, self.m)[0], _ptr(h, self.m)[0],
                                       _ptr(dphi, self.n, True)[0], _ptr(drho, self.m, True)[0],
                                       _ptr(ds, self.m, True)[0], C.byref(st), mem))
        return dphi, drho, ds, st.as_dict()

    def solve_stats_only(self):
        st = SolveStats()
        self._check(lib.bbot_solve(self._h, None, None, None, C.byref(st), BBOT_MEM_DEVICE))
        return st.as_dict()

    def newton_update(self, tau=0.95):
        a = C.c_double()
        self._check(lib.bbot_newton_update(self._h, float(tau), C.byref(a)))
        return a.value

    def ipm_run(self, opts: IpmOpts | None = None, callback=None):
        st = IpmStats()
        log = []

        def _cb(rec, user):
            r = rec.contents
            d = dict(mu=r.mu, newton=r.newton, alpha=r.alpha, res=r.res_norm, **r.solve.as_dict())
            log.append(d)
            if callback:
                callback(d)
        cb = IPM_CB(_cb)
        self._check(lib.bbot_ipm_run(self._h, C.byref(opts) if opts is not None else None, C.byref(st), cb, None))
        return st.as_dict(), log

    def kinetic_energy(self):
        v = C.c_double()
        self._check(lib.bbot_kinetic_energy(self._h, C.byref(v)))
        return v.value

    # ---- inspection
    def get_T(self):
        nnz = C.c_longlong()
        self._check(lib.bbot_get_T(self._h, C.byref(nnz), None, None, None))
        rp = np.empty(self.m + 1, dtype=np.int64)
        ci = np.empty(nnz.value, dtype=np.int32)
        cv = np.empty(nnz.value, dtype=np.float64)
        self._check(lib.bbot_get_T(self._h, C.byref(nnz), rp.ctypes.data_as(C.c_void_p),
                                   ci.ctypes.data_as(C.c_void_p), cv.ctypes.data_as(C.c_void_p)))
        return rp, ci, cv

    def amg_info(self, which):
        nl = C.c_int()
        sizes = (C.c_longlong * 32)()
        self._check(lib.bbot_amg_info(self._h, which, C.byref(nl), sizes))
        return [sizes[i] for i in range(nl.value)]

    def amg_levels(self, which):
        """[(n, nnz, nc)] per level (nnz -1 on level 0) and the tail's first level."""
        out, tail = [], C.c_int()
        for lvl in range(len(self.amg_info(which))):
            n, nnz, nc = C.c_longlong(), C.c_longlong(), C.c_longlong()
            self._check(lib.bbot_amg_level_info(self._h, which, lvl, C.byref(n), C.byref(nnz), C.byref(nc),
                                                C.byref(tail)))
            out.append((n.value, nnz.value, nc.value))
        return out, tail.value

    def amg_agg(self, which, level):
        sizes = self.amg_info(which)
        out = np.empty(sizes[level], dtype=np.int32)
        self._check(lib.bbot_amg_agg(self._h, which, level, out.ctypes.data_as(C.c_void_p)))
        return out

    def amg_vcycle(self, which, b):
        x = np.empty_like(b)
        pb, mem = _ptr(b)
        self._check(lib.bbot_amg_vcycle(self._h, which, pb, _ptr(x, writable=True)[0], mem))
        return x

    def launch_count(self):
        return lib.bbot_launch_count(self._h)

    def mem_usage(self):
        """(used, peak) bytes of the library's device memory pool (bbot_mem_usage)."""
        u, pk = C.c_longlong(), C.c_longlong()
        self._check(lib.bbot_mem_usage(self._h, C.byref(u), C.byref(pk)))
        return u.value, pk.value

    def set_dist(self, rank: int, nranks: int, uid: bytes | None):
        """Time-slab decomposition over NCCL (uid: 128 bytes from nccl_unique_id() on rank 0)."""
        if uid is not None and len(uid) != 128:
            raise ValueError("uid must be 128 bytes")
        self._check(lib.bbot_set_dist(self._h, int(rank), int(nranks), uid))

    def set_dist_virtual(self, rank: int, nranks: int, group: int):
        """Time-slab decomposition among the contexts of THIS process sharing `group` (device-to-
        device exchange; each rank's calls must run concurrently, one thread per rank)."""
        self._check(lib.bbot_set_dist_virtual(self._h, int(rank), int(nranks), int(group)))

    def slab(self):
        a, b = C.c_int(), C.c_int()
        self._check(lib.bbot_get_slab(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_exec_mode(self, use_graph: bool):
        """True: each solve is one CUDA-graph launch (device-side loops); False: eager."""
        self._check(lib.bbot_set_exec_mode(self._h, 1 if use_graph else 0))

    def prof_start(self):
        self._check(lib.bbot_prof_start(self._h))

    def prof_stop(self, by_grid=False):
        """-> {kernel name: (launches, total_ms)}; by_grid: {(name, grid CTAs): (launches, ms)}"""
        need = C.c_longlong()
        buf = C.create_string_buffer(1 << 22)
        self._check(lib.bbot_prof_stop(self._h, buf, len(buf), C.byref(need)))
        out = {}
        for line in buf.value.decode(errors="replace").splitlines():
            name, cnt, ms, grid = line.rsplit("\t", 3)
            key = (name, int(grid)) if by_grid else name
            c0, m0 = out.get(key, (0, 0.0))
            out[key] = (c0 + int(cnt), m0 + float(ms))
        return out
