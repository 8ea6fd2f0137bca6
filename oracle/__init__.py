"""ORACLE TEST INFRASTRUCTURE -- not product code.

ctypes front-ends for
  * ``oracle/_ref/libhlf_refc.so``: the reference's own C++ sources
    (/root/reference/proj/src) compiled unchanged against oracle/shim
    (``RefStepper1d``, ``ref_build_interp``, ``ref_reconstruct_2d`` ...);
  * ``oracle/_build/libhlf_oracle.so``: the d = 1..3 CPU restatement
    (``OracleStepper``), see oracle/hlf_oracle.cpp for the file:line map.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
reference arm may import this package, and only as the checker or the
timed CPU baseline -- never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libhlf_refc.so")
ORACLE_SO = os.path.join(HERE, "_build", "libhlf_oracle.so")
ORACLE_FMA_SO = os.path.join(HERE, "_build", "libhlf_oracle_fma.so")
REF_TESTS = [os.path.join(HERE, "_ref", t) for t in ("test_jet", "test_interpolation", "test_stepper1d")]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(ref: bool = True) -> None:
    """Build the restatement (always) and the compiled reference (when
    /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


_ref_lib = None
_orc_lib = None
_orc_fma_lib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_build_interp.argtypes = [C.c_int, _dp, _dp]
        L.ref_build_interp.restype = C.c_int
        L.ref_reconstruct_2d.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_reconstruct_1d.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref1d_create.argtypes = [C.c_char_p, C.c_uint, C.c_int, C.c_int]
        L.ref1d_create.restype = C.c_void_p
        L.ref1d_destroy.argtypes = [C.c_void_p]
        L.ref1d_info.argtypes = [C.c_void_p, _dp]
        L.ref1d_init.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.ref1d_get.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref1d_set.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref1d_set_dt.argtypes = [C.c_void_p, C.c_double]
        L.ref1d_advance_p.argtypes = [C.c_void_p]
        L.ref1d_advance_v.argtypes = [C.c_void_p]
        L.ref1d_steps.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref1d_steps.restype = C.c_int
        for f in ("ref1d_l2_p", "ref1d_l2_v"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_double
        for f in ("ref1d_conserved_q", "ref1d_conserved_r"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_double]
            getattr(L, f).restype = C.c_double
        L.ref1d_coeff.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.ref1d_forcing.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp]
        L.ref1d_forcing.restype = None
        L.ref1d_has_forcing.argtypes = [C.c_void_p]
        L.ref1d_has_forcing.restype = C.c_int
        for f in ("ref1d_init_modified", "ref1d_init_dual"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.ref1d_get_modified.argtypes = [C.c_void_p] + [_dp] * 5
        L.ref1d_get_dual.argtypes = [C.c_void_p] + [_dp] * 3
        for f in ("ref1d_steps_modified", "ref1d_steps_dual"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, C.c_int]
            getattr(L, f).restype = C.c_int
        L.ref2d_exact.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.ref2d_exact.restype = C.c_int
        L.ref2d_l2_acoustics.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 6 + [C.c_int, _dp, C.c_int, C.c_double]
        L.ref2d_l2_acoustics.restype = C.c_double
        L.ref_convergence_rate.argtypes = [C.c_int, _dp, _dp]
        L.ref_convergence_rate.restype = C.c_double
        L.ref_dt_nominal.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        L.ref_dt_nominal.restype = C.c_double
        L.ref_step_count.argtypes = [C.c_double, C.c_double]
        L.ref_step_count.restype = C.c_int
        _ref_lib = L
    return _ref_lib


def orc_lib(fma: bool = False):
    """The restatement; fma=True loads the build with compiler-contracted FMAs
    (same algorithm, another valid rounding: the long-run drift yardstick)."""
    global _orc_lib, _orc_fma_lib
    cached = _orc_fma_lib if fma else _orc_lib
    if cached is None:
        so = ORACLE_FMA_SO if fma else ORACLE_SO
        if not os.path.exists(so):
            raise FileNotFoundError(f"{so} missing: run `make -C oracle oracle`")
        L = C.CDLL(so)
        L.orc_create.argtypes = [C.c_int, C.c_int, _ip, _ip, C.c_double, C.c_double, C.c_double, C.c_int]
        L.orc_create.restype = C.c_void_p
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_get_M.argtypes = [C.c_int, _dp]
        L.orc_set_M.argtypes = [C.c_void_p, _dp]
        L.orc_num_nodes.argtypes = [C.c_void_p, C.c_int]
        L.orc_num_nodes.restype = C.c_longlong
        L.orc_set_field.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_get_field.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_set_coeff.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.orc_set_forcing.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_set_times.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
        L.orc_get_times.argtypes = [C.c_void_p, _dp]
        L.orc_advance_p.argtypes = [C.c_void_p]
        L.orc_advance_v.argtypes = [C.c_void_p]
        L.orc_advance_n.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_advance_n.restype = C.c_int
        L.orc_reconstruct.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_set_slab.argtypes = [C.c_void_p, C.c_int]
        L.orc_get_layer.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.orc_set_halo.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.orc_add_separable.argtypes = [C.c_int, _ip, _dp, C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp, _dp]
        if fma:
            _orc_fma_lib = L
        else:
            _orc_lib = L
        cached = L
    return cached


# ---------------------------------------------------------------- reference


def ref_build_interp(m: int) -> tuple[np.ndarray, float]:
    n = 2 * m + 2
    M = np.zeros(n * n)
    cond = np.zeros(1)
    if ref_lib().ref_build_interp(m, _ptr(M), _ptr(cond)) != 0:
        raise ValueError("ConfigError")
    return M.reshape(n, n), float(cond[0])


def ref_reconstruct_2d(m, c00, c10, c01, c11) -> np.ndarray:
    n = 2 * m + 2
    out = np.zeros(n * n)
    args = [np.ascontiguousarray(c, dtype=np.float64).ravel() for c in (c00, c10, c01, c11)]
    ref_lib().ref_reconstruct_2d(m, *[_ptr(a) for a in args], _ptr(out))
    return out.reshape(n, n)


def ref2d_exact(name: str, f: int, x: float, y: float, t: float, h: float, n: int) -> np.ndarray:
    out = np.zeros(n * n)
    if ref_lib().ref2d_exact(name.encode(), f, x, y, t, h, n, _ptr(out)) != 0:
        raise ValueError(name)
    return out.reshape(n, n)


class RefStepper1d:
    """The reference's own ``Stepper1d`` (proj/src/stepper1d.cpp) behind ctypes."""

    def __init__(self, problem: str, m: int, K: int, seed: int = 1234):
        self.L = ref_lib()
        self.h_ = self.L.ref1d_create(problem.encode(), seed, m, K)
        if not self.h_:
            raise ValueError(f"cannot build reference stepper for {problem}")
        self.m, self.K = m, K
        info = np.zeros(4)
        self.L.ref1d_info(self.h_, _ptr(info))
        self.x_min, self.x_max, self.c_max, self.h = (float(v) for v in info)

    def __del__(self):
        if getattr(self, "h_", None):
            self.L.ref1d_destroy(self.h_)
            self.h_ = None

    def init_leapfrog(self, dt: float, t0: float = 0.0):
        self.L.ref1d_init(self.h_, dt, t0)

    def get(self):
        n1 = self.m + 1
        p = np.zeros(self.K * n1)
        v = np.zeros(self.K * n1)
        t = np.zeros(3)
        self.L.ref1d_get(self.h_, _ptr(p), _ptr(v), _ptr(t))
        return p.reshape(self.K, n1), v.reshape(self.K, n1), tuple(float(x) for x in t)

    def set(self, p, v, times):
        p = np.ascontiguousarray(p, dtype=np.float64).ravel()
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        t = np.asarray(times, dtype=np.float64)
        self.L.ref1d_set(self.h_, _ptr(p), _ptr(v), _ptr(t))

    def set_dt(self, dt):
        self.L.ref1d_set_dt(self.h_, dt)

    def advance_p(self):
        self.L.ref1d_advance_p(self.h_)

    def advance_v(self):
        self.L.ref1d_advance_v(self.h_)

    def steps(self, n: int, first: int = 0) -> int:
        return self.L.ref1d_steps(self.h_, n, first)

    def l2_p(self) -> float:
        return self.L.ref1d_l2_p(self.h_)

    def l2_v(self) -> float:
        return self.L.ref1d_l2_v(self.h_)

    def conserved_q(self, c: float = 1.0) -> float:
        return self.L.ref1d_conserved_q(self.h_, c)

    def conserved_r(self, c: float = 1.0) -> float:
        return self.L.ref1d_conserved_r(self.h_, c)

    def coeff(self, which: int, on_dual: bool) -> np.ndarray:
        n = 2 * self.m + 2
        out = np.zeros(self.K * n)
        self.L.ref1d_coeff(self.h_, which, int(on_dual), _ptr(out))
        return out.reshape(self.K, n)

    def forcing(self, on_dual: bool, t: float) -> np.ndarray:
        """forcing_at(x_j, t)(r) at every node: [K, 2m+1, 2m+2] (the table of hlf_set_forcing)"""
        n = 2 * self.m + 2
        out = np.zeros(self.K * (n - 1) * n)
        self.L.ref1d_forcing(self.h_, int(on_dual), t, _ptr(out))
        return out.reshape(self.K, n - 1, n)

    def has_forcing(self) -> bool:
        return bool(self.L.ref1d_has_forcing(self.h_))

    # the reference's alternative time schemes (stepper1d.cpp:174-272)
    def init_modified(self, dt: float, t0: float = 0.0):
        self.L.ref1d_init_modified(self.h_, dt, t0)

    def get_modified(self):
        """(p primary, v primary, p dual, v dual) as [K, m+1] arrays, and (t, dt)"""
        n1 = self.m + 1
        arrs = [np.zeros(self.K * n1) for _ in range(4)]
        tdt = np.zeros(2)
        self.L.ref1d_get_modified(self.h_, *[_ptr(a) for a in arrs], _ptr(tdt))
        return [a.reshape(self.K, n1) for a in arrs], tuple(tdt)

    def steps_modified(self, n: int, first: int = 0) -> int:
        return self.L.ref1d_steps_modified(self.h_, n, first)

    def init_dual(self, dt: float, t0: float = 0.0):
        self.L.ref1d_init_dual(self.h_, dt, t0)

    def get_dual(self):
        """(p, v) on the primary grid as [K, m+1] arrays, and (t, dt)"""
        n1 = self.m + 1
        p, v, tdt = np.zeros(self.K * n1), np.zeros(self.K * n1), np.zeros(2)
        self.L.ref1d_get_dual(self.h_, _ptr(p), _ptr(v), _ptr(tdt))
        return (p.reshape(self.K, n1), v.reshape(self.K, n1)), tuple(tdt)

    def steps_dual(self, n: int, first: int = 0) -> int:
        return self.L.ref1d_steps_dual(self.h_, n, first)


def ref_dt_nominal(dim: int, cfl: float, h: float, c_max: float) -> float:
    return ref_lib().ref_dt_nominal(dim, cfl, h, c_max)


def ref_step_count(T: float, dt: float) -> int:
    return ref_lib().ref_step_count(T, dt)


def ref_convergence_rate(hs, es) -> float:
    hs = np.ascontiguousarray(hs, dtype=np.float64)
    es = np.ascontiguousarray(es, dtype=np.float64)
    return ref_lib().ref_convergence_rate(len(hs), _ptr(hs), _ptr(es))


# ---------------------------------------------------------------- restatement


def oracle_M(m: int) -> np.ndarray:
    n = 2 * m + 2
    M = np.zeros(n * n)
    orc_lib().orc_get_M(m, _ptr(M))
    return M.reshape(n, n)


def add_separable(d, N, x0, h, offset, length, amp, w, phase, out):
    """out[node][coef] += amp * prod_ax sin_jet(w_ax, phase_ax) (x-major)."""
    Na = (C.c_int * 3)(*(list(N) + [1] * (3 - len(N))))
    x0a = np.array(list(x0) + [0.0] * (3 - len(x0)), dtype=np.float64)
    wa = np.array(list(w) + [0.0] * (3 - len(w)), dtype=np.float64)
    pa = np.array(list(phase) + [0.0] * (3 - len(phase)), dtype=np.float64)
    orc_lib().orc_add_separable(d, Na, _ptr(x0a), h, offset, length, amp, _ptr(wa), _ptr(pa), _ptr(out))


class OracleStepper:
    """d-dimensional Hermite-leapfrog restatement (oracle/hlf_oracle.cpp).

    Fields: 0 = p on the primary grid, 1..d = velocity components on the dual
    grid.  Host layout [node][coef], both x-major."""

    def __init__(self, d, m, K, h, boundary=None, ap=-1.0, av=-1.0, threads=None, fma=False):
        self.L = orc_lib(fma)
        self.d, self.m = d, m
        K = list(K) if hasattr(K, "__len__") else [K] * d
        boundary = list(boundary) if boundary is not None else [0] * d
        Ka = (C.c_int * 3)(*(K + [1] * (3 - d)))
        Ba = (C.c_int * 3)(*(boundary + [0] * (3 - d)))
        if threads is None:
            threads = os.cpu_count() or 1
        self.h_ = self.L.orc_create(d, m, Ka, Ba, h, ap, av, threads)
        if not self.h_:
            raise ValueError("bad oracle configuration")
        self.K, self.boundary, self.h = K, boundary, h
        self.F = (m + 1) ** d
        self.E = (2 * m + 2) ** d

    def __del__(self):
        if getattr(self, "h_", None):
            self.L.orc_destroy(self.h_)
            self.h_ = None

    def num_nodes(self, grid: int) -> int:
        return int(self.L.orc_num_nodes(self.h_, grid))

    def set_field(self, f: int, a):
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        assert a.size == self.num_nodes(0 if f == 0 else 1) * self.F
        self.L.orc_set_field(self.h_, f, _ptr(a))

    def get_field(self, f: int) -> np.ndarray:
        out = np.zeros(self.num_nodes(0 if f == 0 else 1) * self.F)
        self.L.orc_get_field(self.h_, f, _ptr(out))
        return out.reshape(-1, self.F)

    def set_coeff(self, grid: int, which: int, jets):
        if jets is None:
            self.L.orc_set_coeff(self.h_, grid, which, None)
            return
        jets = np.ascontiguousarray(jets, dtype=np.float64).ravel()
        assert jets.size == self.num_nodes(grid) * self.E
        self.L.orc_set_coeff(self.h_, grid, which, _ptr(jets))

    def set_forcing(self, grid: int, table):
        """forcing levels z(r) for the half steps updating `grid`:
        [nodes, 2m+1, n^d] (hlf_set_forcing's table); None clears"""
        if table is None:
            self.L.orc_set_forcing(self.h_, grid, None)
            return
        table = np.ascontiguousarray(table, dtype=np.float64).ravel()
        assert table.size == self.num_nodes(grid) * (2 * self.m + 1) * self.E
        self.L.orc_set_forcing(self.h_, grid, _ptr(table))

    def set_M(self, M):
        M = np.ascontiguousarray(M, dtype=np.float64).ravel()
        self.L.orc_set_M(self.h_, _ptr(M))

    def set_times(self, t_p, t_v, dt):
        self.L.orc_set_times(self.h_, t_p, t_v, dt)

    def get_times(self):
        t = np.zeros(3)
        self.L.orc_get_times(self.h_, _ptr(t))
        return tuple(float(x) for x in t)

    def advance_p(self):
        self.L.orc_advance_p(self.h_)

    def advance_v(self):
        self.L.orc_advance_v(self.h_)

    def advance_n(self, n: int, first: int = 0) -> int:
        return self.L.orc_advance_n(self.h_, n, first)

    # z-slab mode (tests of the multi-GPU halo logic on CPU)
    def set_slab(self, on: bool = True):
        self.L.orc_set_slab(self.h_, int(on))

    def layer_size(self, field: int) -> int:
        nx, ny = (self.num_nodes(0) if field == 0 else self.num_nodes(1)), 1
        K = self.K
        if field == 0:
            Np = [k + 1 if b == 1 else k for k, b in zip(K, self.boundary)]
            return Np[0] * Np[1] * self.F
        return K[0] * K[1] * self.F

    def get_layer(self, field: int, z: int) -> np.ndarray:
        out = np.zeros(self.layer_size(field))
        self.L.orc_get_layer(self.h_, field, z, _ptr(out))
        return out

    def set_halo(self, kind: int, comp: int, data):
        a = np.ascontiguousarray(data, dtype=np.float64).ravel()
        self.L.orc_set_halo(self.h_, kind, comp, _ptr(a))

    def reconstruct(self, corners) -> np.ndarray:
        c = np.ascontiguousarray(corners, dtype=np.float64).ravel()
        out = np.zeros(self.E)
        self.L.orc_reconstruct(self.h_, _ptr(c), _ptr(out))
        return out
