"""Host-side mirror of the reference's solver interface (proj/include/hlf) over
the C-ABI of lib/libhlf_b200.so.

Names, argument meaning and error behaviour follow the reference:
  ConfigError / InstabilityError(step)         config.hpp:15-24
  SchemeConfig.validate / dt_nominal_1d/_2d    config.hpp:30-44, config.cpp:27-32
  step_count(T, dt)                            config.cpp:34-38
  Grid1d.over / Grid2d.over                    grid.hpp:7-39, grid.cpp:9-33
  build_interp_operator(m) -> InterpOperator   interpolation.hpp:14-22
  Stepper.advance_p / advance_v / step_system  stepper1d.hpp:72-74
The staggered state lives on the device inside the Stepper (the reference's
caller-owned State1d, stepper1d.hpp:49-52, becomes set_field/get_field plus the
t_p/t_v/dt properties).  Every compute call runs the sm_100a kernels; nothing
here computes a half step on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as _L

PERIODIC = 0
REFLECTIVE = 1
PRIMARY = 0
DUAL = 1


class ConfigError(RuntimeError):
    """hlf::ConfigError (config.hpp:15-17)."""


class InstabilityError(RuntimeError):
    """hlf::InstabilityError (config.hpp:19-24): carries the step index."""

    def __init__(self, step: int, what: str):
        super().__init__(what)
        self.step = step


class CudaError(RuntimeError):
    pass


def _check(status: int, handle=None):
    if status == _L.HLF_OK:
        return
    msg = _L.lib().hlf_last_error(handle)
    msg = msg.decode() if msg else ""
    if status == _L.HLF_CONFIG_ERROR:
        raise ConfigError(msg)
    if status == _L.HLF_INSTABILITY:
        step = int(msg.rsplit(" ", 1)[-1]) if msg else -1
        raise InstabilityError(step, msg)
    if status == _L.HLF_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise CudaError(msg or f"status {status}")


# ---------------------------------------------------------------- config


def step_count(T: float, dt_nominal: float) -> int:
    """n = ceil(T / dt_nominal) (config.cpp:34-38)."""
    if not T > 0.0:
        raise ConfigError("final time must be positive")
    if not dt_nominal > 0.0:
        raise ConfigError("nominal dt must be positive")
    return int(math.ceil(T / dt_nominal))


def plan_steps(T: float, dt_nominal: float):
    """(n, dt) of the reference's caller rule: n = step_count(T, dt_nominal),
    dt = T / n (config.cpp:34-38, tests/test_stepper1d.cpp:33-35), computed by
    the C-ABI (hlf_plan_steps)."""
    n = C.c_int(0)
    dt = C.c_double(0.0)
    _check(_L.lib().hlf_plan_steps(T, dt_nominal, C.byref(n), C.byref(dt)), None)
    return n.value, dt.value


# time schemes (hlf::Variant, config.hpp:9; hlf_b200.h HLF_SCHEME_*)
SCHEME_LEAPFROG, SCHEME_MODIFIED, SCHEME_DUAL_HERMITE, SCHEME_MODIFIED_ADVECTION = 0, 1, 2, 3


@dataclass
class SchemeConfig:
    """hlf::SchemeConfig (config.hpp:30-44); dt_nominal_3d extends the 2D rule
    with 1/sqrt(3)."""

    m: int = 2
    cfl: float = 0.9
    m_cap: int = 8

    def validate(self):
        if self.m < 0 or self.m > self.m_cap:
            raise ConfigError(f"scheme order m must be in [0, {self.m_cap}]")
        if not (self.cfl > 0.0) or not math.isfinite(self.cfl):
            raise ConfigError("cfl must be positive and finite")

    def dt_nominal_1d(self, h: float, c_max: float) -> float:
        return self.cfl * h / c_max

    def dt_nominal_2d(self, h: float, c_max: float) -> float:
        return self.cfl * h / math.sqrt(2.0) / c_max

    def dt_nominal_3d(self, h: float, c_max: float) -> float:
        return self.cfl * h / math.sqrt(3.0) / c_max

    def dt_nominal(self, dim: int, h: float, c_max: float) -> float:
        return (self.dt_nominal_1d, self.dt_nominal_2d, self.dt_nominal_3d)[dim - 1](h, c_max)


@dataclass
class Grid:
    """Uniform grid with a common spacing (Grid1d/Grid2d, grid.hpp:7-39)."""

    x_min: tuple
    h: float
    K: tuple

    @property
    def dim(self) -> int:
        return len(self.K)

    @staticmethod
    def over(lo: Sequence[float], hi: Sequence[float], K) -> "Grid":
        lo = list(lo)
        hi = list(hi)
        Ks = list(K) if hasattr(K, "__len__") else [K] * len(lo)
        for k in Ks:
            if k < 2:
                raise ConfigError("grid needs K >= 2")
        hs = []
        for a, b, k in zip(lo, hi, Ks):
            if not b > a:
                raise ConfigError("grid needs a nonempty box")
            hs.append((b - a) / k)
        for x in hs[1:]:
            if abs(x - hs[0]) > 1e-12 * abs(hs[0]):
                raise ConfigError("grid must be square (equal spacing in x and y)")
        return Grid(tuple(lo), hs[0], tuple(Ks))

    def primary(self, ax: int, i: int) -> float:
        return self.x_min[ax] + i * self.h

    def dual(self, ax: int, i: int) -> float:
        return self.x_min[ax] + (i + 0.5) * self.h


class Grid1d(Grid):
    @staticmethod
    def over(x_min: float, x_max: float, K: int) -> Grid:  # grid.cpp:9-17
        return Grid.over([x_min], [x_max], [K])


class Grid2d(Grid):
    @staticmethod
    def over(x_min, x_max, y_min, y_max, K: int) -> Grid:  # grid.cpp:19-33
        return Grid.over([x_min, y_min], [x_max, y_max], [K, K])


class Grid3d(Grid):
    @staticmethod
    def over(x_min, x_max, y_min, y_max, z_min, z_max, K) -> Grid:
        return Grid.over([x_min, y_min, z_min], [x_max, y_max, z_max], K)


@dataclass
class InterpOperator:
    """hlf::InterpOperator (interpolation.hpp:14-19)."""

    m: int
    n: int
    M: np.ndarray = field(repr=False)
    condition: float = 0.0


def build_interp_operator(m: int) -> InterpOperator:
    n = 2 * m + 2
    M = np.zeros(n * n if 0 <= m <= 8 else 1)
    cond = C.c_double(0.0)
    _check(_L.lib().hlf_build_interp_operator(m, M.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cond)))
    return InterpOperator(m, n, M.reshape(n, n), cond.value)


# ---------------------------------------------------------------- stepper


class Stepper:
    """Hermite-leapfrog stepper on the B200 for d = 1, 2, 3.

    Fields: 0 = p (primary grid), 1..d = velocity components (dual grid).
    Host arrays are [node][coef], both x-major (see include/hlf_b200.h)."""

    def __init__(self, grid: Grid, m: int, boundary=None, ap: float = -1.0, av: float = -1.0,
                 variable_ap: bool = False, M: np.ndarray | None = None, device: int = 0,
                 stream: int | None = None, z_slab: bool = False, scheme: int = 0):
        SchemeConfig(m=m).validate()  # Stepper1d ctor guard (stepper1d.cpp:95-98)
        L = _L.lib()
        d = grid.dim
        boundary = list(boundary) if boundary is not None else [PERIODIC] * d
        desc = _L.HlfDesc()
        desc.dim = d
        desc.m = m
        for ax in range(3):
            desc.K[ax] = grid.K[ax] if ax < d else 1
            desc.x_min[ax] = grid.x_min[ax] if ax < d else 0.0
            desc.boundary[ax] = boundary[ax] if ax < d else PERIODIC
        desc.h = grid.h
        desc.ap = ap
        desc.av = av
        desc.variable_ap = int(variable_ap)
        self.op = build_interp_operator(m)
        self._M = np.ascontiguousarray(M if M is not None else self.op.M, dtype=np.float64).ravel()
        desc.M = self._M.ctypes.data_as(C.POINTER(C.c_double))
        desc.device = device
        desc.stream = stream
        desc.z_slab = int(z_slab)
        desc.scheme = int(scheme)
        h = C.c_void_p()
        _check(L.hlf_create(C.byref(desc), C.byref(h)), None)
        self._h = h
        self._L = L
        self.grid, self.m, self.dim = grid, m, d
        self.scheme = int(scheme)
        self.boundary = boundary
        self.ap, self.av = ap, av
        self.n1, self.n = m + 1, 2 * m + 2
        self.F = self.n1 ** d
        self.E = self.n ** d
        self.device = device

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._L.hlf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, status):
        _check(status, self._h)

    # -- geometry
    def num_nodes(self, grid: int) -> int:
        return int(self._L.hlf_num_nodes(self._h, grid))

    def field_nodes(self, f: int) -> int:
        # leapfrog: p primary, v dual; modified / dual-Hermite: even fields primary
        primary = f == 0 if self.scheme == SCHEME_LEAPFROG else f % 2 == 0
        return self.num_nodes(PRIMARY if primary else DUAL)

    def node_shape(self, f: int) -> tuple:
        K = self.grid.K
        if f == 0:
            return tuple(k + 1 if b == REFLECTIVE else k for k, b in zip(K, self.boundary))
        return tuple(K)

    # -- state
    def set_field(self, f: int, host: np.ndarray):
        a = np.ascontiguousarray(host, dtype=np.float64)
        if a.size != self.field_nodes(f) * self.F:
            raise ValueError("field buffer has the wrong size")
        self._c(self._L.hlf_set_field(self._h, f, a.ctypes.data))

    def set_field_ptr(self, f: int, host_ptr: int):
        """Upload from a host pointer (e.g. pinned torch memory) of the right size."""
        self._c(self._L.hlf_set_field(self._h, f, host_ptr))

    def get_field(self, f: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.field_nodes(f), self.F), dtype=np.float64)
        self._c(self._L.hlf_get_field(self._h, f, out.ctypes.data))
        return out

    def get_field_ptr(self, f: int, host_ptr: int):
        self._c(self._L.hlf_get_field(self._h, f, host_ptr))

    def set_coeff(self, grid: int, jets: np.ndarray):
        a = np.ascontiguousarray(jets, dtype=np.float64)
        if a.size != self.num_nodes(grid) * self.E:
            raise ValueError("coefficient buffer has the wrong size")
        self._c(self._L.hlf_set_coeff(self._h, grid, a.ctypes.data))

    def set_coeff_separable(self, c0: float, c1: float, w: Sequence[float], phase: Sequence[float]):
        """ap = -(c0 + c1 prod sin(w x + phase)) on both grids
        (hlf_set_coeff_separable; generated in-kernel in 3D for m <= 3)."""
        w3 = (C.c_double * 3)(*(list(w) + [0.0] * (3 - len(w))))
        p3 = (C.c_double * 3)(*(list(phase) + [0.0] * (3 - len(phase))))
        self._c(self._L.hlf_set_coeff_separable(self._h, c0, c1, w3, p3))

    def set_forcing(self, grid: int, table: np.ndarray):
        """forcing jets z_r (r = 0..2m, each an n^d tensor jet, x-major) at
        every node of `grid` for the next half step updating that grid
        (hlf_set_forcing: PRIMARY -> advance_p at t_v, DUAL -> advance_v at
        t_p): [nodes, 2m+1, n^d].  d > 1 runs the faithful generic kernel."""
        a = np.ascontiguousarray(table, dtype=np.float64)
        if a.size != self.num_nodes(grid) * (self.n - 1) * self.E:
            raise ValueError("forcing table has the wrong size")
        self._c(self._L.hlf_set_forcing(self._h, grid, a.ctypes.data))

    def set_graph_steps(self, steps: int):
        """advance_n replays runs of `steps` steps as one CUDA graph (0: off)"""
        self._c(self._L.hlf_set_graph_steps(self._h, steps))

    def clear_forcing(self):
        self._c(self._L.hlf_clear_forcing(self._h))

    def set_times(self, t_p: float, t_v: float, dt: float):
        self._c(self._L.hlf_set_times(self._h, t_p, t_v, dt))

    def times(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._c(self._L.hlf_get_times(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def t_p(self):
        return self.times()[0]

    @property
    def t_v(self):
        return self.times()[1]

    @property
    def dt(self):
        return self.times()[2]

    @dt.setter
    def dt(self, value: float):
        self._c(self._L.hlf_set_dt(self._h, value))

    # -- stepping
    def advance_p(self):
        self._c(self._L.hlf_advance_p(self._h))

    def advance_v(self):
        self._c(self._L.hlf_advance_v(self._h))

    def advance_p_indexed(self, step_index: int):
        self._c(self._L.hlf_advance_p_indexed(self._h, step_index))

    def advance_v_indexed(self, step_index: int):
        self._c(self._L.hlf_advance_v_indexed(self._h, step_index))

    def advance_layers(self, half: int, step_index: int, z_begin: int, z_end: int):
        """Half step (0 = pressure, 1 = velocity) over target layers
        [z_begin, z_end) only, no time update (3D; z-slab overlap)."""
        self._c(self._L.hlf_advance_layers(self._h, half, step_index, z_begin, z_end))

    def commit_half(self, half: int):
        """t_p (0) or t_v (1) += dt after a half step done in layer ranges."""
        self._c(self._L.hlf_commit_half(self._h, half))

    def step_system(self, step_index: int):
        self._c(self._L.hlf_step(self._h, step_index))

    def advance_n(self, n: int, first_step: int = 0):
        self._c(self._L.hlf_advance_n(self._h, n, first_step))

    def advance_to(self, T: float, first_step: int = 0) -> int:
        """Advance from the current t_p to T in steps of the current dt, indexed
        first_step.. (hlf_advance_to): the caller loop of
        tests/test_stepper1d.cpp:33-38.  dt is fixed when the staggered state is
        initialised (init_leapfrog, stepper1d.cpp:131-145), so it must divide
        T - t_p; pick it with plan_steps(T, dt_nominal) first.  Returns the
        number of steps run; ConfigError if dt does not divide T - t_p."""
        n = C.c_int(0)
        self._c(self._L.hlf_advance_to(self._h, T, first_step, C.byref(n)))
        return n.value

    def poll_finite(self) -> int:
        bad = C.c_int(-1)
        self._c(self._L.hlf_poll_finite(self._h, C.byref(bad)))
        return bad.value

    def clear_finite(self):
        self._c(self._L.hlf_clear_finite(self._h))

    def synchronize(self):
        self._c(self._L.hlf_synchronize(self._h))

    # -- device data
    def field_device(self, f: int):
        ptr = C.c_void_p()
        layer = C.c_int64()
        coef = C.c_int64()
        layers = C.c_int()
        self._c(self._L.hlf_field_device(self._h, f, C.byref(ptr), C.byref(layer), C.byref(coef), C.byref(layers)))
        return ptr.value, layer.value, coef.value, layers.value

    def fill_separable(self, f: int, amp: float, w: Sequence[float], phase: Sequence[float]):
        w3 = (C.c_double * 3)(*(list(w) + [0.0] * (3 - len(w))))
        p3 = (C.c_double * 3)(*(list(phase) + [0.0] * (3 - len(phase))))
        self._c(self._L.hlf_fill_separable(self._h, f, amp, w3, p3))

    def error_separable(self, f: int, amp: float, w: Sequence[float], phase: Sequence[float]):
        """(rms value error, max scaled-jet error) of field f against
        amp * prod sin(w x + phase), computed on the device."""
        w3 = (C.c_double * 3)(*(list(w) + [0.0] * (3 - len(w))))
        p3 = (C.c_double * 3)(*(list(phase) + [0.0] * (3 - len(phase))))
        rms, mx = C.c_double(), C.c_double()
        self._c(self._L.hlf_error_separable(self._h, f, amp, w3, p3, C.byref(rms), C.byref(mx)))
        return rms.value, mx.value

    def l2_error_separable(self, f: int, amp: float, w: Sequence[float], phase: Sequence[float]) -> float:
        """Gauss-quadrature L2 error of field f against amp * prod sin(w x +
        phase) (l2_error_1d/2d, analysis.cpp:241-285), computed on the device."""
        w3 = (C.c_double * 3)(*(list(w) + [0.0] * (3 - len(w))))
        p3 = (C.c_double * 3)(*(list(phase) + [0.0] * (3 - len(phase))))
        out = C.c_double()
        self._c(self._L.hlf_l2_error_separable(self._h, f, amp, w3, p3, C.byref(out)))
        return out.value

    def energy_1d(self, kind: int, c: float = 1.0) -> float:
        """1D discrete energy on the device: kind 0 = conserved_q (after
        advance_p), 1 = conserved_r (after advance_v), analysis.cpp:221-239."""
        out = C.c_double()
        self._c(self._L.hlf_energy_1d(self._h, kind, c, C.byref(out)))
        return out.value

    def zero_field(self, f: int):
        self._c(self._L.hlf_zero_field(self._h, f))

    def halo_ptr(self, kind: int, comp: int, send: bool):
        ptr = C.c_void_p()
        cnt = C.c_int64()
        fn = self._L.hlf_halo_send_ptr if send else self._L.hlf_halo_recv_ptr
        self._c(fn(self._h, kind, comp, C.byref(ptr), C.byref(cnt)))
        return ptr.value, cnt.value

    def enable_path_counters(self, on: bool = True):
        """Count the CTAs of the tiled kernels and which of them took the TMA
        box loads (hlf_enable_path_counters; enabling again resets)."""
        self._c(self._L.hlf_enable_path_counters(self._h, int(on)))

    def time_launches(self, steps: int = 2, first_step: int = 0) -> dict:
        """Mean device ms of every kernel launch of the two half steps over
        `steps` leapfrog steps (hlf_time_launches; CUDA events on the solver
        stream; the steps advance the state)."""
        ms = (C.c_double * 6)()
        nl = (C.c_int * 2)()
        self._c(self._L.hlf_time_launches(self._h, steps, first_step, ms, nl))
        return {"vel": [ms[i] for i in range(nl[0])], "pre": [ms[3 + i] for i in range(nl[1])]}

    def path_counters(self) -> dict:
        a = (C.c_int64 * 6)()
        self._c(self._L.hlf_read_path_counters(self._h, a))
        out = {}
        for i, kind in enumerate(("vel", "pre")):
            out[kind] = {"ctas": a[3 * i], "tma_rows": a[3 * i + 1], "tma_targets": a[3 * i + 2]}
        return out

    @property
    def launch_count(self) -> int:
        return int(self._L.hlf_launch_count(self._h))

    @property
    def kernel_variant(self) -> int:
        return int(self._L.hlf_kernel_variant(self._h))

    @kernel_variant.setter
    def kernel_variant(self, v: int):
        self._c(self._L.hlf_set_kernel_variant(self._h, v))


def Stepper1d(grid: Grid, m: int, **kw) -> Stepper:
    return Stepper(grid, m, **kw)


def Stepper2d(grid: Grid, m: int, **kw) -> Stepper:
    return Stepper(grid, m, **kw)


def Stepper3d(grid: Grid, m: int, **kw) -> Stepper:
    return Stepper(grid, m, **kw)


class MaxwellTM2d:
    """2D Maxwell TM system of the reference's problem catalog (problem.hpp:34-37,
    maxwell_cavity_problem, problems.cpp:162-183):
        dEz/dt = dHy/dx - dHx/dy,  dHx/dt = -dEz/dy,  dHy/dt = dEz/dx,
    Ez on the primary grid, Hx / Hy on the dual grid, PEC walls by default.
    With p = Ez, v = -Hy, u = Hx it is exactly the acoustics system the
    steppers run (dp/dt = -(dv/dx + du/dy), dv/dt = -dp/dx, du/dt = -dp/dy,
    ap = av = -1), and a PEC wall (Ez = 0, normal H odd) is the reflective
    wall of the acoustic kernels (p zero on the wall line, tangential velocity
    odd).  This wrapper only maps the fields; every kernel is the acoustic one."""

    def __init__(self, grid: Grid, m: int, boundary=None, **kw):
        if grid.dim != 2:
            raise ConfigError("Maxwell TM is a 2D system")
        self.stepper = Stepper(grid, m, boundary=boundary if boundary is not None else [REFLECTIVE] * 2,
                               ap=-1.0, av=-1.0, **kw)

    def set_fields(self, Ez: np.ndarray, Hx: np.ndarray, Hy: np.ndarray):
        self.stepper.set_field(0, Ez)
        self.stepper.set_field(1, -np.asarray(Hy, dtype=np.float64))
        self.stepper.set_field(2, Hx)

    def get_fields(self):
        """(Ez, Hx, Hy) as [node][coef] jets"""
        s = self.stepper
        return s.get_field(0), s.get_field(2), -s.get_field(1)

    def __getattr__(self, name):  # stepping, times, accessors: the acoustic stepper's
        return getattr(self.stepper, name)

