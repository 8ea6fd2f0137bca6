"""z-slab domain decomposition of the 3D Hermite-leapfrog step across GPUs.

One process per GPU (torch.distributed, NCCL).  Rank r owns cells
z in [r Kz, (r+1) Kz) of a periodic domain:
  * before advance_p (pressure half step) it needs the dual v layer z = -1,
    i.e. the previous rank's last v layer  -> v halo, 3 components;
  * before advance_v (velocity half step) it needs the primary p layer z = Kz,
    i.e. the next rank's first p layer      -> p halo.
A layer of one field is contiguous in the SoA layout [layer][coef][y][x], so
each halo is one NCCL send/recv of the layer with no packing.  The halos
land directly in the solver's ghost layers (hlf_halo_recv_ptr).  The exchange
is issued on the solver's stream; with one rank the library wraps z itself.

The exchange logic only needs a backend with advance_p_indexed,
advance_v_indexed and halo views; `Stepper` (CUDA) is the product backend,
the tests drive the same logic over gloo with a CPU backend.
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import _lib as _L
from .solver import PERIODIC, ConfigError, Grid, Stepper, _check, build_interp_operator


class _DevArray:
    """__cuda_array_interface__ view of solver-owned device memory."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, count: int):
    import torch
    return torch.as_tensor(_DevArray(ptr, count), device="cuda")


class HaloExchanger:
    """Pairs the z halo sends/receives of one slab with its ring neighbours.

    `views(kind, comp, send)` returns the tensor a halo is sent from / received
    into (kind 0 = p layer, 1 = v layer of component comp).  For the CUDA
    backend the tensors alias the solver's own layers, so `pack`/`unpack` are
    no-ops; a host backend may copy in `pack(kind)` / `unpack(kind)`."""

    def __init__(self, rank: int, world: int, views, pack=None, unpack=None):
        self.rank, self.world = rank, world
        self.prev = (rank - 1) % world
        self.next = (rank + 1) % world
        self.p_send = views(0, 0, True)
        self.p_recv = views(0, 0, False)
        self.v_send = [views(1, c, True) for c in range(3)]
        self.v_recv = [views(1, c, False) for c in range(3)]
        self.pack = pack or (lambda kind: None)
        self.unpack = unpack or (lambda kind: None)

    def _p_ops(self):
        # my p layer 0 is the previous rank's layer Kz; my layer Kz comes from the next rank
        import torch.distributed as dist
        return [dist.P2POp(dist.isend, self.p_send, self.prev), dist.P2POp(dist.irecv, self.p_recv, self.next)]

    def _v_ops(self):
        # my last v layer is the next rank's ghost z = -1; my ghost comes from the previous rank
        import torch.distributed as dist
        ops = []
        for c in range(3):
            ops.append(dist.P2POp(dist.isend, self.v_send[c], self.next))
            ops.append(dist.P2POp(dist.irecv, self.v_recv[c], self.prev))
        return ops

    def start(self, kind: int):
        """Issue the halo exchange of kind 0 (p) / 1 (v) and return its
        requests.  With NCCL the transfers are ordered after the work already
        queued on the current stream and run concurrently with what is
        queued next; `finish` makes the current stream wait for them."""
        import torch.distributed as dist
        self.pack(kind)
        return dist.batch_isend_irecv(self._p_ops() if kind == 0 else self._v_ops())

    def finish(self, kind: int, reqs):
        for r in reqs:
            r.wait()
        self.unpack(kind)

    def exchange_p(self):
        self.finish(0, self.start(0))

    def exchange_v(self):
        self.finish(1, self.start(1))


def slab_step(solver, halo, step_index: int, overlap: bool = True):
    """One full leapfrog step of a slab (step_system order, stepper1d.cpp:168-172):
    v halo -> advance_p -> p halo -> advance_v.

    With `overlap` (and a backend that advances layer ranges) each halo is in
    flight while the layers that do not need it are updated: the pressure half
    step needs the v halo only for p layer 0, the velocity half step needs the
    p halo only for v layer Kz-1.  p layer 0 is final before its halo is sent."""
    if not halo:
        solver.advance_p_indexed(step_index)
        solver.advance_v_indexed(step_index)
        return
    if not (overlap and hasattr(solver, "advance_layers")):
        halo.exchange_v()
        solver.advance_p_indexed(step_index)
        halo.exchange_p()
        solver.advance_v_indexed(step_index)
        return
    kz = solver.grid.K[2]
    reqs = halo.start(1)
    solver.advance_layers(0, step_index, 1, kz)      # p interior: no v halo needed
    halo.finish(1, reqs)
    solver.advance_layers(0, step_index, 0, 1)       # p layer 0 reads the v halo
    solver.commit_half(0)
    reqs = halo.start(0)                             # sends the final p layer 0
    solver.advance_layers(1, step_index, 0, kz - 1)  # v interior: no p halo needed
    halo.finish(0, reqs)
    solver.advance_layers(1, step_index, kz - 1, kz)  # v layer Kz-1 reads the p halo
    solver.commit_half(1)


class SlabStepper:
    """3D acoustic stepper on one z-slab of a periodic box (one rank per GPU)."""

    def __init__(self, K_global, h: float, m: int, rank: int = 0, world: int = 1, device: int = 0,
                 stream=None, x_min=(-1.0, -1.0, -1.0)):
        Kx, Ky, Kz = K_global
        if Kz % world:
            raise ValueError("global z cells must divide evenly across ranks")
        self.K_global = tuple(K_global)
        self.kz = Kz // world
        self.rank, self.world = rank, world
        self.m, self.h = m, h
        self.stream = stream
        x0 = (x_min[0], x_min[1], x_min[2] + rank * self.kz * h)
        grid = Grid(x0, h, (Kx, Ky, self.kz))
        if stream is None:
            # the solver and the NCCL halos must share one stream (halo sends
            # follow the kernels that write the sent layer; kernels follow the
            # receives): give the solver a torch stream the exchange runs under
            import torch
            stream = torch.cuda.Stream(device=device)
        self.stream = stream
        sptr = stream.cuda_stream
        self.solver = Stepper(grid, m, device=device, stream=sptr, z_slab=world > 1)
        self.halo = None
        if world > 1:
            def views(kind, comp, send):
                ptr, cnt = self.solver.halo_ptr(kind, comp, send)
                return device_view(ptr, cnt)
            self.halo = HaloExchanger(rank, world, views)

    # ---- data
    def init_mode(self, cfl: float = 0.9, t0: float = 0.0):
        """Standing mode of the periodic global box, p = cos(wt t) prod_a
        sin(w_a x_a) with w_a = 2 pi / L_a (on [-1, 1]^3: sin(pi x) sin(pi y)
        sin(pi z)), and its velocity v_c = -(w_c / wt) sin(wt t) cos(w_c x_c)
        prod_{a != c} sin(w_a x_a) at t0 + dt/2 (leapfrog staggering,
        stepper1d.cpp:131-145): an exact solution on any box, exact jets on the
        device; dt = cfl h / sqrt(3)."""
        s = self.solver
        w = [2.0 * math.pi / (k * self.h) for k in self.K_global]
        wt = math.sqrt(sum(x * x for x in w))
        dt = cfl * self.h / math.sqrt(3.0)
        tv = t0 + dt / 2
        for f in range(4):
            s.zero_field(f)
        s.fill_separable(0, math.cos(wt * t0), w, [0.0] * 3)
        for c in range(3):
            ph = [math.pi / 2 if a == c else 0.0 for a in range(3)]
            s.fill_separable(1 + c, -(w[c] / wt) * math.sin(wt * tv), w, ph)
        s.set_times(t0, tv, dt)
        return dt

    # ---- stepping
    def step(self, step_index: int):
        import torch
        # NCCL orders the halo transfers after the solver stream's queued work
        with torch.cuda.stream(self.stream):
            slab_step(self.solver, self.halo, step_index)

    def launch_count(self) -> int:
        return self.solver.launch_count

    def poll_finite(self) -> int:
        return self.solver.poll_finite()

    def kernel_times(self, steps: int = 2):
        """Mean device ms of every launch of the velocity half step (1 launch at
        m = 3) and the pressure half step (2: V_x+V_y merged, V_z), from CUDA
        events the library records around each kernel on the solver stream
        (hlf_time_launches; one rank's kernels, halos not included)."""
        t = self.solver.time_launches(steps, 10_000)
        return {"vel": t["vel"], "pre": t["pre"], "vel_ms": sum(t["vel"]), "pre_ms": sum(t["pre"])}

    def e2e(self, steps: int, dof_per_step: int):
        """End to end through the C-ABI: upload the staggered state from pinned
        host memory (hlf_set_field), advance `steps` leapfrog steps
        (hlf_advance_n semantics: one finite check at the end), download it
        (hlf_get_field).  Returns the e2e JSON object."""
        import torch
        s = self.solver
        bufs = []
        for f in range(4):
            n = s.field_nodes(f) * s.F
            bufs.append(torch.empty(n, dtype=torch.float64, pin_memory=True))
        torch.cuda.synchronize()
        for f in range(4):
            s.get_field_ptr(f, bufs[f].data_ptr())  # a real state to upload
        nbytes = sum(b.numel() * 8 for b in bufs)
        t_p, t_v, dt = s.times()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in range(4):
            s.set_field_ptr(f, bufs[f].data_ptr())
        s.set_times(t_p, t_v, dt)
        for i in range(steps):
            self.step(i)
        bad = s.poll_finite()
        for f in range(4):
            s.get_field_ptr(f, bufs[f].data_ptr())
        sec = time.perf_counter() - t0
        del bufs
        return {"value": dof_per_step * steps / sec, "unit": "DOF-updates/s",
                "h2d_bytes_per_step": nbytes / steps, "d2h_bytes_per_step": nbytes / steps,
                "job": {"leapfrog_steps": steps, "h2d_bytes": nbytes, "d2h_bytes": nbytes, "seconds": sec,
                        "api": "hlf_set_field x4 (pinned host AoS) + hlf_advance_p/v_indexed x steps + "
                               "hlf_poll_finite + hlf_get_field x4, wall clock", "finite": bad < 0}}


TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_COPY = 0, 1, 2


class SlabGroup:
    """The C++ host's multi-GPU path (hlf_slabs_*, csrc/hlf_slabs.cu): one
    process drives n z-slab solvers of a periodic 3D box, slab r on
    devices[r], with the one-layer halos of every half step exchanged by NCCL
    (distinct devices) or peer copies (any devices, e.g. several slabs on one
    GPU), overlapped with the interior layers.  Host data per slab use the
    solver layout (x-major AoS [node][coef] of that slab's nodes)."""

    def __init__(self, K_global, h: float, m: int, devices, transport: int = TRANSPORT_AUTO,
                 x_min=(-1.0, -1.0, -1.0), ap: float = -1.0, av: float = -1.0):
        L = _L.lib()
        d = _L.HlfDesc()
        d.dim = 3
        d.m = m
        for a in range(3):
            d.K[a] = K_global[a]
            d.x_min[a] = x_min[a]
            d.boundary[a] = PERIODIC
        d.h = h
        d.ap, d.av = ap, av
        self._M = np.ascontiguousarray(build_interp_operator(m).M, dtype=np.float64).ravel()
        d.M = self._M.ctypes.data_as(_L._dp)
        devs = (_L.C.c_int * len(devices))(*devices)
        g = _L.C.c_void_p()
        st = L.hlf_slabs_create(_L.C.byref(d), len(devices), devs, transport, _L.C.byref(g))
        if st != _L.HLF_OK:
            msg = L.hlf_slabs_last_error(None)
            raise ConfigError((msg or b"").decode()) if st == _L.HLF_CONFIG_ERROR else RuntimeError(
                f"hlf_slabs_create: status {st}: {(msg or b'').decode()}")
        self._g, self._L = g, L
        self.n = len(devices)
        self.m, self.F = m, (m + 1) ** 3
        self.K_global = tuple(K_global)
        self.kz = K_global[2] // self.n

    def close(self):
        if getattr(self, "_g", None):
            self._L.hlf_slabs_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def transport(self) -> int:
        return int(self._L.hlf_slabs_transport(self._g))

    def _solver(self, r: int):
        return self._L.hlf_slabs_solver(self._g, r)

    def _chk(self, st):
        if st != _L.HLF_OK:
            msg = (self._L.hlf_slabs_last_error(self._g) or b"").decode()
            if st == _L.HLF_INSTABILITY:
                from .solver import InstabilityError
                raise InstabilityError(int(msg.rsplit(" ", 1)[-1]), msg)
            raise RuntimeError(f"slab group: status {st}: {msg}")

    def set_field(self, r: int, f: int, host):
        a = np.ascontiguousarray(host, dtype=np.float64)
        s = self._solver(r)
        _check(self._L.hlf_set_field(s, f, a.ctypes.data), s)

    def get_field(self, r: int, f: int):
        s = self._solver(r)
        grid = 0 if f == 0 else 1
        out = np.empty((int(self._L.hlf_num_nodes(s, grid)), self.F))
        _check(self._L.hlf_get_field(s, f, out.ctypes.data), s)
        return out

    def set_times(self, t_p, t_v, dt):
        self._chk(self._L.hlf_slabs_set_times(self._g, t_p, t_v, dt))

    def times(self, r: int = 0):
        a, b, c = _L.C.c_double(), _L.C.c_double(), _L.C.c_double()
        s = self._solver(r)
        _check(self._L.hlf_get_times(s, _L.C.byref(a), _L.C.byref(b), _L.C.byref(c)), s)
        return a.value, b.value, c.value

    def advance_n(self, steps: int, first_step: int = 0):
        self._chk(self._L.hlf_slabs_advance_n(self._g, steps, first_step))

    def synchronize(self):
        self._chk(self._L.hlf_slabs_synchronize(self._g))
