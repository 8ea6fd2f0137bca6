"""The z-slab decomposition (paper_1808_10481_b200/distributed.py) on CPU:
world_size 2, 3, 4 and 8 over gloo (3 and 4 make prev != next, so a swapped
send / receive direction cannot pass), each rank stepping its slab with the oracle (as the
compute backend) through the product's HaloExchanger / slab_step logic; the
gathered result must equal a single-domain run bit for bit (SURVEY.md
sec. 8(e)).  The GPU path uses the same exchange code with NCCL and the
solver's own halo layers."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1808_10481_b200.distributed import HaloExchanger, slab_step

M_ORDER = 2
K = [6, 5, 24]  # z divisible by 2, 3, 4 and 8


def full_state(seed=11):
    rng = np.random.default_rng(seed)
    F = (M_ORDER + 1) ** 3
    n = K[0] * K[1] * K[2]
    return [rng.standard_normal((n, F)) * 0.6 ** np.arange(F) for _ in range(4)]


def slab_of(a, z0, kz):
    F = a.shape[1]
    return a.reshape(K[0], K[1], K[2], F)[:, :, z0:z0 + kz, :].reshape(-1, F)


class OracleSlab:
    """CPU backend with the solver's slab interface (advance_*_indexed + halos)."""

    def __init__(self, rank, world, h):
        self.kz = K[2] // world
        self.o = O.OracleStepper(3, M_ORDER, [K[0], K[1], self.kz], h, threads=1)
        self.o.set_slab(True)
        F = (M_ORDER + 1) ** 3
        plane = K[0] * K[1] * F
        self.send = {(0, 0): torch.zeros(plane, dtype=torch.float64)}
        self.recv = {(0, 0): torch.zeros(plane, dtype=torch.float64)}
        for c in range(3):
            self.send[(1, c)] = torch.zeros(plane, dtype=torch.float64)
            self.recv[(1, c)] = torch.zeros(plane, dtype=torch.float64)

    def views(self, kind, comp, send):
        return (self.send if send else self.recv)[(kind, comp)]

    def pack(self, kind):
        if kind == 0:
            self.send[(0, 0)].copy_(torch.from_numpy(self.o.get_layer(0, 0)))
        else:
            for c in range(3):
                self.send[(1, c)].copy_(torch.from_numpy(self.o.get_layer(1 + c, self.kz - 1)))

    def unpack(self, kind):
        if kind == 0:
            self.o.set_halo(0, 0, self.recv[(0, 0)].numpy())
        else:
            for c in range(3):
                self.o.set_halo(1, c, self.recv[(1, c)].numpy())

    def advance_p_indexed(self, i):
        self.o.advance_p()

    def advance_v_indexed(self, i):
        self.o.advance_v()


def _worker(rank, world, port, steps, out_q, swap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = 2.0 / K[0]
    be = OracleSlab(rank, world, h)
    kz = be.kz
    state = full_state()
    for f in range(4):
        be.o.set_field(f, slab_of(state[f], rank * kz, kz))
    dt = 0.2 * h
    be.o.set_times(0.0, dt / 2, dt)
    halo = HaloExchanger(rank, world, be.views, be.pack, be.unpack)
    if swap:  # deliberately wrong ring direction (test sensitivity)
        halo.prev, halo.next = halo.next, halo.prev
    for i in range(steps):
        slab_step(be, halo, i)
    out_q.put((rank, [be.o.get_field(f) for f in range(4)]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_slabs(world, steps, swap=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, q, swap)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def single_domain(steps):
    h = 2.0 / K[0]
    o = O.OracleStepper(3, M_ORDER, K, h, threads=1)
    state = full_state()
    for f in range(4):
        o.set_field(f, state[f])
    dt = 0.2 * h
    o.set_times(0.0, dt / 2, dt)
    assert o.advance_n(steps) == -1
    return [o.get_field(f) for f in range(4)]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_slab_decomposition_matches_single_domain(world):
    steps = 3
    results = run_slabs(world, steps)
    ref = single_domain(steps)
    kz = K[2] // world
    for f in range(4):
        for r in range(world):
            got = results[r][f]
            assert np.array_equal(got, slab_of(ref[f], r * kz, kz)), (f, r)


def test_swapped_ring_direction_is_detected():
    # with three ranks prev != next: exchanging with the wrong neighbour must
    # change the result (the world = 2 test alone could not tell)
    steps = 2
    results = run_slabs(3, steps, swap=True)
    ref = single_domain(steps)
    kz = K[2] // 3
    assert any(not np.array_equal(results[r][f], slab_of(ref[f], r * kz, kz)) for f in range(4) for r in range(3))
