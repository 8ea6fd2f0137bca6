"""The product multi-GPU path with real torch.distributed point-to-point
exchanges: two, three and four ranks (processes) on one GPU over gloo (three
and four make prev != next, so a swapped ring direction cannot pass), each owning a z-slab
SlabStepper (the CUDA solver with z_slab = True) stepped by distributed.slab_step
in its overlapped order (interior layers with the halo in flight, the
boundary layer after it lands, hlf_advance_layers).  gloo needs host tensors,
so the halo views are staged through the exchanger's pack / unpack hooks; with
NCCL (bench.py --gpus N) the same code sends the solver's device layers
directly.  The gathered state must equal one periodic single-domain solver
bit for bit."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

M_ORDER = 3
K = [36, 4, 24]  # z divisible by 2, 3, 4 and 8


def _state(seed=5):
    rng = np.random.default_rng(seed)
    F = (M_ORDER + 1) ** 3
    n = K[0] * K[1] * K[2]
    return [rng.standard_normal((n, F)) * 0.6 ** np.arange(F) for _ in range(4)]


def _slab(a, z0, kz):
    F = a.shape[1]
    return np.ascontiguousarray(a.reshape(K[0], K[1], K[2], F)[:, :, z0:z0 + kz, :].reshape(-1, F))


def _worker(rank, world, port, steps, overlap, out_q):
    import torch.distributed as dist
    from paper_1808_10481_b200.distributed import HaloExchanger, SlabStepper, device_view, slab_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    h = 2.0 / K[0]
    st = SlabStepper(tuple(K), h, M_ORDER, rank=rank, world=world, device=0)
    s = st.solver
    kz = st.kz
    state = _state()
    for f in range(4):
        s.set_field(f, _slab(state[f], rank * kz, kz))
    dt = 0.25 * h
    s.set_times(0.0, dt / 2, dt)
    dev = {}
    host = {}
    for kind, comps in ((0, [0]), (1, [0, 1, 2])):
        for c in comps:
            for send in (True, False):
                ptr, cnt = s.halo_ptr(kind, c, send)
                dev[(kind, c, send)] = device_view(ptr, cnt)
                host[(kind, c, send)] = torch.zeros(cnt, dtype=torch.float64)

    def pack(kind):
        torch.cuda.synchronize()
        for (k, c, send), t in host.items():
            if k == kind and send:
                t.copy_(dev[(k, c, True)])

    def unpack(kind):
        for (k, c, send), t in host.items():
            if k == kind and not send:
                dev[(k, c, False)].copy_(t)
        torch.cuda.synchronize()

    halo = HaloExchanger(rank, world, lambda k, c, send: host[(k, c, send)], pack, unpack)
    for i in range(steps):
        slab_step(s, halo, i, overlap=overlap)
    s.synchronize()
    out_q.put((rank, [s.get_field(f) for f in range(4)], s.times()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("overlap", [True, False])
def test_ranks_on_one_gpu_match_single_domain(world, overlap):
    import paper_1808_10481_b200 as H
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, overlap, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, fields, times = q.get(timeout=600)
        results[r] = (fields, times)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    h = 2.0 / K[0]
    full = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), M_ORDER)
    state = _state()
    for f in range(4):
        full.set_field(f, state[f])
    dt = 0.25 * h
    full.set_times(0.0, dt / 2, dt)
    for i in range(steps):
        full.step_system(i)
    kz = K[2] // world
    for f in range(4):
        ref = full.get_field(f)
        for r in range(world):
            assert np.array_equal(results[r][0][f], _slab(ref, r * kz, kz)), (f, r)
    for r in range(world):
        assert results[r][1] == full.times()
