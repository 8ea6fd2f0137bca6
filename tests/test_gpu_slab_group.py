"""The C++ host's multi-GPU z-slab path (hlf_slabs_*, csrc/hlf_slabs.cu) on
one GPU: n slabs of one periodic box exchange their halos every half step
(peer copies between slabs sharing device 0; NCCL self send/recv for one
slab) overlapped with the interior layers, and the gathered state must equal
one solver over the whole box bit for bit.  n = 3 and 4
make the ring's previous and next slab distinct, so a swapped direction
cannot pass."""
import numpy as np
import pytest

import paper_1808_10481_b200 as H
from paper_1808_10481_b200.distributed import TRANSPORT_AUTO, TRANSPORT_COPY, TRANSPORT_NCCL, SlabGroup

pytestmark = pytest.mark.gpu

M_ORDER = 3
K = [64, 4, 12]


def state(seed=3):
    rng = np.random.default_rng(seed)
    F = (M_ORDER + 1) ** 3
    n = K[0] * K[1] * K[2]
    return [rng.standard_normal((n, F)) * 0.6 ** np.arange(F) for _ in range(4)]


def slab(a, z0, kz):
    F = a.shape[1]
    return np.ascontiguousarray(a.reshape(K[0], K[1], K[2], F)[:, :, z0:z0 + kz, :].reshape(-1, F))


def reference(steps, dt):
    h = 2.0 / K[0]
    full = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), M_ORDER)
    st = state()
    for f in range(4):
        full.set_field(f, st[f])
    full.set_times(0.0, dt / 2, dt)
    full.advance_n(steps)
    return full


@pytest.mark.parametrize("n,transport", [(2, TRANSPORT_COPY), (3, TRANSPORT_COPY), (4, TRANSPORT_COPY),
                                         (1, TRANSPORT_NCCL), (3, TRANSPORT_AUTO)])
def test_slab_group_matches_one_domain(n, transport):
    h = 2.0 / K[0]
    dt = 0.25 * h
    steps = 4
    g = SlabGroup(tuple(K), h, M_ORDER, [0] * n, transport=transport)
    assert g.transport == (TRANSPORT_COPY if transport == TRANSPORT_AUTO else transport)
    st = state()
    kz = K[2] // n
    for r in range(n):
        for f in range(4):
            g.set_field(r, f, slab(st[f], r * kz, kz))
    g.set_times(0.0, dt / 2, dt)
    g.advance_n(steps)
    full = reference(steps, dt)
    for r in range(n):
        assert g.times(r) == full.times()
    for f in range(4):
        ref = full.get_field(f)
        for r in range(n):
            assert np.array_equal(g.get_field(r, f), slab(ref, r * kz, kz)), (f, r)


def test_slab_group_rejects_bad_splits():
    with pytest.raises(H.ConfigError):
        SlabGroup((64, 4, 12), 2.0 / 64, 3, [0] * 5)  # 12 layers do not split into 5
    with pytest.raises(H.ConfigError):
        SlabGroup((64, 4, 12), 2.0 / 64, 3, [0, 0], transport=TRANSPORT_NCCL)  # NCCL: one device per slab


def test_eight_slabs_match_one_domain():
    """The 8-GPU decomposition of BASELINE.json config 5 (8 z slabs, a
    periodic ring of halo exchanges), all slabs on one GPU with peer copies:
    bit-exact against one domain over 4 steps (K_z = 16: 2 layers per slab, so
    every layer is a halo layer for a neighbour)."""
    global K
    saved = K
    K = [64, 4, 16]
    try:
        n = 8
        h = 2.0 / K[0]
        dt = 0.25 * h
        g = SlabGroup(tuple(K), h, M_ORDER, [0] * n, transport=TRANSPORT_COPY)
        st = state()
        kz = K[2] // n
        for r in range(n):
            for f in range(4):
                g.set_field(r, f, slab(st[f], r * kz, kz))
        g.set_times(0.0, dt / 2, dt)
        g.advance_n(4)
        full = reference(4, dt)
        for f in range(4):
            ref = full.get_field(f)
            for r in range(n):
                assert np.array_equal(g.get_field(r, f), slab(ref, r * kz, kz)), (f, r)
    finally:
        K = saved
