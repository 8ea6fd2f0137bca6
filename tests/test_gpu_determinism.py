"""Race evidence without a sanitizer (compute-sanitizer is closed on this GPU
pool, profiles/r2/sanitize_racecheck_unavailable.log).  The tiled kernels'
correctness rests on barrier / mbarrier ordering (TMA boxes completing on
mbarriers, a lane-private target stage, cross-proxy fences before a stage is
refilled); a missing ordering shows up as run-to-run differences or as a
difference between the loader paths.  So: the bench-shaped TMA path is run
repeatedly and must be bitwise reproducible, and it must equal bit for bit the
per-node cp.async loaders (HLF_NO_TMA / HLF_NO_TMA_T: same arithmetic,
different data movement and synchronisation)."""
import os

import numpy as np
import pytest

import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu


def run(d, m, K, boundary, steps, env=None):
    old = {k: os.environ.get(k) for k in ("HLF_NO_TMA", "HLF_NO_TMA_T")}
    try:
        for k in old:
            os.environ.pop(k, None)
        for k, v in (env or {}).items():
            os.environ[k] = v
        g = H.Stepper(H.Grid([-1.0] * d, 2.0 / K[0], tuple(K)), m, boundary=boundary)
        rng = np.random.default_rng(77)
        for f in range(d + 1):
            g.set_field(f, rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F))
        g.enable_path_counters()
        dt = 0.25 * g.grid.h
        g.set_times(0.0, dt / 2, dt)
        g.advance_n(steps)
        return [g.get_field(f) for f in range(d + 1)], g.path_counters()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("d,m,K,boundary", [(3, 3, [96, 6, 70], [0, 0, 0]), (3, 2, [96, 6, 70], [0, 1, 1]),
                                            (2, 3, [128, 96], [0, 0]), (2, 4, [128, 96], [1, 0])])
def test_tma_path_is_reproducible_and_equals_per_node_loads(d, m, K, boundary):
    ref, c = run(d, m, K, boundary, 6)
    assert c["pre"]["tma_rows"] > 0 and c["vel"]["tma_targets"] > 0
    for _ in range(4):
        again, _ = run(d, m, K, boundary, 6)
        for a, b in zip(ref, again):
            assert np.array_equal(a, b)
    plain, c2 = run(d, m, K, boundary, 6, {"HLF_NO_TMA": "1", "HLF_NO_TMA_T": "1"})
    assert c2["pre"]["tma_rows"] == 0 and c2["vel"]["tma_targets"] == 0
    for a, b in zip(ref, plain):
        assert np.array_equal(a, b)
