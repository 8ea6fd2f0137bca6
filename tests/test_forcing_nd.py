"""The d-dimensional forcing term on the CPU side: the manufactured forced
waves of tests/forcing_waves.py (the reference's variable_speed_problem,
problems.cpp:37-61, generalised to 2D / 3D) through the oracle's restatement
of ck_recurrence_variable with z (stepper1d.cpp:22-38) must converge at the
scheme's order; the device runs the same tables in tests/test_gpu_forcing_nd.py."""
import math

import numpy as np
import pytest

import oracle as O
from forcing_waves import ForcedWave, jets, run


def test_wave_algebra_matches_closed_forms():
    w = ForcedWave(2)
    X = w.nodes(5, 0.4, True, 2)
    t = 0.3
    th = X.sum(1) - t
    c2 = 1 + 0.5 * np.sin(X[:, 0]) * np.sin(X[:, 1])
    assert np.allclose(jets(w.u, X, t, 0, 0.4, 6)[:, 0], np.sin(th))
    assert np.allclose(jets(w.z, X, t, 0, 0.4, 6)[:, 0], np.cos(th) * (2 * c2 - 1))
    # d/dt of z and the scaled x-derivative entry (h / 1!) dz/dx
    dzdt = np.sin(th) * (2 * c2 - 1)
    assert np.allclose(jets(w.z, X, t, 1, 0.4, 6)[:, 0], dzdt)
    dzdx = -np.sin(th) * (2 * c2 - 1) + np.cos(th) * np.cos(X[:, 0]) * np.sin(X[:, 1])
    assert np.allclose(jets(w.z, X, t, 0, 0.4, 6)[:, 6], 0.4 * dzdx)  # entry [1][0], x-major
    assert np.allclose(jets(w.ap, X, 0.0, 0, 0.4, 6)[:, 0], -c2)


@pytest.mark.parametrize("m,Ks,rmin", [(2, [8, 16, 32], 4.5), (3, [8, 16], 7.0)])
def test_oracle_forced_wave_converges_2d(m, Ks, rmin):
    w = ForcedWave(2)
    errs = [run(O.OracleStepper(2, m, [K] * 2, 2 * math.pi / K), w, K, m, 1.0, 0.9, True) for K in Ks]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(rates) >= rmin, (errs, rates)
