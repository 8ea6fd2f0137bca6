"""Manufactured forced problems in 2D / 3D for the forcing path (test helper).

The reference's variable-speed problem (problems.cpp:37-61: c^2 = 1 + sin(x)/2,
p = v = sin(x - t), forcing z chosen so the pair solves p_t = ap v_x + z,
v_t = av p_x) generalised to d dimensions on the periodic box [0, 2 pi]^d:

  c^2 = 1 + s_d prod_a sin(x_a)   (s_2 = 1/2, s_3 = 1/2)
  p = v_a = sin(theta),  theta = sum_a x_a - t
  p_t = -c^2 div v + z   =>   z = cos(theta) (d c^2 - 1)

Every function is kept as a finite sum of complex exponentials
c e^{i (k.x + w t)}, so products, time derivatives and the reference's scaled
jets (h^q / q! d^q, jet.hpp:7-9; sin_jet, jet.cpp:65-74) are exact closed forms.
forcing_table(...)[node][r][e] is ForcingAt's z(r) (stepper1d.cpp:113-119) as a
tensor jet: the table hlf_set_forcing takes."""
import math

import numpy as np


def expo_sin(k, w=0.0, ph=0.0):
    """sin(k.x + w t + ph) as exponential terms [(c, k, w)]"""
    k = np.asarray(k, dtype=float)
    a = np.exp(1j * ph) / 2j
    return [(a, k, w), (np.conj(a), -k, -w)]  # real sum: the second term is the conjugate


def expo_cos(k, w=0.0, ph=0.0):
    k = np.asarray(k, dtype=float)
    a = np.exp(1j * ph) / 2
    return [(a, k, w), (np.conj(a), -k, -w)]


def const(c, d):
    return [(complex(c), np.zeros(d), 0.0)]


def mul(A, B):
    return [(ca * cb, ka + kb, wa + wb) for ca, ka, wa in A for cb, kb, wb in B]


def add(*terms):
    out = []
    for t in terms:
        out += t
    return out


def scale(A, s):
    return [(c * s, k, w) for c, k, w in A]


def jets(terms, X, t, r, h, n):
    """scaled n^d tensor jets (x-major) of d^r/dt^r of the real sum at the
    points X [N, d] and time t: [N, n^d]"""
    N, d = X.shape
    q = np.arange(n)
    fact = np.array([math.factorial(i) for i in range(n)], dtype=float)
    out = np.zeros((N,) + (n,) * d, dtype=complex)
    for c, k, w in terms:
        base = c * (1j * w) ** r * np.exp(1j * (X @ k + w * t))  # [N]
        J = base.reshape((N,) + (1,) * d)
        for a in range(d):
            fa = (1j * k[a] * h) ** q / fact  # [n]
            shape = [1] * (d + 1)
            shape[a + 1] = n
            J = J * fa.reshape(shape)
        out += J
    return out.real.reshape(N, n ** d)


class ForcedWave:
    """p = v_a = sin(sum x - t) with c^2 = 1 + 0.5 prod sin(x_a) on [0, 2 pi]^d"""

    def __init__(self, d):
        self.d = d
        ones = np.ones(d)
        sprod = const(1.0, d)
        for a in range(d):
            e = np.zeros(d)
            e[a] = 1.0
            sprod = mul(sprod, expo_sin(e))
        self.c2 = add(const(1.0, d), scale(sprod, 0.5))
        self.ap = scale(self.c2, -1.0)
        self.u = expo_sin(ones, -1.0)  # p and every v_a
        # z = cos(theta) (d c^2 - 1)
        self.z = mul(expo_cos(ones, -1.0), add(scale(self.c2, float(d)), const(-1.0, d)))
        self.c_max = math.sqrt(1.5)

    @staticmethod
    def nodes(K, h, dual, d):
        """node coordinates, x-major ([ix][iy][iz]), periodic box from 0"""
        off = 0.5 * h if dual else 0.0
        axes = [off + h * np.arange(K) for _ in range(d)]
        G = np.meshgrid(*axes, indexing="ij")
        return np.stack([g.ravel() for g in G], axis=1)

    def field(self, X, t, h, m):
        """[N, (m+1)^d] jets of the exact solution (the node's stored jet)"""
        n1, d = m + 1, self.d
        n = 2 * m + 2
        J = jets(self.u, X, t, 0, h, n).reshape((-1,) + (n,) * d)
        return J[(slice(None),) + (slice(0, n1),) * d].reshape(len(X), n1 ** d)

    def coeff(self, X, h, m):
        return jets(self.ap, X, 0.0, 0, h, 2 * m + 2)

    def forcing_table(self, X, t, h, m):
        n = 2 * m + 2
        return np.stack([jets(self.z, X, t, r, h, n) for r in range(n - 1)], axis=1)


def run(s, wave, K, m, T, cfl, oracle):
    """advance solver `s` (device Stepper or OracleStepper) over [0, T] with the
    forcing tables set before every half step (advance_p at (primary, t_v),
    advance_v at (dual, t_p)); returns the max-norm error of p's jets at T
    relative to the exact jets' max"""
    d = wave.d
    h = 2 * math.pi / K
    Xp, Xd = wave.nodes(K, h, False, d), wave.nodes(K, h, True, d)
    n = math.ceil(T / (cfl * h / (wave.c_max * math.sqrt(d))))
    dt = T / n
    s.set_field(0, wave.field(Xp, 0.0, h, m))
    for a in range(d):
        s.set_field(1 + a, wave.field(Xd, dt / 2, h, m))
    for grid, X in ((0, Xp), (1, Xd)):
        if oracle:
            s.set_coeff(grid, 0, wave.coeff(X, h, m))
        else:
            s.set_coeff(grid, wave.coeff(X, h, m))
    s.set_times(0.0, dt / 2, dt)
    times = s.get_times if oracle else s.times
    for _ in range(n):
        s.set_forcing(0, wave.forcing_table(Xp, times()[1], h, m))
        s.advance_p()
        s.set_forcing(1, wave.forcing_table(Xd, times()[0], h, m))
        s.advance_v()
    exact = wave.field(Xp, times()[0], h, m)
    return np.abs(s.get_field(0) - exact).max() / np.abs(exact).max()
