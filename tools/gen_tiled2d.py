"""Generate paper_1808_10481_b200/csrc/tiled2d_gen.cuh: stage code of the tiled
2D Hermite-leapfrog kernel (kernels_tiled2d.cu), m = 1..4.

2D pipeline (y-marching; x is the lane axis):
  X stage   task (l_y, q_x parity): half x-line between source nodes i, i+1 of
            the new source row -> ring_new[q_x][l_y][cell]
  Y + CK    warp = parity class (PX, PY): y half-lines (outputs q_y = PY mod 2)
            between ring rows j, j+1 for the class's q_x columns, then the
            closed-form odd CK sum of the leapfrog update for every target
            component, class-specialised (2D bodies are small).
Rows of M are pre-scaled by s! (P~[q] = qx! qy! P[q]), the CK coefficient of
multi-index b is GM[b] = G_|b| |b|!/b! and every output is scaled by 1/o!
(SURVEY.md App. A.3 for d = 2).
Usage: python tools/gen_tiled2d.py
"""
from __future__ import annotations

import os
from math import factorial

TXC = 32
RAWX = TXC + 2  # 33 nodes used; 34 keeps TMA rows 16 B multiples
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "paper_1808_10481_b200", "csrc", "tiled2d_gen.cuh")


def bindex2(b, mm):
    idx = 0
    for a0 in range(mm + 1):
        for a1 in range(mm + 1 - a0):
            if (a0, a1) == tuple(b):
                return idx
            idx += 1
    raise ValueError(b)


def mzero(r, l, mm):
    """M[r][l] is exactly zero for even rows r >= 2 and l = 0; the host checks
    it (hlf_capi.cu, m_mirror) and these terms are not emitted (m <= 3: from
    m = 4 on the reference's LU inverse leaves round-off there, which is kept)."""
    return mm <= 3 and l == 0 and r >= 2 and r % 2 == 0


def half_line(mm, srcL, srcR, outs, tmp, lines, ind="  ", sh=0):
    """parity-split line; sh = 1 uses row s+1 of M for output s (merged
    pressure kernel: the divergence shift moved into the sweep), rows past
    2m+1 give the literal 0.0."""
    n1, n = mm + 1, 2 * mm + 2
    need_s, need_d = set(), set()
    for s in outs:
        if s + sh >= n:
            continue
        for l in range(n1):
            if not mzero(s + sh, l, mm):
                (need_s if (s + sh + l) % 2 == 0 else need_d).add(l)
    for l in sorted(need_s):
        lines.append(f"{ind}const double {tmp}s{l} = {srcL(l)} + {srcR(l)};")
    for l in sorted(need_d):
        lines.append(f"{ind}const double {tmp}d{l} = {srcR(l)} - {srcL(l)};")
    res = {}
    for s in outs:
        r = s + sh
        if r >= n:
            res[s] = "0.0"
            continue
        expr = "0.0"
        for l in range(n1):
            if mzero(r, l, mm):
                continue
            if (r + l) % 2 == 0:
                expr = f"fma(P.ML[{r * n1 + l}], {tmp}s{l}, {expr})"
            else:
                expr = f"fma(-P.ML[{r * n1 + l}], {tmp}d{l}, {expr})"
        name = f"{tmp}o{s}"
        lines.append(f"{ind}const double {name} = {expr};")
        res[s] = name
    return res


def gen_x(mm, px, sh=0, suffix=""):
    n1, n = mm + 1, 2 * mm + 2
    L = [f"__device__ __forceinline__ void t2_m{mm}_x_px{px}{suffix}(const T2Params& P, const double* __restrict__ rb,",
         "                                             double* __restrict__ wb) {",
         "  // rb = raw + l_y*RAWX + cell (raw row layout [f = lx*n1 + ly][node]);  wb = ring_new + l_y*TXC + cell"]
    qxs = [q for q in range(n) if q % 2 == px]
    res = half_line(mm, lambda l: f"rb[{(l * n1) * RAWX}]", lambda l: f"rb[{(l * n1) * RAWX + 1}]", qxs, "x", L, sh=sh)
    for q in qxs:
        L.append(f"  wb[{(q * n1) * TXC}] = {res[q]};")
    L.append("}")
    return "\n".join(L)


def gen_class(mm, PX, PY, comps, name):
    """y half-lines for the class columns + CK for target components comps
    (component index c: 0 = x, 1 = y derivative axis)."""
    n1, n = mm + 1, 2 * mm + 2
    nh = n // 2
    L = [f"__device__ __forceinline__ void {name}(const T2Params& P, const double* __restrict__ ro,",
         "    const double* __restrict__ rn, const double* __restrict__ tg, int lane, double* const* dptr,",
         "    bool active, bool& bad) {",
         "  // ro/rn = ring + lane; tg = staged targets [t][f][cell]"]
    # P~ for the class: columns qx = PX + 2 ix, rows qy = PY + 2 iy
    for ix in range(nh):
        qx = PX + 2 * ix
        res = half_line(mm, lambda l, qx=qx: f"ro[{(qx * n1 + l) * TXC}]", lambda l, qx=qx: f"rn[{(qx * n1 + l) * TXC}]",
                        [PY + 2 * iy for iy in range(nh)], f"c{ix}_", L)
        for iy in range(nh):
            L.append(f"  const double p{ix}_{iy} = {res[PY + 2 * iy]};")
    for t, c in enumerate(comps):
        e = [int(c == a) for a in range(2)]
        for ox in range(n1):
            for oy in range(n1):
                if ((ox + e[0]) & 1) != PX or ((oy + e[1]) & 1) != PY:
                    continue
                terms = []
                for b0 in range(mm + 1):
                    for b1 in range(mm + 1 - b0):
                        qx, qy = ox + 2 * b0 + e[0], oy + 2 * b1 + e[1]
                        if qx >= n or qy >= n:
                            continue
                        terms.append((bindex2((b0, b1), mm), (qx - PX) // 2, (qy - PY) // 2))
                expr = "0.0"
                for bi, ix, iy in terms:
                    expr = f"fma(P.GM[{bi}], p{ix}_{iy}, {expr})"
                f = ox * n1 + oy
                inv = 1.0 / (factorial(ox) * factorial(oy))
                L.append(f"  {{ const double v = fma({expr}, {inv!r}, tg[{(t * n1 * n1 + f) * TXC} + lane]); bad |= !isfinite(v);"
                         f" if (active) dptr[{t}][{f} * P.t_plane] = v; }}")
    L.append("}")
    return "\n".join(L)


def gen_class_merged(mm, PX, PY, name):
    """merged pressure (V_x + V_y) y half-lines + CK for class (PX, PY):
    P~ = My (Mx^{+1} V_x) + My^{+1} (Mx V_y), ring A holds the shifted x-lines
    of V_x, ring B the x-lines of V_y; the CK then has no index shift."""
    n1, n = mm + 1, 2 * mm + 2
    nh = n // 2
    L = [f"__device__ __forceinline__ void {name}(const T2Params& P, const double* __restrict__ ro,",
         "    const double* __restrict__ rn, const double* __restrict__ rob, const double* __restrict__ rnb,",
         "    const double* __restrict__ tg, int lane, double* const* dptr, bool active, bool& bad) {",
         "  // ro/rn = ring A + lane, rob/rnb = ring B + lane; tg = staged targets [f][cell]"]
    for ix in range(nh):
        qx = PX + 2 * ix
        outs = [PY + 2 * iy for iy in range(nh)]
        ra = half_line(mm, lambda l, qx=qx: f"ro[{(qx * n1 + l) * TXC}]", lambda l, qx=qx: f"rn[{(qx * n1 + l) * TXC}]",
                       outs, f"a{ix}_", L)
        rb = half_line(mm, lambda l, qx=qx: f"rob[{(qx * n1 + l) * TXC}]", lambda l, qx=qx: f"rnb[{(qx * n1 + l) * TXC}]",
                       outs, f"b{ix}_", L, sh=1)
        for iy in range(nh):
            terms = [t for t in (ra[PY + 2 * iy], rb[PY + 2 * iy]) if t != "0.0"]
            L.append(f"  const double p{ix}_{iy} = {' + '.join(terms) if terms else '0.0'};")
    for ox in range(n1):
        for oy in range(n1):
            if (ox & 1) != PX or (oy & 1) != PY:
                continue
            expr = "0.0"
            for b0 in range(mm + 1):
                for b1 in range(mm + 1 - b0):
                    qx, qy = ox + 2 * b0, oy + 2 * b1
                    if qx >= n or qy >= n:
                        continue
                    expr = f"fma(P.GM[{bindex2((b0, b1), mm)}], p{(qx - PX) // 2}_{(qy - PY) // 2}, {expr})"
            f = ox * n1 + oy
            inv = 1.0 / (factorial(ox) * factorial(oy))
            L.append(f"  {{ const double v = fma({expr}, {inv!r}, tg[{f * TXC} + lane]); bad |= !isfinite(v);"
                     f" if (active) dptr[0][{f} * P.t_plane] = v; }}")
    L.append("}")
    return "\n".join(L)


def main():
    parts = ["// GENERATED by tools/gen_tiled2d.py -- do not edit.",
             "// Stage code of the tiled 2D Hermite-leapfrog kernel (kernels_tiled2d.cu).", "#pragma once", ""]
    for mm in (1, 2, 3, 4):
        parts.append(f"// ---------------- m = {mm}")
        for px in range(2):
            parts += [gen_x(mm, px), ""]
            parts += [gen_x(mm, px, sh=1, suffix="_sh"), ""]
        for kind, comps in (("vel", [0, 1]), ("pre0", [0]), ("pre1", [1])):
            for w in range(4):
                PX, PY = (w >> 1) & 1, w & 1
                parts += [gen_class(mm, PX, PY, comps, f"t2_m{mm}_{kind}_{w}"), ""]
            parts.append(f"__device__ __forceinline__ void t2_m{mm}_{kind}(int w, const T2Params& P, const double* ro,")
            parts.append("    const double* rn, const double* tg, int lane, double* const* dptr, bool active, bool& bad) {")
            parts.append("  switch (w) {")
            for w in range(4):
                parts.append(f"    case {w}: t2_m{mm}_{kind}_{w}(P, ro, rn, tg, lane, dptr, active, bad); break;")
            parts.append("    default: break;")
            parts.append("  }")
            parts.append("}")
            parts.append("")
        for w in range(4):
            PX, PY = (w >> 1) & 1, w & 1
            parts += [gen_class_merged(mm, PX, PY, f"t2_m{mm}_prem_{w}"), ""]
        parts.append(f"__device__ __forceinline__ void t2_m{mm}_prem(int w, const T2Params& P, const double* ro,")
        parts.append("    const double* rn, const double* rob, const double* rnb, const double* tg, int lane,")
        parts.append("    double* const* dptr, bool active, bool& bad) {")
        parts.append("  switch (w) {")
        for w in range(4):
            parts.append(f"    case {w}: t2_m{mm}_prem_{w}(P, ro, rn, rob, rnb, tg, lane, dptr, active, bad); break;")
        parts.append("    default: break;")
        parts.append("  }")
        parts.append("}")
        parts.append("")
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
