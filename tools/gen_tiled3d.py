"""Generate paper_1808_10481_b200/csrc/tiled3d_gen.cuh: straight-line stage code
for the tiled 3D kernel (kernels_tiled3d.cu), for m = 1, 2, 3.

Why generated: the stage bodies are hundreds of FMAs with compile-time operand
indices.  Expressed as templates/unrolled loop nests they made nvcc's optimizer
run for tens of minutes; explicit statements compile in seconds.  The code is
also organised to keep the hot instruction footprint small (the first version
specialised everything per parity class and ran out of instruction cache):

  m{m}_xy_px{p}   fused X+Y stage of one (l_z, q_x parity) task: 2(m+1) half
                  x-lines (outputs q_x = p mod 2) feeding the y-lines in registers
  m{m}_z_pz{p}    z stage of one parity class: P~[q] for the class's columns
  m{m}_ck_*       closed-form CK sum of one target component in class-local
                  indices (deduplicated: for odd m it depends only on the shift
                  of the derivative axis, so 6 bodies serve all 24 (class, c))

Math (rows of M pre-scaled by s!):
  P~[q] = qx! qy! qz! P[q];  parity split of every 1D line:
  out[s] = sum_{l = s mod 2} ML[s][l] (L_l + R_l) - sum_{l != s mod 2} ML[s][l] (R_l - L_l)
  out_c[o] = (1/o!) sum_{|b| <= m} GM[b] P~[o + 2b + e_c],  GM[b] = G_|b| |b|!/b!
Usage: python tools/gen_tiled3d.py   (writes the header; committed)
"""
from __future__ import annotations

import itertools
import os

TXC = 32
RAWX = TXC + 2  # raw row stride: 33 nodes used, 34 for 16 B aligned TMA row copies
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "paper_1808_10481_b200", "csrc", "tiled3d_gen.cuh")


def bindex(b, mm):
    idx = 0
    for a0 in range(mm + 1):
        for a1 in range(mm + 1 - a0):
            for a2 in range(mm + 1 - a0 - a1):
                if (a0, a1, a2) == tuple(b):
                    return idx
                idx += 1
    raise ValueError(b)


def mzero(r, l, mm):
    """M[r][l] is exactly zero for even rows r >= 2 and l = 0 (the value
    coefficient of the even Taylor orders); the host checks it for the fast
    kernels (hlf_capi.cu, m_mirror) and these terms are not emitted.  From m = 4
    on the reference's LU inverse leaves round-off there, which is kept."""
    return mm <= 3 and l == 0 and r >= 2 and r % 2 == 0


def half_line(mm, srcL, srcR, outs, tmp, lines, sh=0):
    """outputs s in `outs` of a parity-split line from L/R expressions.  sh = 1
    uses row s+1 of M for output s (the index shift of a divergence term,
    merged pressure kernel); rows past 2m+1 give the literal 0.0."""
    n1, n = mm + 1, 2 * mm + 2
    need_s, need_d = set(), set()
    for s in outs:
        if s + sh >= n:
            continue
        for l in range(n1):
            if not mzero(s + sh, l, mm):
                (need_s if (s + sh + l) % 2 == 0 else need_d).add(l)
    for l in sorted(need_s):
        lines.append(f"  const double {tmp}s{l} = {srcL(l)} + {srcR(l)};")
    for l in sorted(need_d):
        lines.append(f"  const double {tmp}d{l} = {srcR(l)} - {srcL(l)};")
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
        lines.append(f"  const double {name} = {expr};")
        res[s] = name
    return res


def gen_xy(mm, px, shx=0, shy=0, acc=False, suffix=""):
    """fused X+Y task; shx / shy shift the x / y rows (merged pressure kernel:
    V_x enters through rows q_x+1, V_y through rows q_y+1); acc adds into the
    ring instead of storing."""
    n1, n = mm + 1, 2 * mm + 2
    L = [f"__device__ __forceinline__ void m{mm}_xy_px{px}{suffix}(const TParams& P, const double* __restrict__ rb,",
         "                                                  double* __restrict__ wb) {",
         "  // rb = raw + l_z*2*RAWX + lane;  wb = ring_new + l_z*TXC + lane"]
    qxs = [q for q in range(n) if q % 2 == px]
    xh = {}
    for sy in range(2):
        for ly in range(n1):
            def off(lx, side, sy=sy, ly=ly):
                return f"rb[{((lx * n1 * n1 + ly * n1) * 2 + sy) * RAWX + side}]"
            res = half_line(mm, lambda l: off(l, 0), lambda l: off(l, 1), qxs, f"x{sy}{ly}", L, shx)
            for q, nm in res.items():
                xh[(sy, ly, q)] = nm
    for qx in qxs:
        if qx + shx >= n:  # the whole x row is zero
            if not acc:
                for qy in range(n):
                    L.append(f"  wb[{(qx * n + qy) * n1 * TXC}] = 0.0;")
            continue
        res = half_line(mm, lambda l, qx=qx: xh[(0, l, qx)], lambda l, qx=qx: xh[(1, l, qx)],
                        list(range(n)), f"y{qx}", L, shy)
        for qy, nm in res.items():
            o = (qx * n + qy) * n1 * TXC
            if acc:
                if nm != "0.0":
                    L.append(f"  wb[{o}] += {nm};")
            else:
                L.append(f"  wb[{o}] = {nm};")
    L.append("}")
    return "\n".join(L)


def gen_xy_merged(mm, px):
    """merged pressure XY task: C = (My x Mx^{+1}) V_x + (My^{+1} x Mx) V_y for
    the task's q_x parity, summed in registers (one ring store per value)."""
    n1, n = mm + 1, 2 * mm + 2
    L = [f"__device__ __forceinline__ void m{mm}_xy_px{px}_vxy(const TParams& P, const double* __restrict__ rbx,",
         "    const double* __restrict__ rby, double* __restrict__ wb) {",
         "  // rbx / rby = raw V_x / raw V_y + l_z*2*RAWX + lane;  wb = ring_new + l_z*TXC + lane"]
    qxs = [q for q in range(n) if q % 2 == px]
    xh = {}
    for fld, rb, shx in (("a", "rbx", 1), ("b", "rby", 0)):
        for sy in range(2):
            for ly in range(n1):
                def off(lx, side, sy=sy, ly=ly, rb=rb):
                    return f"{rb}[{((lx * n1 * n1 + ly * n1) * 2 + sy) * RAWX + side}]"
                res = half_line(mm, lambda l: off(l, 0), lambda l: off(l, 1), qxs, f"{fld}{sy}{ly}", L, shx)
                for q, nm in res.items():
                    xh[(fld, sy, ly, q)] = nm
    for qx in qxs:
        parts = {}
        for fld, shy in (("a", 0), ("b", 1)):
            if fld == "a" and qx + 1 >= n:
                continue  # V_x row q_x+1 does not exist
            res = half_line(mm, lambda l, qx=qx, fld=fld: xh[(fld, 0, l, qx)],
                            lambda l, qx=qx, fld=fld: xh[(fld, 1, l, qx)], list(range(n)), f"y{fld}{qx}", L, shy)
            for qy, nm in res.items():
                if nm != "0.0":
                    parts.setdefault(qy, []).append(nm)
        for qy in range(n):
            terms = parts.get(qy, [])
            expr = " + ".join(terms) if terms else "0.0"
            L.append(f"  wb[{(qx * n + qy) * n1 * TXC}] = {expr};")
    L.append("}")
    return "\n".join(L)


def gen_z(mm, pz):
    n1, n = mm + 1, 2 * mm + 2
    nh = n // 2
    L = [f"__device__ __forceinline__ void m{mm}_z_pz{pz}(const TParams& P, const double* __restrict__ ro,",
         f"    const double* __restrict__ rn, double (&pt)[{nh}][{nh}][{nh}]) {{",
         "  // ro/rn = ring + ((PX*n + PY)*n1)*TXC + lane"]
    for ix in range(nh):
        for iy in range(nh):
            off = ((2 * ix) * n + 2 * iy) * n1 * TXC
            L.append("  {")
            sub = []
            res = half_line(mm, lambda l, off=off: f"ro[{off + l * TXC}]", lambda l, off=off: f"rn[{off + l * TXC}]",
                            [pz + 2 * iz for iz in range(nh)], "z", sub)
            L.extend("  " + s for s in sub)
            for iz in range(nh):
                L.append(f"    pt[{ix}][{iy}][{iz}] = {res[pz + 2 * iz]};")
            L.append("  }")
    L.append("}")
    return "\n".join(L)


def ck_body(mm, c, cls):
    """CK for target component c in parity class cls = (PX, PY, PZ); returns
    (list of (jx, jy, jz) outputs, list of statements)."""
    n1, n = mm + 1, 2 * mm + 2
    nh = n // 2
    P = cls
    e = [int(c == a) for a in range(3)]
    outs = []
    for ox in range(n1):
        for oy in range(n1):
            for oz in range(n1):
                o = (ox, oy, oz)
                if all(((o[a] + e[a]) & 1) == P[a] for a in range(3)):
                    outs.append(o)
    stm = []
    for o in outs:
        j = tuple((o[a] - ((P[a] - e[a]) & 1)) // 2 for a in range(3))
        terms = []
        for b0 in range(mm + 1):
            for b1 in range(mm + 1 - b0):
                for b2 in range(mm + 1 - b0 - b1):
                    b = (b0, b1, b2)
                    q = [o[a] + 2 * b[a] + e[a] for a in range(3)]
                    if any(x >= n for x in q):
                        continue
                    i = tuple((q[a] - P[a]) // 2 for a in range(3))
                    terms.append((bindex(b, mm), i))
        for bi, i in terms:
            stm.append(f"  acc[{j[0]}][{j[1]}][{j[2]}] = fma(P.GM[{bi}], pt[{i[0]}][{i[1]}][{i[2]}], acc[{j[0]}][{j[1]}][{j[2]}]);")
    return outs, stm


def gen_vel_q_shared(mm):
    """Velocity launch, one CK body for every class: the Q entries any class
    needs (class-local q in [0, jh]^3 with at most one coordinate = jh:
    v_c[o] = Q[o + e_c] reads q = j + (1 - P_c) e_c), 2624 instead of 3360
    FMAs per cell at m = 3; the class picks its three components' entries
    (warp-uniform shifts) in m3_vel_pick."""
    n1, n = mm + 1, 2 * mm + 2
    nh, jh = n // 2, (n1 + 1) // 2
    L = [f"__device__ __forceinline__ void m{mm}_vel_qs(const TParams& P, const double (&pt)[{nh}][{nh}][{nh}],",
         f"    double (&Q)[{jh + 1}][{jh + 1}][{jh + 1}]) {{"]
    for q in itertools.product(range(jh + 1), repeat=3):
        if sum(1 for x in q if x == jh) > 1:
            continue
        nm = f"Q[{q[0]}][{q[1]}][{q[2]}]"
        L.append(f"  {nm} = 0.0;")
        for b0 in range(mm + 1):
            for b1 in range(mm + 1 - b0):
                for b2 in range(mm + 1 - b0 - b1):
                    b = (b0, b1, b2)
                    i = [q[a] + b[a] for a in range(3)]
                    if any(x >= nh for x in i):
                        continue
                    L.append(f"  {nm} = fma(P.GM[{bindex(b, mm)}], pt[{i[0]}][{i[1]}][{i[2]}], {nm});")
    L.append("}")
    return "\n".join(L)


# ---------------------------------------------------------------- y-first XY
# m = 3: the y sweep runs first, once per source node and (q_x, q_z) pair (the
# two source rows of a cell row belong to that row alone, so no line is swept
# twice), in place over the raw stage; the x sweep then runs on the y results
# of neighbouring nodes.  x-first sweeps every source row for both cell rows
# that share it (2 (m+1)^2 x-lines per cell instead of (m+1)^2).
#   raw / Y index: (((qx*n1 + qy)*n1 + qz)*2 + sy)*RAWX + node; the y line of
#   (qx, qz) at a node reads slots (qy, sy) and writes output jy to slot
#   (qy, sy) = (jy >> 1, jy & 1).
def yslot(mm, qx, jy, qz):
    n1 = mm + 1
    return (((qx * n1 + (jy >> 1)) * n1 + qz) * 2 + (jy & 1)) * RAWX


def gen_yline(mm, shy, suffix):
    n1, n = mm + 1, 2 * mm + 2
    L = [f"__device__ __forceinline__ void m{mm}_yl{suffix}(const TParams& P, double* __restrict__ yb) {{",
         "  // yb = raw + (qx*n1*n1 + qz)*2*RAWX + node: one y line, in place"]
    src = {}
    for sy in range(2):
        for l in range(n1):
            nm = f"r{sy}{l}"
            L.append(f"  const double {nm} = yb[{(l * n1 * 2 + sy) * RAWX}];")
            src[(sy, l)] = nm
    res = half_line(mm, lambda l: src[(0, l)], lambda l: src[(1, l)], list(range(n)), "y", L, shy)
    for jy in range(n):
        L.append(f"  yb[{((jy >> 1) * n1 * 2 + (jy & 1)) * RAWX}] = {res[jy]};")
    L.append("}")
    return "\n".join(L)


def gen_xtask(mm, jyp, merged):
    """x lines of one (q_z, j_y parity) task: jy = jyp, jyp+2, ...; full lines
    (all n outputs j_x) into the ring.  merged: V_x through rows q_x+1 plus V_y."""
    n1, n = mm + 1, 2 * mm + 2
    if merged:
        L = [f"__device__ __forceinline__ void m{mm}_xt{jyp}_vxy(const TParams& P, const double* __restrict__ xbx,",
             "    const double* __restrict__ xby, double* __restrict__ wb) {"]
        flds = (("a", "xbx", 1), ("b", "xby", 0))
    else:
        L = [f"__device__ __forceinline__ void m{mm}_xt{jyp}(const TParams& P, const double* __restrict__ xbx,",
             "    double* __restrict__ wb) {"]
        flds = (("a", "xbx", 0),)
    L.append("  // xb = Y + qz*2*RAWX + lane;  wb = ring_new + qz*TXC + lane")
    for jy in range(jyp, n, 2):
        # one FMA chain per output over both fields' sum / difference terms
        # (the merged launch: no separate add of the two lines)
        chains = {jx: "0.0" for jx in range(n)}
        for fld, xb, shx in flds:
            def off(l, side, jy=jy, xb=xb):
                return f"{xb}[{yslot(mm, l, jy, 0) + side}]"
            need_s, need_d = set(), set()
            for jx in range(n):
                r = jx + shx
                for l in range(n1):
                    if r < n and not mzero(r, l, mm):
                        (need_s if (r + l) % 2 == 0 else need_d).add(l)
            for l in sorted(need_s):
                L.append(f"  const double {fld}{jy}s{l} = {off(l, 0)} + {off(l, 1)};")
            for l in sorted(need_d):
                L.append(f"  const double {fld}{jy}d{l} = {off(l, 1)} - {off(l, 0)};")
            for jx in range(n):
                r = jx + shx
                if r >= n:
                    continue
                for l in range(n1):
                    if mzero(r, l, mm):
                        continue
                    if (r + l) % 2 == 0:
                        chains[jx] = f"fma(P.ML[{r * n1 + l}], {fld}{jy}s{l}, {chains[jx]})"
                    else:
                        chains[jx] = f"fma(-P.ML[{r * n1 + l}], {fld}{jy}d{l}, {chains[jx]})"
        for jx in range(n):
            L.append(f"  wb[{(jx * n + jy) * n1 * TXC}] = {chains[jx]};")
    L.append("}")
    return "\n".join(L)


# ---------------------------------------------------------------- z-folded CK
# Pressure launches, m = 3: the z sweep is folded into the CK.  For output
# o = (ox, oy, oz) of class parity (PX, PY, PZo) and a ring column (jx, jy) =
# (ox + 2a, oy + 2b) (class-local ix = jxo + a, iy = jyo + b):
#   sum_c GM[a,b,c] P~[jx, jy, oz + 2c + sh] = sum_l R[a,b][jzo][l] w_l,
#   R[a,b][jzo][l] = sum_c GM[a,b,c] (+-) s! M[s][l],  s = oz + 2c + sh < n,
# w_l = sigma_l (s + l even) or delta_l (odd) of the column's two ring layers
# (sh = 1: the V_z divergence term's index shift).  4 FMAs per (column,
# output) instead of the z half line (16) plus the CK terms that read it.
# The host fills R (TParams.RZ[PZo][ab][jzo][l], kernels_tiled3d.cu rz_table).
def ab_index(a, b, mm):
    idx = 0
    for a0 in range(mm + 1):
        for b0 in range(mm + 1 - a0):
            if (a0, b0) == (a, b):
                return idx
            idx += 1
    raise ValueError((a, b))


def rz_zero(mm, sh, pzo, jzo, l):
    """R[..][jzo][l] is exactly zero when every row s it sums has M[s][l] = 0"""
    n = 2 * mm + 2
    oz = pzo + 2 * jzo
    rows = [oz + 2 * c + sh for c in range(mm + 1) if oz + 2 * c + sh < n]
    return all(mzero(r, l, mm) for r in rows)


def gen_zf(mm, pzo, sh):
    n1, n = mm + 1, 2 * mm + 2
    nh, jh = n // 2, (n1 + 1) // 2
    nab = (mm + 1) * (mm + 2) // 2
    L = [f"__device__ __forceinline__ void m{mm}_zf_s{sh}_pz{pzo}(const TParams& P, const double* __restrict__ ro,",
         f"    const double* __restrict__ rn, double (&acc)[{jh}][{jh}][{jh}]) {{",
         "  // ro/rn = ring + ((PX*n + PY)*n1)*TXC + lane (non-V7 layout); class = output parity"]
    for ix in range(nh):
        for iy in range(nh):
            terms = []
            for jxo in range(jh):
                for jyo in range(jh):
                    a, b = ix - jxo, iy - jyo
                    if a < 0 or b < 0 or a + b > mm:
                        continue
                    for jzo in range(jh):
                        if pzo + 2 * jzo <= mm:  # o_z <= m (m = 2: PZo = 1 has one output layer)
                            terms.append((jxo, jyo, jzo, ab_index(a, b, mm)))
            if not terms:
                continue
            off = ((2 * ix) * n + 2 * iy) * n1 * TXC
            L.append("  {")
            # sigma / delta the terms need: w_l = sigma_l if (oz + sh + l) even
            need = set()
            for (_, _, jzo, _) in terms:
                for l in range(n1):
                    if not rz_zero(mm, sh, pzo, jzo, l):
                        need.add(l)
            for l in sorted(need):
                if (pzo + sh + l) % 2 == 0:
                    L.append(f"    const double w{l} = ro[{off + l * TXC}] + rn[{off + l * TXC}];")
                else:
                    L.append(f"    const double w{l} = rn[{off + l * TXC}] - ro[{off + l * TXC}];")
            for (jxo, jyo, jzo, ab) in terms:
                nm = f"acc[{jxo}][{jyo}][{jzo}]"
                expr = nm
                for l in range(n1):
                    if rz_zero(mm, sh, pzo, jzo, l):
                        continue
                    expr = f"fma(P.RZ[{((pzo * nab + ab) * jh + jzo) * n1 + l}], w{l}, {expr})"
                L.append(f"    {nm} = {expr};")
            L.append("  }")
    L.append("}")
    return "\n".join(L)


def main():
    parts = ["// GENERATED by tools/gen_tiled3d.py -- do not edit.",
             "// Stage code of the tiled 3D Hermite-leapfrog kernel (kernels_tiled3d.cu).",
             "#pragma once", ""]
    for mm in (1, 2, 3):
        n1, n = mm + 1, 2 * mm + 2
        nh, jh = n // 2, (n1 + 1) // 2
        parts.append(f"// ---------------- m = {mm}")
        for px in range(2):
            parts.append(gen_xy(mm, px))
            parts.append("")
            # merged pressure (V_x + V_y) launch: C = (My x Mx^{+1}) V_x + (My^{+1} x Mx) V_y
            parts.append(gen_xy(mm, px, shx=1, suffix="_vx"))
            parts.append("")
            parts.append(gen_xy(mm, px, shy=1, acc=True, suffix="_vy"))
            parts.append("")
            parts.append(gen_xy_merged(mm, px))
            parts.append("")
        for pz in range(2):
            parts.append(gen_z(mm, pz))
            parts.append("")
        bodies = {}
        dispatch = {}
        for c in range(3):
            for w in range(8):
                cls = ((w >> 2) & 1, (w >> 1) & 1, w & 1)
                outs, stm = ck_body(mm, c, cls)
                key = "\n".join(stm)
                if key not in bodies:
                    fname = f"m{mm}_ck_{len(bodies)}"
                    bodies[key] = fname
                    parts.append(f"__device__ __forceinline__ void {fname}(const TParams& P, const double (&pt)[{nh}][{nh}][{nh}],")
                    parts.append(f"    double (&acc)[{jh}][{jh}][{jh}]) {{")
                    parts.extend(stm)
                    parts.append("}")
                    parts.append("")
                dispatch[(c, w)] = bodies[key]
        parts.append(f"__device__ __forceinline__ void m{mm}_ck(int c, int w, const TParams& P,")
        parts.append(f"    const double (&pt)[{nh}][{nh}][{nh}], double (&acc)[{jh}][{jh}][{jh}]) {{")
        # group (c, w) by body to keep the dispatch small
        by_body = {}
        for (c, w), fn in dispatch.items():
            by_body.setdefault(fn, []).append(c * 8 + w)
        parts.append("  switch (c * 8 + w) {")
        for fn, keys in by_body.items():
            for k in keys:
                parts.append(f"    case {k}:")
            parts.append(f"      {fn}(P, pt, acc);")
            parts.append("      break;")
        parts.append("    default: break;")
        parts.append("  }")
        parts.append("}")
        parts.append("")
        # merged pressure launch: the index shift sits in the sweep rows, so the
        # CK has no shift (c = -1); per class w (deduplicated)
        ns = {}
        parts.append(f"__device__ __forceinline__ void m{mm}_ck_noshift(int w, const TParams& P,")
        parts.append(f"    const double (&pt)[{nh}][{nh}][{nh}], double (&acc)[{jh}][{jh}][{jh}]) {{")
        parts.append("  switch (w) {")
        for w in range(8):
            cls = ((w >> 2) & 1, (w >> 1) & 1, w & 1)
            outs, stm = ck_body(mm, -1, cls)
            key = "\n".join(stm)
            fn = bodies.get(key)
            if fn is None:
                fn = ns.get(key)
            parts.append(f"    case {w}:")
            if fn is not None:
                parts.append(f"      {fn}(P, pt, acc);")
            else:
                parts.extend("    " + x for x in stm)
            parts.append("      break;")
        parts.append("    default: break;")
        parts.append("  }")
        parts.append("}")
        parts.append("")
        if mm >= 2:
            # z-folded CK of the pressure launches (m = 2, 3)
            for sh in range(2):
                for pzo in range(2):
                    parts.append(gen_zf(mm, pzo, sh))
                    parts.append("")
        if mm == 3:
            parts.append(gen_vel_q_shared(mm))
            parts.append("")
            # y-first XY stage (kernels_tiled3d.cu, m = 3)
            parts.append(gen_yline(mm, 0, ""))
            parts.append("")
            parts.append(gen_yline(mm, 1, "_sh"))
            parts.append("")

            for jyp in range(2):
                parts.append(gen_xtask(mm, jyp, False))
                parts.append("")
                parts.append(gen_xtask(mm, jyp, True))
                parts.append("")
        parts.append(f"// m = {mm}: {len(bodies)} distinct CK bodies")
        parts.append("")
    with open(OUT, "w") as f:
        f.write("\n".join(parts))
    print("wrote", OUT)




# ====================================================================== v7
# Z + CK stage with the two q_z-parity classes in one warp (m = 3):
#   warp = (PX, PY, cell half), lane = (cell in half, PZ = lane >> 4).
# Both halves read the same ring words (shared-memory broadcast), the z half
# line uses per-lane rows cz[iz][l] = s! M[PZ + 2 iz][l] and the per-lane sign
# g = (-1)^PZ:  P~[PZ + 2 iz] = sum_l cz[iz][l] (L_l + g (-1)^l R_l).
# The CK bodies are class-local (c, shift); the z shift of PZ = 0 lanes is an
# in-register shift of pt before the z-component body.
def v7_gen_z(mm):
    n1, n = mm + 1, 2 * mm + 2
    nh = n // 2
    L = [f"__device__ __forceinline__ void v7_m{mm}_z(const double* __restrict__ ro, const double* __restrict__ rn,",
         f"    const double (&cz)[{nh}][{n1}], double g, double (&pt)[{nh}][{nh}][{nh}]) {{",
         "  // ro/rn = ring + ((PX*n + PY)*n1)*TXC + cell"]
    for ix in range(nh):
        for iy in range(nh):
            off = ((2 * ix) * n + 2 * iy) * n1 * TXC
            L.append("  {")
            for l in range(n1):
                sg = "g" if l % 2 == 0 else "-g"
                L.append(f"    const double u{l} = fma({sg}, rn[{off + l * TXC}], ro[{off + l * TXC}]);")
            for iz in range(nh):
                expr = "0.0"
                for l in range(n1):
                    expr = f"fma(cz[{iz}][{l}], u{l}, {expr})"
                L.append(f"    pt[{ix}][{iy}][{iz}] = {expr};")
            L.append("  }")
    L.append("}")
    return "\n".join(L)


def v7_gen_ck(mm, c, sh):
    n1, n = mm + 1, 2 * mm + 2
    nh, jh = n // 2, (n1 + 1) // 2
    e = [int(c == a) for a in range(3)]
    L = [f"__device__ __forceinline__ void v7_m{mm}_ck_c{c}_s{sh}(const TParams& P, const double (&pt)[{nh}][{nh}][{nh}],",
         f"    double (&acc)[{jh}][{jh}][{jh}]) {{"]
    for jx in range(jh):
        for jy in range(jh):
            for jz in range(jh):
                j = (jx, jy, jz)
                for b0 in range(mm + 1):
                    for b1 in range(mm + 1 - b0):
                        for b2 in range(mm + 1 - b0 - b1):
                            b = (b0, b1, b2)
                            i = [j[a] + b[a] + sh * e[a] for a in range(3)]
                            if any(x >= nh for x in i):
                                continue
                            L.append(f"  acc[{jx}][{jy}][{jz}] = fma(P.GM[{bindex(b, mm)}], pt[{i[0]}][{i[1]}][{i[2]}], acc[{jx}][{jy}][{jz}]);")
    L.append("}")
    return "\n".join(L)


def v7_gen_zck(mm, c, sh, zsel=False):
    """Z stage fused with the CK (streaming): for each class column (ix, iy)
    the z half line gives P~[ix][iy][*] (4 values), which are folded into the
    accumulators right away (every CK term that reads this column), so only one
    column of P~ is live at a time instead of all 64 (register pressure ->
    deeper load pipelining, and the ring loads interleave with the CK FMAs).
    zsel: the z component of the V_z pressure launch, whose PZ = 0 lanes read
    P~ one z index up (per-lane select inside the column)."""
    n1, n = mm + 1, 2 * mm + 2
    nh, jh = n // 2, (n1 + 1) // 2
    e = [int(c == a) for a in range(3)]
    name = f"v7_m{mm}_zck_c{c}_s{sh}" if not zsel else f"v7_m{mm}_zck_zsel"
    L = [f"__device__ __forceinline__ void {name}(const TParams& P, const double* __restrict__ ro,",
         f"    const double* __restrict__ rn, const double (&cz)[{nh}][{n1}], double g, int pz,",
         f"    double (&acc)[{jh}][{jh}][{jh}]) {{",
         "  // ro/rn = ring + ((PX*n + PY)*n1)*TXC + cell"]
    if not zsel:
        L.append("  (void)pz;")
    # CK terms grouped by the class column they read
    terms = {}
    for jx in range(jh):
        for jy in range(jh):
            for jz in range(jh):
                j = (jx, jy, jz)
                for b0 in range(mm + 1):
                    for b1 in range(mm + 1 - b0):
                        for b2 in range(mm + 1 - b0 - b1):
                            b = (b0, b1, b2)
                            i = [j[a] + b[a] + sh * e[a] for a in range(3)]
                            if any(x >= nh for x in i):
                                continue
                            terms.setdefault((i[0], i[1]), []).append((j, bindex(b, mm), i[2]))
    for ix in range(nh):
        for iy in range(nh):
            if (ix, iy) not in terms:
                continue  # no CK term reads this column
            off = ((2 * ix) * n + 2 * iy) * n1 * TXC
            L.append("  {")
            for l in range(n1):
                sg = "g" if l % 2 == 0 else "-g"
                L.append(f"    const double u{l} = fma({sg}, rn[{off + l * TXC}], ro[{off + l * TXC}]);")
            need = sorted({iz for (_, _, iz) in terms[(ix, iy)]})
            top = max(need) + (1 if zsel else 0)
            for iz in range(min(top, nh - 1) + 1):
                expr = "0.0"
                for l in range(n1):
                    expr = f"fma(cz[{iz}][{l}], u{l}, {expr})"
                L.append(f"    const double p{iz} = {expr};")
            if zsel:
                # PZ = 0 lanes read P~ one z index up (row 2 iz + 2; past the top: 0)
                for iz in need:
                    up = f"p{iz + 1}" if iz + 1 < nh else "0.0"
                    L.append(f"    const double q{iz} = pz ? p{iz} : {up};")
            for (j, bi, iz) in terms[(ix, iy)]:
                src = f"q{iz}" if zsel else f"p{iz}"
                L.append(f"    acc[{j[0]}][{j[1]}][{j[2]}] = fma(P.GM[{bi}], {src}, acc[{j[0]}][{j[1]}][{j[2]}]);")
            L.append("  }")
    L.append("}")
    return "\n".join(L)


def main_v7():
    out = os.path.join(HERE, "..", "paper_1808_10481_b200", "csrc", "tiled3d_v7_gen.cuh")
    mm = 3
    parts = ["// GENERATED by tools/gen_tiled3d.py (v7) -- do not edit.",
             "// Z + CK stage with q_z-parity pairs per warp, m = 3 (kernels_tiled3d.cu).", "#pragma once", "",
             v7_gen_z(mm), ""]
    for c in range(3):
        for sh in range(2):
            parts += [v7_gen_ck(mm, c, sh), ""]
    # fused (streaming) Z + CK bodies of the pressure launches
    for c in range(2):
        for sh in range(2):
            parts += [v7_gen_zck(mm, c, sh), ""]
    parts += [v7_gen_zck(mm, 2, 0, zsel=True), ""]
    with open(out, "w") as f:
        f.write("\n".join(parts))
    print("wrote", out)


if __name__ == "__main__":
    main()
    main_v7()
