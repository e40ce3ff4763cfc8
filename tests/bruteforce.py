"""Independent brute-force literal implementations of Alg. 1 and Alg. 2,
written in pure Python over a DENSE adjacency matrix (the view of Fig. 3,
P:652-661), used only to pin the C oracle on tiny graphs (n <= 8).

Shares no code with oracle/ (different language, different data structure,
math.hypot for the distance).  PAPER.md citations:
  f_a = ||c_i-c_j||^2 / K, f_r = -R K^2 / ||c_i-c_j||      §2.2 P:524-528 (reading C1)
  f(i,c) = sum_adj f_a u_ij + sum_nonadj f_r u_ij            §2.2
  c_i += Step f/||f||; Energy += ||f||^2                     Alg. 1
  Step *= 0.999 per iteration                                Alg. 1
  minibatch: forces frozen, then batch update                Alg. 2
"""
import math


def dense_adj(n, rowptr, colidx):
    A = [[False] * n for _ in range(n)]
    for i in range(n):
        for k in range(int(rowptr[i]), int(rowptr[i + 1])):
            A[i][int(colidx[k])] = True
    return A


def _force(n, A, c, i, K, R, repulse_neighbors=False, a=2.0, r=-1.0):
    fx = fy = 0.0
    for j in range(n):
        if j == i:
            continue
        dist = math.hypot(c[j][0] - c[i][0], c[j][1] - c[i][1])
        if dist == 0.0:
            continue
        ux = (c[j][0] - c[i][0]) / dist
        uy = (c[j][1] - c[i][1]) / dist
        rep = -R * K * K * math.pow(dist, r)     # (a, r)-model, reading C15
        if A[i][j]:
            att = math.pow(dist, a) / K
            fx += att * ux
            fy += att * uy
            if repulse_neighbors:
                fx += rep * ux
                fy += rep * uy
        else:
            fx += rep * ux
            fy += rep * uy
    return fx, fy


def alg1(n, A, c0, iters, K=1.0, R=1.0, step0=1.0, factor=0.999):
    """Algorithm 1: Gauss-Seidel, immediate update."""
    c = [[float(p[0]), float(p[1])] for p in c0]
    step = step0
    energies = []
    for _ in range(iters):
        energy = 0.0
        for i in range(n):
            fx, fy = _force(n, A, c, i, K, R)
            norm = math.hypot(fx, fy)
            if norm > 0:
                c[i][0] += step * fx / norm
                c[i][1] += step * fy / norm
            energy += norm * norm
        energies.append(energy)
        step *= factor
    return c, energies


def alg2(n, A, c0, iters, BS, K=1.0, R=1.0, step0=1.0, factor=0.999,
         repulse_neighbors=False, a=2.0, r=-1.0, perms=None):
    """Algorithm 2 semantics: consecutive minibatches, forces of
    a batch against frozen coordinates, then the batch update.  perms: one
    vertex order per iteration (batch randomisation, §4.3.3):
    batch t is perms[it][t BS : (t+1) BS]; None = the sequential order."""
    c = [[float(p[0]), float(p[1])] for p in c0]
    step = step0
    energies = []
    BS = min(BS, n)
    for it in range(iters):
        energy = 0.0
        order = list(range(n)) if perms is None else [int(v) for v in perms[it]]
        for lo in range(0, n, BS):
            batch = order[lo:min(lo + BS, n)]
            ct = [_force(n, A, c, i, K, R, repulse_neighbors, a, r) for i in batch]
            for i, (fx, fy) in zip(batch, ct):
                norm = math.hypot(fx, fy)
                if norm > 0:
                    c[i][0] += step * fx / norm
                    c[i][1] += step * fy / norm
                energy += norm * norm
        energies.append(energy)
        step *= factor
    return c, energies


# --------------------------------------------------------------- BatchLayoutBH
# An independent literal BatchLayoutBH (Alg. S1-S3) for tiny n:
# the quadtree is built GEOMETRICALLY -- a cell is an integer square of the
# 2^16 x 2^16 quantisation grid, its vertices are those whose quantised
# coordinates fall inside, children are its four sub-squares -- with no
# Morton codes, interleaving or sorting (the C oracle sorts codes).  Cell
# order: (x low, y low), (x high, y low), (x low, y high), (x high, y high).
# Readings B1-B9 of DESIGN.md §3; decisions in fp32 via numpy.float32.
import numpy as _np

_F = _np.float32


def _quant(v, vmin, scale, degenerate):
    if degenerate:
        return 0
    t = _F(_F(v) - _F(vmin)) * _F(scale)
    q = math.floor(float(t))
    return min(max(q, 0), 65535)


def _bh_cell(ids, qxy, snap, x0, y0, size, level):
    """Alg. S1 on the cell [x0, x0+size) x [y0, y0+size) of the grid."""
    node = {"level": level, "ids": ids}
    if len(ids) == 1 or level == 16:
        node["children"] = []
        sx = sum(float(snap[j][0]) for j in ids)
        sy = sum(float(snap[j][1]) for j in ids)
    else:
        half = size // 2
        node["children"] = []
        sx = sy = 0.0
        for (ox, oy) in ((0, 0), (half, 0), (0, half), (half, half)):
            sub = [j for j in ids if x0 + ox <= qxy[j][0] < x0 + ox + half
                   and y0 + oy <= qxy[j][1] < y0 + oy + half]
            if sub:
                ch = _bh_cell(sub, qxy, snap, x0 + ox, y0 + oy, half, level + 1)
                node["children"].append(ch)
                sx += ch["sx"]
                sy += ch["sy"]
    node["sx"], node["sy"] = sx, sy
    node["cx"] = _F(sx / len(ids))
    node["cy"] = _F(sy / len(ids))
    return node


def bh_build(snap):
    """snap: list of fp32 (x, y).  Returns (root, D)."""
    n = len(snap)
    xs = [_F(p[0]) for p in snap]
    ys = [_F(p[1]) for p in snap]
    D = max(_F(max(xs) - min(xs)), _F(max(ys) - min(ys)))
    degenerate = not (D > 0)
    scale = _F(0) if degenerate else _F(_F(65536.0) / D)
    qxy = [(_quant(xs[j], min(xs), scale, degenerate), _quant(ys[j], min(ys), scale, degenerate))
           for j in range(n)]
    return _bh_cell(list(range(n)), qxy, snap, 0, 0, 65536, 0), D


def _bh_rep(node, i, c, D, theta, CK2):
    """Alg. S2 calcRepulsiveForce (B1, B2, B8, B9)."""
    fx = fy = 0.0
    if not node["children"]:
        for j in node["ids"]:
            if j == i:
                continue
            dx, dy = c[j][0] - c[i][0], c[j][1] - c[i][1]
            d2 = dx * dx + dy * dy
            if d2 > 0:
                fx -= CK2 * dx / d2
                fy -= CK2 * dy / d2
        return fx, fy
    qx, qy = _F(c[i][0]), _F(c[i][1])
    ddx, ddy = _F(node["cx"] - qx), _F(node["cy"] - qy)
    dd2 = _F(_F(ddx * ddx) + _F(ddy * ddy))
    DL = _F(math.ldexp(float(D), -node["level"]))
    th = _F(theta)
    if _F(_F(th * th) * dd2) > _F(DL * DL):
        dx, dy = float(node["cx"]) - c[i][0], float(node["cy"]) - c[i][1]
        d2 = dx * dx + dy * dy
        if d2 > 0:
            m = len(node["ids"])
            fx -= m * CK2 * dx / d2
            fy -= m * CK2 * dy / d2
        return fx, fy
    for ch in node["children"]:
        gx, gy = _bh_rep(ch, i, c, D, theta, CK2)
        fx += gx
        fy += gy
    return fx, fy


def bh_layout(n, A, c0, iters, BS, theta, K=1.0, R=1.0, step0=1.0, factor=0.999):
    """Alg. S3: tree from the iteration-start coordinates (rounded to fp32),
    attraction over neighbours + tree repulsion (B3), batch update."""
    c = [[float(p[0]), float(p[1])] for p in c0]
    step = step0
    energies = []
    BS = min(BS, n)
    for _ in range(iters):
        energy = 0.0
        snap = [(_F(p[0]), _F(p[1])) for p in c]
        root, D = bh_build(snap)
        for lo in range(0, n, BS):
            batch = range(lo, min(lo + BS, n))
            ct = []
            for i in batch:
                fx = fy = 0.0
                for j in range(n):
                    if A[i][j]:
                        dist = math.hypot(c[j][0] - c[i][0], c[j][1] - c[i][1])
                        if dist > 0:
                            fx += dist * dist / K * (c[j][0] - c[i][0]) / dist
                            fy += dist * dist / K * (c[j][1] - c[i][1]) / dist
                rx, ry = _bh_rep(root, i, c, D, theta, R * K * K)
                ct.append((fx + rx, fy + ry))
            for i, (fx, fy) in zip(batch, ct):
                norm = math.hypot(fx, fy)
                if norm > 0:
                    c[i][0] += step * fx / norm
                    c[i][1] += step * fy / norm
                energy += norm * norm
        energies.append(energy)
        step *= factor
    return c, energies
