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


def _force(n, A, c, i, K, R, repulse_neighbors=False):
    fx = fy = 0.0
    for j in range(n):
        if j == i:
            continue
        dist = math.hypot(c[j][0] - c[i][0], c[j][1] - c[i][1])
        if dist == 0.0:
            continue
        ux = (c[j][0] - c[i][0]) / dist
        uy = (c[j][1] - c[i][1]) / dist
        rep = -R * K * K / dist
        if A[i][j]:
            att = dist ** 2 / K
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
         repulse_neighbors=False):
    """Algorithm 2 semantics: consecutive minibatches, forces of
    a batch against frozen coordinates, then the batch update."""
    c = [[float(p[0]), float(p[1])] for p in c0]
    step = step0
    energies = []
    BS = min(BS, n)
    for _ in range(iters):
        energy = 0.0
        for lo in range(0, n, BS):
            batch = range(lo, min(lo + BS, n))
            ct = [_force(n, A, c, i, K, R, repulse_neighbors) for i in batch]
            for i, (fx, fy) in zip(batch, ct):
                norm = math.hypot(fx, fy)
                if norm > 0:
                    c[i][0] += step * fx / norm
                    c[i][1] += step * fy / norm
                energy += norm * norm
        energies.append(energy)
        step *= factor
    return c, energies
