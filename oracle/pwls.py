"""Penalised weighted least squares with camera gains minimised out (paper §5, App. A).

eqn,pls:  Psi(x,{g}) = 1/2||A_1x - y_1||^2_W1 + sum_{c>=2} 1/2||A_cx - g_c y_c||^2_Wc
                                   + nu ||x||_1 + R(x),   x >= 0,  g_1 = 1
Weights absorbed: A~ = W^1/2 A, y~ = W^1/2 y.
Optimal gains eqn,optimal,gain: g_c = y~_c^T A~_c x / y~_c^T y~_c.
Regulariser eqn,reg, literal: R = (beta/2) sum_j sum_{l in N_j} psi(x_j - x_l),
  N_j = in-grid 26-neighbours, psi(t) = t^2/2.  Each unordered pair is
  therefore counted twice; grad_j R = beta * sum_{l in N_j} (x_j - x_l).
Gradient of the profiled cost (envelope theorem): sum_c A~_c^T (A~_c x - g_c y~_c) + grad R + nu.
Majoriser with the constant of reading Z16: d = sum_c A~_c^T A~_c 1 + 36 beta
  (the paper's 26 beta holds only when each pair is counted once; see tests).
FISTA (tab,alg missing, reading Z18): x_{k+1} = max(0, z_k - grad(z_k)/d),
  t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2, z_{k+1} = x_{k+1} + ((t_k - 1)/t_{k+1})(x_{k+1} - x_k),
  gains recomputed at z_k before each gradient, x_0 = z_0 = 0, t_0 = 1, no restart.
"""
import itertools

import numpy as np

NEIGHBOURS = [o for o in itertools.product((-1, 0, 1), repeat=3) if o != (0, 0, 0)]
MAJORISER_C = 36.0


def _shift_pairs(shape, o):
    """Slices (a, b) such that x[a] and x[b] are neighbours at offset o, both in-grid."""
    a, b = [], []
    for d, n in zip(o, shape):
        if d == 1:
            a.append(slice(0, n - 1)); b.append(slice(1, n))
        elif d == -1:
            a.append(slice(1, n)); b.append(slice(0, n - 1))
        else:
            a.append(slice(0, n)); b.append(slice(0, n))
    return tuple(a), tuple(b)


def reg_value(x, beta):
    x = np.asarray(x, np.float64)
    total = 0.0
    for o in NEIGHBOURS:
        a, b = _shift_pairs(x.shape, o)
        total += 0.5 * np.sum((x[a] - x[b]) ** 2)
    return 0.5 * beta * total


def reg_grad(x, beta):
    x = np.asarray(x, np.float64)
    g = np.zeros_like(x)
    for o in NEIGHBOURS:
        a, b = _shift_pairs(x.shape, o)
        g[a] += x[a] - x[b]
    return beta * g


def stats(Ax, y, w):
    """[y~^T A~x, y~^T y~, ||A~x||^2] in fp64."""
    Ax, y, w = (np.asarray(v, np.float64).ravel() for v in (Ax, y, w))
    return np.array([np.sum(w * y * Ax), np.sum(w * y * y), np.sum(w * Ax * Ax)])


def gains(all_stats):
    g = [1.0]
    for s in all_stats[1:]:
        if s[1] <= 0.0:
            raise ValueError("zero-norm weighted data for camera >= 2")
        g.append(s[0] / s[1])
    return np.array(g)


def cost(x, Ax, ys, ws, gam, beta, nu):
    c = 0.0
    for Axc, y, w, g in zip(Ax, ys, ws, gam):
        r = np.asarray(Axc, np.float64).ravel() - g * np.asarray(y, np.float64).ravel()
        c += 0.5 * np.sum(np.asarray(w, np.float64).ravel() * r * r)
    return c + nu * np.sum(x) + reg_value(x, beta)


def gradient(x, ops, ys, ws, beta, nu, return_parts=False):
    """Profiled PWLS gradient at x (ops: objects with forward/adjoint on flat arrays)."""
    x = np.asarray(x, np.float64)
    Ax = [op.forward(x) for op in ops]
    st = [stats(a, y, w) for a, y, w in zip(Ax, ys, ws)]
    gam = gains(st)
    g = np.zeros(x.size)
    for op, a, y, w, gc in zip(ops, Ax, ys, ws, gam):
        r = np.asarray(w, np.float64).ravel() * (a - gc * np.asarray(y, np.float64).ravel())
        g += op.adjoint(r)
    g = g.reshape(x.shape) + reg_grad(x, beta) + nu
    if return_parts:
        return g, Ax, st, gam
    return g


def profiled_cost(x, ops, ys, ws, beta, nu):
    x = np.asarray(x, np.float64)
    Ax = [op.forward(x) for op in ops]
    gam = gains([stats(a, y, w) for a, y, w in zip(Ax, ys, ws)])
    return cost(x, Ax, ys, ws, gam, beta, nu)


def majoriser(ops, ws, beta, shape):
    ones = np.ones(shape)
    d = np.zeros(int(np.prod(shape)))
    for op, w in zip(ops, ws):
        d += op.adjoint(np.asarray(w, np.float64).ravel() * op.forward(ones))
    # floor uncovered voxels (no camera sees them, beta = 0) so the step stays finite
    return np.maximum(d.reshape(shape) + MAJORISER_C * beta, 1e-12)


def subset_views(k_s, k_t, n_subsets, m):
    """View subset S_m of the angular plane (sec,subset P:383-386): the K = k_s k_t views ordered
    lexicographically with k_s varying fastest (reading R5: k = k_t k_s_count + k_s, the storage order of
    P:85-87), every n_subsets-th one starting at m.  Returned as (k_s, k_t) pairs."""
    return [(k % k_s, k // k_s) for k in range(k_s * k_t) if k % n_subsets == m]


def gradient_subset(x, ops, ys, ws, beta, nu, n_subsets, m):
    """View-subset approximation of the profiled gradient, eqn,subset in reading Z19:
    y^_c = (K_c/|S|) sum_{k in S} A_ck x;  gains from y^_c (eqn,optimal,gain with A_c x -> y^_c);
    g = sum_c (K_c/|S|) sum_{k in S} A_ck^T W_c (y^_c - g_c y_c) + grad R + nu."""
    x = np.asarray(x, np.float64)
    Ax, sc, views = [], [], []
    for op in ops:
        cam = op.camera
        v = subset_views(cam.ks, cam.kt, n_subsets, m)
        s = cam.ks * cam.kt / len(v)
        views.append(v)
        sc.append(s)
        Ax.append(s * op.forward(x, v))
    gam = gains([stats(a, y, w) for a, y, w in zip(Ax, ys, ws)])
    g = np.zeros(x.size)
    for op, a, y, w, gc, s, v in zip(ops, Ax, ys, ws, gam, sc, views):
        r = np.asarray(w, np.float64).ravel() * (a - gc * np.asarray(y, np.float64).ravel())
        g += s * op.adjoint(r, v)
    return g.reshape(x.shape) + reg_grad(x, beta) + nu


def fista(ops, ys, ws, beta, nu, shape, iters, d=None, callback=None, n_subsets=1):
    if d is None:
        d = majoriser(ops, ws, beta, shape)
    x = np.zeros(shape)
    z = np.zeros(shape)
    t = 1.0
    for it in range(iters):
        # n_subsets > 1: ordered-subsets acceleration, subset it mod n_subsets at iteration it (sec,subset)
        if n_subsets > 1:
            g = gradient_subset(z, ops, ys, ws, beta, nu, n_subsets, it % n_subsets)
        else:
            g = gradient(z, ops, ys, ws, beta, nu)
        x_new = np.maximum(0.0, z - g / d)
        t_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        z = x_new + ((t - 1.0) / t_new) * (x_new - x)
        x, t = x_new, t_new
        if callback is not None:
            callback(it, x)
    return x
