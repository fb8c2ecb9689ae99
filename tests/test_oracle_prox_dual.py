"""Pin of the oracle's prox-regularised pair solve (reading #2, prox_eps > 0) against
strong duality, an independent route to the same unique minimiser.

The primal  min_y 1/2||K^T y + b||^2 + eps/2||y - y_prev||^2  s.t. y >= 0, kappa^T y = 1
(Eq. 19, plus the proximal term) has the concave dual over w in R^{d+1}
    g(w) = w.b - 1/2||w||^2 + min_{y in Y} [(K w).y + eps/2||y - y_prev||^2],
maximised at w* = u* = K^T y* + b, with y* = Pi_Y(y_prev - K w*/eps).  Here the dual is
maximised by plain projected fixed-point-free means (scipy BFGS on -g, then a polish
by the exact piecewise-linear solve of u(w) = w on the final support), and the primal
y recovered by the Euclidean projection -- no Lemke, no LCP.  The oracle's dense Lemke
must return the same y.  (NEXT f4's GPU solver uses a semismooth Newton on the same
dual; this test shares no code with it.)"""
import numpy as np
import pytest
from scipy.optimize import minimize

from test_oracle_lcp import random_pair


def proj_Y(c, kappa):
    """Euclidean projection onto {y >= 0, kappa^T y = 1}, kappa >= 0 with some kappa_k > 0:
    entries with kappa_k = 0 are clipped at 0; the others are max(0, c_k - tau kappa_k),
    tau the root of the decreasing sum kappa^T y(tau) = 1 (found by sorting breakpoints)."""
    y = np.maximum(c, 0.0)
    lam = kappa > 0
    cl, kl = c[lam], kappa[lam]
    order = np.argsort(-cl / kl)  # breakpoints tau_k = c_k / kappa_k, descending
    for m in range(1, len(order) + 1):
        S = order[:m]
        tau = (kl[S] @ cl[S] - 1.0) / (kl[S] @ kl[S])
        nxt = cl[order[m]] / kl[order[m]] if m < len(order) else -np.inf
        if nxt <= tau:
            break
    y[lam] = np.maximum(cl - tau * kl, 0.0)
    return y


def dual_solve(K, b, kappa, eps, yp):
    def neg_g(w):
        y = proj_Y(yp - K @ w / eps, kappa)
        u = K.T @ y + b
        g = w @ b - 0.5 * w @ w + (K @ w) @ y + 0.5 * eps * np.sum((y - yp) ** 2)
        return -g, -(u - w)  # Danskin: grad g = u(w) - w
    w = minimize(neg_g, K.T @ yp + b, jac=True, method="BFGS", options={"gtol": 1e-13, "maxiter": 5000}).x
    # polish: on the support S of y(w), u(w) = w is linear in w; solve it exactly
    for _ in range(5):
        c = yp - K @ w / eps
        y = proj_Y(c, kappa)
        S = y > 0
        F = S & (kappa > 0)
        Jm = np.diag(S.astype(float))
        if F.any():
            kf = np.where(F, kappa, 0.0)
            Jm -= np.outer(kf, kf) / (kf @ kf)
        # u(w) = K^T J (yp - K w / eps) + K^T y0 + b, with y0 the affine offset of the projection
        y0 = y - Jm @ c
        A = np.eye(len(w)) + K.T @ Jm @ K / eps
        w_new = np.linalg.solve(A, K.T @ Jm @ yp + K.T @ y0 + b)
        if np.array_equal(proj_Y(yp - K @ w_new / eps, kappa) > 0, S):
            w = w_new
            break
        w = w_new
    return proj_Y(yp - K @ w / eps, kappa)


@pytest.mark.parametrize("eps", [1e-3, 1e-2, 1e-1, 1.0])
def test_prox_pair_solve_equals_dual(orc, eps):
    rng = np.random.default_rng(61)
    worst = 0.0
    for trial in range(150):
        Ar, br, Co, do, R, rho = random_pair(rng)
        n = len(br) + len(do) + 1
        yp = rng.uniform(0, 0.5, n) * (rng.uniform(size=n) < 0.6)
        zeta, xi = rng.normal(0, 0.5), rng.normal(0, 0.5, 2)
        y, st, *_ = orc.pair_solve(Ar, br, Co, do, R, rho, zeta, xi, prox_eps=eps, y_prev=yp)
        assert st == 0
        K, bvec, *_ = orc.pair_lcp(Ar, br, Co, do, R, rho, zeta, xi)
        kappa = np.r_[br, np.zeros(len(do) + 1)]
        yd = dual_solve(K, bvec, kappa, eps, yp)
        err = np.abs(y - yd).max() / max(1.0, np.abs(yd).max())
        worst = max(worst, err)
    # both exact up to rounding; condition 1 + ||K||^2/eps <= 1 + 25/eps for these pairs
    assert worst <= max(1e-10, 1e-14 * (1 + 25.0 / eps)), worst
