/* orc.c -- plain, slow, sequential FP64 CPU ORACLE of the ADMM hot path of
 * arXiv 2406.07048 ("GPU-accelerated collision avoidance ... scale-based
 * collision detection ... ADMM").
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py; never by the product path.
 * Shares no code with paper_2406_07048_b200/ or include/.
 *
 * Every function follows the paper's equations in the paper's order; citations
 * are PAPER.md line numbers (P:n).  Where the paper is silent the DESIGN.md
 * reading number is given (reading #k).  Compile with -ffp-contract=off: every
 * fused multiply-add below is an explicit fma() (reading #18, FMA policy).
 *
 * Pins (tests/test_oracle_*.py) -- what ties each function to something other
 * than itself:
 *   orc_scale_lp       closed-form boxes, scipy HiGHS primal+dual LP, SAT
 *                      disjointness, SPEC examples, metamorphic scalings
 *   orc_pair_lcp       KKT (Eq. 22) certificate; elimination round trip;
 *                      projection definition of u*; slab closed form
 *   orc_lemke          SPEC LCP examples, 2^n complementary-basis enumeration
 *   orc_primal_step    zero-obstacle step == dense KKT LQ solve (numpy);
 *                      GN gradient/Hessian vs finite differences
 *   orc_multiplier_update  identity zeta+ - zeta = T (Eq. 10) recomputed in numpy
 *   r_pri / r_dual     Eq. 18's sums recomputed in numpy from consecutive iterates
 *                      (sum ||zeta+ - zeta||^2 + ||xi+ - xi||^2, sum ||lambda+ - lambda||^2
 *                      + ||mu+ - mu||^2, gamma excluded), tests/test_oracle_stop.py
 *   orc_check_stopping SPEC S:526-528 examples ('<=' boundary), monotone in eps
 *   orc_admm_solve     = the first k of the fixed-K history meeting Eq. 18, per scene;
 *                      a frozen scene's iterate = the K-iteration run stopped there
 *   orc_admm_iterate_mt  bitwise = orc_admm_iterate (scene fan-out)
 *   box block (f1)     zero-obstacle fixed point == box-constrained LQ optimum
 *                      (scipy lsq_linear; KKT certificate with state bounds);
 *                      infinite bounds == no bounds, bitwise
 *   whole ADMM         translation equivariance, obstacle-permutation invariance
 *   Lemke's choice among non-unique QP minimisers: parity unpinned (only the
 *   rules L1-L7 of DESIGN.md reading #4 define it).
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "orc.h"

#define MAXN 64
#define MAXD 3

static double dmax(double a, double b) { return a > b ? a : b; }

/* ---------------------------------------------------------------------------
 * Pose R(s_t), rho(s_t)   (reading #9)
 * ------------------------------------------------------------------------- */
void orc_pose(int model, const int* idx, int d, const double* s, double* R, double* rho) {
  for (int a = 0; a < d; ++a)
    for (int c = 0; c < d; ++c) R[a * d + c] = (a == c) ? 1.0 : 0.0;
  for (int a = 0; a < d; ++a) rho[a] = s[idx[a]];
  if (model == ORC_POSE_SE2) {
    double th = s[idx[2]];
    double c = cos(th), sn = sin(th);
    R[0] = c; R[1] = -sn;
    R[2] = sn; R[3] = c;
  } else if (model == ORC_POSE_TRANS_YAW) {
    double ps = s[idx[3]];
    double c = cos(ps), sn = sin(ps);
    R[0] = c; R[1] = -sn; R[2] = 0.0;
    R[3] = sn; R[4] = c;  R[5] = 0.0;
    R[6] = 0.0; R[7] = 0.0; R[8] = 1.0;
  }
}

/* Pair (t, obstacle j) with a moving obstacle (NEXT f3): by translation invariance the
 * robot posed at rho meets O_j + t*step_j exactly as the robot posed at
 * rho - t*step_j meets O_j, so every pair computation takes this shifted origin. */
static void obstacle_frame(const orc_problem* P, int b, int j, int t, const double* rho, double* rho_j) {
  for (int a = 0; a < P->dim; ++a) rho_j[a] = rho[a];
  if (!P->obs_step) return;
  const double* st = P->obs_step + ((long long)b * P->n_obs + j) * P->dim;
  for (int a = 0; a < P->dim; ++a) rho_j[a] = rho[a] - (double)t * st[a];
}

/* ---------------------------------------------------------------------------
 * Eq. 3: alpha* = min alpha s.t. A x <= b alpha, C x <= d, with the
 * robot posed: x = R^T (y - rho) in world coordinates y, so the robot
 * rows read (R a_k)^T y - b_k alpha <= (R a_k)^T rho.
 * Plain brute force over vertices: the LP in z = (y, alpha) has d+1 variables and
 * a pointed feasible region (bounded obstacle), so its optimum is attained at a
 * vertex = a nonsingular (d+1)-subset of rows, solved exactly and kept if
 * feasible.  Returns 0, or -1 if no feasible vertex (empty obstacle).
 * ------------------------------------------------------------------------- */
static int solve_small(int m, double* A, double* bb, double* x) {
  /* Gaussian elimination with partial pivoting on an m x m system (m <= 4). */
  double scale = 0.0;
  for (int i = 0; i < m * m; ++i) scale = dmax(scale, fabs(A[i]));
  if (scale == 0.0) return -1;
  for (int k = 0; k < m; ++k) {
    int piv = k;
    for (int i = k + 1; i < m; ++i)
      if (fabs(A[i * m + k]) > fabs(A[piv * m + k])) piv = i;
    if (fabs(A[piv * m + k]) < 1e-12 * scale) return -1;
    if (piv != k) {
      for (int c = 0; c < m; ++c) {
        double t = A[k * m + c]; A[k * m + c] = A[piv * m + c]; A[piv * m + c] = t;
      }
      double t = bb[k]; bb[k] = bb[piv]; bb[piv] = t;
    }
    for (int i = k + 1; i < m; ++i) {
      double f = A[i * m + k] / A[k * m + k];
      for (int c = k; c < m; ++c) A[i * m + c] -= f * A[k * m + c];
      bb[i] -= f * bb[k];
    }
  }
  for (int i = m - 1; i >= 0; --i) {
    double acc = bb[i];
    for (int c = i + 1; c < m; ++c) acc -= A[i * m + c] * x[c];
    x[i] = acc / A[i * m + i];
  }
  return 0;
}

int orc_scale_lp(int d, int nr, const double* A, const double* b, const double* R,
                 const double* rho, int no, const double* C, const double* dv,
                 double* alpha_out, double* y_out) {
  int m = nr + no, nv = d + 1;
  double G[MAXN][MAXD + 1], h[MAXN];
  for (int k = 0; k < nr; ++k) {
    double ra[MAXD];
    for (int a = 0; a < d; ++a) {
      ra[a] = 0.0;
      for (int c = 0; c < d; ++c) ra[a] += R[a * d + c] * A[k * d + c];
    }
    h[k] = 0.0;
    for (int a = 0; a < d; ++a) { G[k][a] = ra[a]; h[k] += ra[a] * rho[a]; }
    G[k][d] = -b[k];
  }
  for (int l = 0; l < no; ++l) {
    for (int a = 0; a < d; ++a) G[nr + l][a] = C[l * d + a];
    G[nr + l][d] = 0.0;
    h[nr + l] = dv[l];
  }
  int sub[MAXD + 1];
  for (int i = 0; i < nv; ++i) sub[i] = i;
  double best = INFINITY;
  double besty[MAXD + 1] = {0};
  if (m < nv) return -1;
  for (;;) {
    double Ms[16], rhs[4], z[4];
    for (int r = 0; r < nv; ++r) {
      for (int c = 0; c < nv; ++c) Ms[r * nv + c] = G[sub[r]][c];
      rhs[r] = h[sub[r]];
    }
    if (solve_small(nv, Ms, rhs, z) == 0) {
      int feas = 1;
      for (int i = 0; i < m && feas; ++i) {
        double lhs = 0.0, mag = fabs(h[i]);
        for (int c = 0; c < nv; ++c) { lhs += G[i][c] * z[c]; mag += fabs(G[i][c] * z[c]); }
        if (lhs - h[i] > 1e-9 * (1.0 + mag)) feas = 0;
      }
      if (feas && z[d] < best) {
        best = z[d];
        for (int c = 0; c < nv; ++c) besty[c] = z[c];
      }
    }
    /* next combination (lexicographic) */
    int i = nv - 1;
    while (i >= 0 && sub[i] == m - nv + i) --i;
    if (i < 0) break;
    ++sub[i];
    for (int j = i + 1; j < nv; ++j) sub[j] = sub[j - 1] + 1;
  }
  if (!(best < INFINITY)) return -1;
  *alpha_out = best;
  if (y_out)
    for (int c = 0; c < d; ++c) y_out[c] = besty[c];
  return 0;
}

/* ---------------------------------------------------------------------------
 * Eq. 19: per-pair QP  min 1/2 ||K^T y + b||^2, kappa^T y = eta, y >= 0
 *   rows of K: lambda_k: (0, a_k^T); mu_l: (d_l - c_l^T rho, c_l^T R); gamma: (1, 0)
 *   b = (1 + zeta, xi), kappa = (b_i, 0, 0), eta = 1.
 * K is n x (d+1), row-major.  c_l^T rho and c_l^T R accumulate left to right with
 * fma (FMA policy, reading #18).
 * ------------------------------------------------------------------------- */
void orc_build_K(int d, int nr, const double* A, int no, const double* C, const double* dv,
                 const double* R, const double* rho, double* K) {
  int w = d + 1;
  for (int k = 0; k < nr; ++k) {
    K[k * w] = 0.0;
    for (int a = 0; a < d; ++a) K[k * w + 1 + a] = A[k * d + a];
  }
  for (int l = 0; l < no; ++l) {
    double* row = K + (nr + l) * w;
    double cr = 0.0;
    for (int a = 0; a < d; ++a) cr = fma(C[l * d + a], rho[a], cr);
    row[0] = dv[l] - cr;
    for (int m = 0; m < d; ++m) {
      double acc = 0.0;
      for (int a = 0; a < d; ++a) acc = fma(C[l * d + a], R[a * d + m], acc);
      row[1 + m] = acc;
    }
  }
  double* g = K + (nr + no) * w;
  g[0] = 1.0;
  for (int a = 0; a < d; ++a) g[1 + a] = 0.0;
}

/* index e of the eliminated component: argmax_k b_k, lowest k on ties (reading #3) */
int orc_elim_index(int nr, const double* b) {
  int e = 0;
  for (int k = 1; k < nr; ++k)
    if (b[k] > b[e]) e = k;
  return e;
}

/* Eqs. 20-21 then Eqs. 24-25.
 * U = all indices but e, in original order.
 *   ratio_r = kappa_r / b_e;  Ktil_r = K_r - ratio_r K_e  (fma per column)
 *   btil    = b + K_e / b_e;  kaptil = ratio_U;  etatil = 1 / b_e
 *   M = [[Ktil Ktil^T, kaptil], [-kaptil^T, 0]],  q = [Ktil btil; etatil]
 * Outputs M (n x n) and q (n), n = nr + no + 1.  Also returns K (n x (d+1)),
 * bvec (d+1) and e for the caller. */
void orc_pair_lcp(int d, int nr, const double* A, const double* b, int no, const double* C,
                  const double* dv, const double* R, const double* rho, double zeta,
                  const double* xi, double prox_eps, const double* y_prev, double* K, double* bvec,
                  int* e_out, double* M, double* q) {
  int n = nr + no + 1, w = d + 1;
  orc_build_K(d, nr, A, no, C, dv, R, rho, K);
  bvec[0] = 1.0 + zeta;
  for (int a = 0; a < d; ++a) bvec[1 + a] = xi[a];
  int e = orc_elim_index(nr, b);
  *e_out = e;
  double be = b[e];
  double Kt[MAXN][MAXD + 1], kt[MAXN], bt[MAXD + 1];
  int r = 0;
  for (int k = 0; k < n; ++k) {
    if (k == e) continue;
    double kappa = (k < nr) ? b[k] : 0.0;
    double ratio = kappa / be;
    for (int c = 0; c < w; ++c) Kt[r][c] = fma(-ratio, K[e * w + c], K[k * w + c]);
    kt[r] = ratio;
    ++r;
  }
  for (int c = 0; c < w; ++c) bt[c] = bvec[c] + K[e * w + c] / be;
  double etat = 1.0 / be;
  for (int i = 0; i < n - 1; ++i) {
    for (int j = 0; j < n - 1; ++j) {
      double acc = 0.0;
      for (int c = 0; c < w; ++c) acc = fma(Kt[i][c], Kt[j][c], acc);
      M[i * n + j] = acc;
    }
    M[i * n + (n - 1)] = kt[i];
    M[(n - 1) * n + i] = -kt[i];
    double acc = 0.0;
    for (int c = 0; c < w; ++c) acc = fma(Kt[i][c], bt[c], acc);
    q[i] = acc;
  }
  if (prox_eps > 0.0) {
    /* reading #2 (prox_eps > 0 only): add (eps/2)||y - y_prev||^2 to Eq. 19a, i.e.
     * K' = [K, sqrt(eps) I], b' = [b; -sqrt(eps) y_prev] pushed through Eqs. 20-25:
     *   M_UU += eps (I + kaptil kaptil^T),  q_U -= eps (y_prev_U + kaptil (etatil - y_prev_e)) */
    int ui[MAXN];
    r = 0;
    for (int k = 0; k < n; ++k)
      if (k != e) ui[r++] = k;
    for (int i = 0; i < n - 1; ++i) {
      for (int j = 0; j < n - 1; ++j) {
        double t = fma(kt[i], kt[j], (i == j) ? 1.0 : 0.0);
        M[i * n + j] = fma(prox_eps, t, M[i * n + j]);
      }
      double t = fma(kt[i], etat - y_prev[e], y_prev[ui[i]]);
      q[i] = fma(-prox_eps, t, q[i]);
    }
  }
  M[(n - 1) * n + (n - 1)] = 0.0;
  q[n - 1] = etat;
}

/* ---------------------------------------------------------------------------
 * Lemke's complementary pivoting (rules L1-L7 = reading #4).
 * Textbook full tableau [ I | -M | -1 | q ] over (w, z, z0, rhs); a row means
 * x_B(i) + sum_j T[i][j] x_j = rhs_i.  Columns: w_j = j, z_j = n+j, z0 = 2n,
 * rhs = 2n+1.  Pivot: row r scaled by inv = 1/T[r][c] (one division), other rows
 * T[i][j] = fma(-T[i][c], T[r][j], T[i][j]); the entering column is then set to
 * the unit vector.  Returns ORC_OK / ORC_RAY / ORC_ITER_LIMIT.
 * z_out (n), basis_out (n labels, may be NULL), pivots_out (count incl. the z0 pivot).
 * ------------------------------------------------------------------------- */
static void lemke_pivot(double* T, int n, int W, int r, int c) {
  double inv = 1.0 / T[r * W + c];
  for (int j = 0; j < W; ++j)
    if (j != c) T[r * W + j] = T[r * W + j] * inv;
  T[r * W + c] = 1.0;
  for (int i = 0; i < n; ++i) {
    if (i == r) continue;
    double f = T[i * W + c];
    for (int j = 0; j < W; ++j)
      if (j != c) T[i * W + j] = fma(-f, T[r * W + j], T[i * W + j]);
    T[i * W + c] = 0.0;
  }
}

int orc_lemke(int n, const double* M, const double* q, double pivot_tol, double tie_tol,
              int max_pivots, double* z_out, int* basis_out, int* pivots_out) {
  int W = 2 * n + 2, Z0 = 2 * n, RHS = 2 * n + 1;
  double* T = (double*)calloc((size_t)n * W, sizeof(double));
  int basis[MAXN];
  int status = ORC_OK, pivots = 0;
  for (int i = 0; i < n; ++i) {
    T[i * W + i] = 1.0;
    for (int j = 0; j < n; ++j) T[i * W + n + j] = -M[i * n + j];
    T[i * W + Z0] = -1.0;
    T[i * W + RHS] = q[i];
    basis[i] = i;
  }
  double qmin = q[0];
  for (int i = 1; i < n; ++i)
    if (q[i] < qmin) qmin = q[i];
  if (qmin < 0.0) {
    /* L2: z0 enters; leaving row = argmin q, ties -> largest index */
    double tol = tie_tol * dmax(1.0, fabs(qmin));
    int r = -1;
    for (int i = 0; i < n; ++i)
      if (q[i] <= qmin + tol) r = i;
    int leaving = basis[r];
    lemke_pivot(T, n, W, r, Z0);
    basis[r] = Z0;
    ++pivots;
    int entering = leaving + n; /* L4: complement of w_i is z_i */
    for (;;) {
      if (pivots >= max_pivots) { status = ORC_ITER_LIMIT; break; } /* L7 */
      int col = entering;
      /* L5: ratio test */
      double cmax = 0.0;
      for (int i = 0; i < n; ++i) cmax = dmax(cmax, fabs(T[i * W + col]));
      double thr = pivot_tol * dmax(1.0, cmax);
      int tie[MAXN], nt = 0;
      double theta[MAXN], thmin = INFINITY;
      for (int i = 0; i < n; ++i) {
        double ci = T[i * W + col];
        if (ci > thr) {
          theta[i] = dmax(T[i * W + RHS], 0.0) / ci;
          if (theta[i] < thmin) thmin = theta[i];
        } else {
          theta[i] = INFINITY;
        }
      }
      if (!(thmin < INFINITY)) { status = ORC_RAY; break; }
      double ttol = thmin + tie_tol * dmax(1.0, thmin);
      for (int i = 0; i < n; ++i)
        if (theta[i] <= ttol) tie[nt++] = i;
      int r2 = -1;
      for (int k = 0; k < nt; ++k)
        if (basis[tie[k]] == Z0) r2 = tie[k];
      if (r2 < 0) {
        /* lexicographic rule over the w columns (= B^{-1}) */
        for (int j = 0; j < n && nt > 1; ++j) {
          double v[MAXN], vmin = INFINITY;
          for (int k = 0; k < nt; ++k) {
            v[k] = T[tie[k] * W + j] / T[tie[k] * W + col];
            if (v[k] < vmin) vmin = v[k];
          }
          double vtol = vmin + tie_tol * dmax(1.0, fabs(vmin));
          int m2 = 0;
          for (int k = 0; k < nt; ++k)
            if (v[k] <= vtol) tie[m2++] = tie[k];
          nt = m2;
        }
        r2 = tie[0]; /* smallest row index among the survivors */
      }
      int leaving2 = basis[r2];
      lemke_pivot(T, n, W, r2, col);
      basis[r2] = col;
      ++pivots;
      if (leaving2 == Z0) break; /* L6 */
      entering = (leaving2 < n) ? leaving2 + n : leaving2 - n;
    }
  }
  for (int j = 0; j < n; ++j) z_out[j] = 0.0;
  for (int i = 0; i < n; ++i)
    if (basis[i] >= n && basis[i] < 2 * n) z_out[basis[i] - n] = T[i * W + RHS];
  if (basis_out)
    for (int i = 0; i < n; ++i) basis_out[i] = basis[i];
  *pivots_out = pivots;
  free(T);
  return status;
}

/* ---------------------------------------------------------------------------
 * One pair: Eq. 19 -> Eqs. 20-21 -> Eq. 24 -> Lemke -> recovery:
 *   y_U = z[0..n-2], phi = z[n-1], y_e = (1 - sum_{k != e} b_k lambda_k) / b_e.
 * Status ORC_NEG_YE if y_e < -1e-6.  y_out has n entries.
 * ------------------------------------------------------------------------- */
int orc_pair_solve(int d, int nr, const double* A, const double* b, int no, const double* C,
                   const double* dv, const double* R, const double* rho, double zeta,
                   const double* xi, double prox_eps, const double* y_prev, double pivot_tol,
                   double tie_tol, int max_pivot_factor, double* y_out, int* pivots_out,
                   int* basis_out) {
  int n = nr + no + 1;
  double K[MAXN * (MAXD + 1)], bvec[MAXD + 1], M[MAXN * MAXN], q[MAXN], z[MAXN];
  int e;
  orc_pair_lcp(d, nr, A, b, no, C, dv, R, rho, zeta, xi, prox_eps, y_prev, K, bvec, &e, M, q);
  int st = orc_lemke(n, M, q, pivot_tol, tie_tol, max_pivot_factor * n, z, basis_out, pivots_out);
  int r = 0;
  for (int k = 0; k < n; ++k) {
    if (k == e) continue;
    y_out[k] = z[r++];
  }
  double acc = 0.0;
  for (int k = 0; k < nr; ++k)
    if (k != e) acc = fma(b[k], y_out[k], acc);
  y_out[e] = (1.0 - acc) / b[e];
  if (st == ORC_OK && y_out[e] < -1e-6) st = ORC_NEG_YE;
  return st;
}

/* ---------------------------------------------------------------------------
 * Problem helpers
 * ------------------------------------------------------------------------- */
static long long n_pairs(const orc_problem* P) {
  return (long long)P->n_scenes * P->horizon * P->n_parts * P->n_obs;
}

/* 1 if obstacle (b, j) is in the (i, j, t) table (sensing, NEXT f3) */
static int sensed(const orc_problem* P, int b, int j) {
  return !P->sensed || P->sensed[(long long)b * P->n_obs + j];
}

/* Part i about its scaling centre o_i (reading #22; NEXT f3): b~ = b - A o_i and the
 * pair origin rho_i = rho + R o_i.  Without centres b~ = b, rho_i = rho. */
static void part_frame(const orc_problem* P, int i, const double* R, const double* rho, double* bt,
                       double* rho_i) {
  int d = P->dim, r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
  const double* o = P->part_ctr ? P->part_ctr + (long long)i * d : NULL;
  for (int k = 0; k < nr; ++k) {
    double v = P->part_b[r0 + k];
    if (o)
      for (int a = 0; a < d; ++a) v -= P->part_A[(long long)(r0 + k) * d + a] * o[a];
    bt[k] = v;
  }
  for (int a = 0; a < d; ++a) {
    double v = rho[a];
    if (o)
      for (int c = 0; c < d; ++c) v += R[a * d + c] * o[c];
    rho_i[a] = v;
  }
}

/* Sensing (NEXT f3): obstacle (b, j) is sensed iff it meets the
 * axis-aligned box rho(s0_b) + [-half, half] (world frame) -- i.e. iff the scale
 * factor alpha* (Eq. 3) of that box as a "robot part" against the obstacle is <= 1
 * (1e-9 slack: touching counts as sensed).  Static obstacle positions (t = 0). */
void orc_sense(const orc_problem* P, const double* half, unsigned char* out) {
  int d = P->dim;
  double A[6 * MAXD], bb[6], R[9], rho[3];
  for (int a = 0; a < d; ++a) {
    for (int c = 0; c < d; ++c) {
      A[(2 * a) * d + c] = (a == c) ? 1.0 : 0.0;
      A[(2 * a + 1) * d + c] = (a == c) ? -1.0 : 0.0;
    }
    bb[2 * a] = half[a];
    bb[2 * a + 1] = half[a];
  }
  for (int b = 0; b < P->n_scenes; ++b) {
    orc_pose(P->pose_model, P->pose_idx, d, P->s0 + (long long)b * P->n_state, R, rho);
    for (int a = 0; a < d * d; ++a) R[a] = (a % (d + 1) == 0) ? 1.0 : 0.0; /* world-aligned box */
    for (int j = 0; j < P->n_obs; ++j) {
      int o = b * P->n_obs + j, l0 = P->obs_off[o], no = P->obs_off[o + 1] - l0;
      double alpha;
      int rc = orc_scale_lp(d, 2 * d, A, bb, R, rho, no, P->obs_C + (long long)l0 * d, P->obs_d + l0, &alpha, NULL);
      out[o] = (rc == 0 && alpha <= 1.0 + 1e-9) ? 1 : 0;
    }
  }
}

static const double* dyn_ptr(const orc_problem* P, const double* base, int b, int t, int blk) {
  long long nt = P->dyn_per_time ? P->horizon : 1;
  long long idx = (P->dyn_per_scene ? (long long)b * nt : 0) + (P->dyn_per_time ? t : 0);
  return base + idx * blk;
}

/* dyn_model 1: the unicycle linearised at (sbar, ubar) (f is linear in u, so c does
 * not depend on ubar):  A = I + dt d(v cos th, v sin th, 0, 0)/ds,  B = dt [e_3 | e_2]
 * for u = (a, om),  c = sbar + dt (v cos th, v sin th, 0, 0) - A sbar. */
static void unicycle_ltv(double dt, const double* sb, double* A, double* B, double* c) {
  const double th = sb[2], v = sb[3], cs = cos(th), sn = sin(th);
  for (int a = 0; a < 16; ++a) A[a] = (a % 5 == 0) ? 1.0 : 0.0;
  A[0 * 4 + 2] += -dt * v * sn;
  A[0 * 4 + 3] += dt * cs;
  A[1 * 4 + 2] += dt * v * cs;
  A[1 * 4 + 3] += dt * sn;
  for (int a = 0; a < 8; ++a) B[a] = 0.0;
  B[2 * 2 + 1] = dt;
  B[3 * 2 + 0] = dt;
  const double f[4] = {dt * v * cs, dt * v * sn, 0.0, 0.0};
  for (int a = 0; a < 4; ++a) {
    double acc = 0.0;
    for (int k = 0; k < 4; ++k) acc += A[a * 4 + k] * sb[k];
    c[a] = sb[a] + f[a] - acc;
  }
}

static int n_pose_coords(const orc_problem* P) {
  return P->pose_model == ORC_POSE_TRANSLATION ? P->dim : P->dim + 1;
}

/* O1 initial iterate (reading #11): s_0 fixed, s_t = s_ref_t, u = 0,
 * lambda = 1/sum(b_i) 1 (so b_i^T lambda = 1), mu = 0, gamma = 0, zeta = xi = 0. */
/* ---------------------------------------------------------------------------
 * Box block of IC_0 (Eq. 13c-d; reading #7, NEXT f1).  The boxes are
 * handled by one more ADMM block: a copy w of every bounded state (t = 1..N) and
 * control, the consensus constraint x = w with scaled multiplier l and penalty
 * rho_b.  The primal step (Eq. 16) gains (rho_b/2) ||x - w^k + l^k||^2 and is
 * followed by  w^{k+1} = Pi_box(x^{k+1} + l^k),  l^{k+1} = l^k + x^{k+1} - w^{k+1}
 * (the scaled-form ADMM of P:283-320's reference [boyd2011distributed]).
 * ------------------------------------------------------------------------- */
static int has_box(const orc_problem* P) { return P->s_min || P->s_max || P->u_min || P->u_max; }
static double box_lo(const double* v, int a) { return v ? v[a] : -INFINITY; }
static double box_hi(const double* v, int a) { return v ? v[a] : INFINITY; }
/* 1 if component a has a finite bound on either side */
static int box_on(const double* lo, const double* hi, int a) {
  return box_lo(lo, a) > -INFINITY || box_hi(hi, a) < INFINITY;
}
/* projection onto [lo, hi] */
static double clip(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* w = Pi_box(s, u), l = 0, boxres = 0 (after an initial or user-set iterate) */
void orc_reset_box(const orc_problem* P, orc_iterate* I) {
  if (!has_box(P)) return;
  int B = P->n_scenes, N = P->horizon, ns = P->n_state, nu = P->n_ctrl;
  for (int b = 0; b < B; ++b) {
    for (int t = 0; t <= N; ++t)
      for (int a = 0; a < ns; ++a) {
        long long k = ((long long)b * (N + 1) + t) * ns + a;
        I->ws[k] = clip(I->s[k], box_lo(P->s_min, a), box_hi(P->s_max, a));
        I->ls[k] = 0.0;
      }
    for (int t = 0; t < N; ++t)
      for (int a = 0; a < nu; ++a) {
        long long k = ((long long)b * N + t) * nu + a;
        I->wu[k] = clip(I->u[k], box_lo(P->u_min, a), box_hi(P->u_max, a));
        I->lu[k] = 0.0;
      }
    I->boxres[b] = 0.0;
  }
}

/* Cold start (reading #11): states from the reference (clipped to the box),
 * controls zero (clipped), certificates lambda = 1/sum(b_i), mu = gamma = 0, zeta = xi = 0. */
void orc_init_iterate(const orc_problem* P, orc_iterate* I) {
  int B = P->n_scenes, N = P->horizon, ns = P->n_state, nu = P->n_ctrl, d = P->dim;
  for (int b = 0; b < B; ++b) {
    for (int t = 0; t <= N; ++t)
      for (int a = 0; a < ns; ++a)
        I->s[((long long)b * (N + 1) + t) * ns + a] =
            (t == 0) ? P->s0[b * ns + a]
                     : clip(P->s_ref[((long long)b * (N + 1) + t) * ns + a], box_lo(P->s_min, a),
                            box_hi(P->s_max, a));
    for (int t = 0; t < N; ++t)
      for (int a = 0; a < nu; ++a)
        I->u[((long long)b * N + t) * nu + a] = clip(0.0, box_lo(P->u_min, a), box_hi(P->u_max, a));
  }
  orc_reset_box(P, I);
  long long np = n_pairs(P);
  for (long long p = 0; p < np; ++p) {
    int i = (int)((p / P->n_obs) % P->n_parts);
    int r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
    double sb = 0.0;
    double bt[MAXN], R0[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z0[3] = {0, 0, 0}, r_[3];
    part_frame(P, i, R0, z0, bt, r_);
    for (int k = 0; k < nr; ++k) sb += bt[k];
    for (int k = 0; k < P->ny; ++k) I->y[p * P->ny + k] = (k < nr) ? 1.0 / sb : 0.0;
    I->zeta[p] = 0.0;
    for (int a = 0; a < d; ++a) I->xi[p * d + a] = 0.0;
    if (I->pivots) I->pivots[p] = 0;
    if (I->status) I->status[p] = 0;
  }
}

/* decode p -> (b, t in 1..N, i, j) */
static void decode(const orc_problem* P, long long p, int* b, int* t, int* i, int* j) {
  *j = (int)(p % P->n_obs);
  long long r = p / P->n_obs;
  *i = (int)(r % P->n_parts);
  r /= P->n_parts;
  *t = (int)(r % P->horizon) + 1;
  *b = (int)(r / P->horizon);
}

/* ---------------------------------------------------------------------------
 * ADMM step 1, Eq. 15 via Eq. 19 per pair (sigma factored out,
 * P:356; reading #1 Gauss-Seidel: uses s^k, zeta^k, xi^k).
 * y is overwritten with y^{k+1}; failed pairs keep y^k.
 * rdual[b] = sum ||lambda^{k+1}-lambda^k||^2 + ||mu^{k+1}-mu^k||^2 (Eq. 18b, P:326;
 * gamma excluded, reading #19).  Returns the number of failed pairs.
 * ------------------------------------------------------------------------- */
/* pairs [p0, p1) only, rdual[b] += their terms (the whole sweep: p0 = 0, p1 = #pairs,
 * rdual zeroed first; orc_dual_sweep).  Also the unit of the threaded fan-out. */
static long long dual_sweep_range(const orc_problem* P, orc_iterate* I, long long p0, long long p1, double* rdual) {
  int d = P->dim, N = P->horizon, ns = P->n_state;
  long long fails = 0;
  for (long long p = p0; p < p1; ++p) {
    int b, t, i, j;
    decode(P, p, &b, &t, &i, &j);
    if (!sensed(P, b, j)) {
      if (I->pivots) I->pivots[p] = 0;
      if (I->status) I->status[p] = ORC_OK;
      continue;
    }
    double R[9], rho[3];
    orc_pose(P->pose_model, P->pose_idx, d, I->s + ((long long)b * (N + 1) + t) * ns, R, rho);
    int r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
    int o = b * P->n_obs + j, l0 = P->obs_off[o], no = P->obs_off[o + 1] - l0;
    double ynew[MAXN];
    int piv, basis[MAXN];
    double rj[3];
    double bt[MAXN], rhoi[3];
    part_frame(P, i, R, rho, bt, rhoi);
    obstacle_frame(P, b, j, t, rhoi, rj);
    int st = orc_pair_solve(d, nr, P->part_A + (long long)r0 * d, bt, no,
                            P->obs_C + (long long)l0 * d, P->obs_d + l0, R, rj, I->zeta[p],
                            I->xi + p * d, P->prox_eps, I->y + p * P->ny, P->pivot_tol,
                            P->tie_tol, P->max_pivot_factor, ynew, &piv, basis);
    if (I->zmask) { /* basis labels: w_i = i, z_j = n + j, z0 = 2n */
      const int n = nr + no + 1;
      unsigned zm = 0;
      for (int r = 0; r < n; ++r) {
        if (basis[r] >= n && basis[r] < 2 * n) zm |= 1u << (basis[r] - n);
        if (basis[r] == 2 * n) zm |= 0x80000000u;
      }
      I->zmask[p] = zm;
    }
    if (I->pivots) I->pivots[p] = piv;
    if (I->status) I->status[p] = st;
    if (st != ORC_OK) { ++fails; continue; }
    double* y = I->y + p * P->ny;
    for (int k = 0; k < nr + no; ++k) {
      double df = ynew[k] - y[k];
      rdual[b] += df * df;
    }
    for (int k = 0; k < nr + no + 1; ++k) y[k] = ynew[k];
  }
  return fails;
}

long long orc_dual_sweep(const orc_problem* P, orc_iterate* I, double* rdual) {
  for (int b = 0; b < P->n_scenes; ++b) rdual[b] = 0.0;
  return dual_sweep_range(P, I, 0, n_pairs(P), rdual);
}

/* ---------------------------------------------------------------------------
 * ADMM step 2, Eq. 16 as ONE SQP/Gauss-Newton QP,
 * linearised at s^k (reading #9), with y^{k+1}, zeta^k, xi^k (reading #1):
 *   min sum_{t=1..N} ||s_t - sref_t||^2_Qs + sum_{t=0..N-1} ||u_t||^2_Qu
 *       + sigma/2 sum_p [ (T_p^lin + zeta_p)^2 + ||R_p^lin + xi_p||^2 ]
 *   s.t. s_{t+1} = A_t s_t + B_t u_t + c_t, s_0 fixed
 * Per pair at pose(s^k): u* = K^T y + bvec = (eT, eR); v = C_j^T mu;
 *   dT/drho = -v; dR/dth = (R J)^T v (J = d/dth rotation generator), so
 *   S_t += [[v v^T, 0],[0, g^T g]], g_t += (-eT v, g^T eR),  g = J^T R^T v.
 * Stage: H_t = 2Qs + sigma P^T S_t P, h_t = -2 Qs sref_t + sigma P^T (g_t - S_t P s^k_t).
 * Solved here by condensing states onto controls and a dense Cholesky factor
 * (a different algorithm from the GPU's Riccati recursion).  s, u overwritten.
 * ------------------------------------------------------------------------- */
static int cholesky_solve(int m, double* H, double* rhs) {
  for (int j = 0; j < m; ++j) {
    double s = H[j * m + j];
    for (int k = 0; k < j; ++k) s -= H[j * m + k] * H[j * m + k];
    if (!(s > 0.0)) return -1;
    double l = sqrt(s);
    H[j * m + j] = l;
    for (int i = j + 1; i < m; ++i) {
      double a = H[i * m + j];
      for (int k = 0; k < j; ++k) a -= H[i * m + k] * H[j * m + k];
      H[i * m + j] = a / l;
    }
  }
  for (int i = 0; i < m; ++i) {
    double a = rhs[i];
    for (int k = 0; k < i; ++k) a -= H[i * m + k] * rhs[k];
    rhs[i] = a / H[i * m + i];
  }
  for (int i = m - 1; i >= 0; --i) {
    double a = rhs[i];
    for (int k = i + 1; k < m; ++k) a -= H[k * m + i] * rhs[k];
    rhs[i] = a / H[i * m + i];
  }
  return 0;
}

/* GN aggregates of one scene: S[t][np*np], g[t][np] for t = 1..N (index t-1) */
static void scene_aggregates(const orc_problem* P, const orc_iterate* I, int b, double* S, double* g) {
  int d = P->dim, N = P->horizon, ns = P->n_state, npc = n_pose_coords(P), w = d + 1;
  memset(S, 0, sizeof(double) * N * npc * npc);
  memset(g, 0, sizeof(double) * N * npc);
  for (int t = 1; t <= N; ++t) {
    double R[9], rho[3];
    orc_pose(P->pose_model, P->pose_idx, d, I->s + ((long long)b * (N + 1) + t) * ns, R, rho);
    double* St = S + (t - 1) * npc * npc;
    double* gt = g + (t - 1) * npc;
    for (int i = 0; i < P->n_parts; ++i) {
      int r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
      for (int j = 0; j < P->n_obs; ++j) {
        if (!sensed(P, b, j)) continue;
        long long p = (((long long)b * N + (t - 1)) * P->n_parts + i) * P->n_obs + j;
        int o = b * P->n_obs + j, l0 = P->obs_off[o], no = P->obs_off[o + 1] - l0;
        int n = nr + no + 1;
        double K[MAXN * (MAXD + 1)], rj[3], bt[MAXN], rhoi[3];
        part_frame(P, i, R, rho, bt, rhoi);
        obstacle_frame(P, b, j, t, rhoi, rj);
        orc_build_K(d, nr, P->part_A + (long long)r0 * d, no, P->obs_C + (long long)l0 * d,
                    P->obs_d + l0, R, rj, K);
        const double* y = I->y + p * P->ny;
        double us[MAXD + 1];
        us[0] = 1.0 + I->zeta[p];
        for (int a = 0; a < d; ++a) us[1 + a] = I->xi[p * d + a];
        for (int k = 0; k < n; ++k)
          for (int c = 0; c < w; ++c) us[c] += K[k * w + c] * y[k];
        double eT = us[0];
        const double* eR = us + 1;
        double v[MAXD] = {0};
        for (int l = 0; l < no; ++l)
          for (int a = 0; a < d; ++a) v[a] += y[nr + l] * P->obs_C[(long long)(l0 + l) * d + a];
        for (int a = 0; a < d; ++a) {
          for (int c = 0; c < d; ++c) St[a * npc + c] += v[a] * v[c];
          gt[a] += -eT * v[a];
        }
        if (P->pose_model != ORC_POSE_TRANSLATION) {
          /* w = R^T v;  g = J^T w with J = [[0,-1],[1,0]] (SE2) or its 3D yaw analogue */
          double wv[MAXD] = {0};
          for (int a = 0; a < d; ++a)
            for (int c = 0; c < d; ++c) wv[a] += R[c * d + a] * v[c];
          double gg[MAXD] = {0};
          gg[0] = wv[1];
          gg[1] = -wv[0];
          double gg2 = 0.0, ge = 0.0;
          for (int a = 0; a < d; ++a) { gg2 += gg[a] * gg[a]; ge += gg[a] * eR[a]; }
          St[d * npc + d] += gg2;
          gt[d] += ge;
          if (P->part_ctr) {
            /* scaling centre (reading #22): T depends on theta through rho_i = rho + R o_i,
             * dT/dtheta = tau = -v^T (dR/dtheta) o_i = -w^T G o_i = w_0 o_1 - w_1 o_0 */
            const double* oc = P->part_ctr + (long long)i * d;
            double tau = wv[0] * oc[1] - wv[1] * oc[0];
            for (int a = 0; a < d; ++a) {
              St[a * npc + d] += -v[a] * tau;
              St[d * npc + a] += -v[a] * tau;
            }
            St[d * npc + d] += tau * tau;
            gt[d] += tau * eT;
          }
        }
      }
    }
  }
}

int orc_primal_step(const orc_problem* P, orc_iterate* I) {
  int N = P->horizon, ns = P->n_state, nu = P->n_ctrl, npc = n_pose_coords(P);
  int m = N * nu;
  double sig = P->sigma;
  const int box = has_box(P);
  const double rb = P->box_rho;
  double* S = (double*)malloc(sizeof(double) * N * npc * npc);
  double* g = (double*)malloc(sizeof(double) * N * npc);
  double* F = (double*)malloc(sizeof(double) * ns * m);   /* s_t = F U + f */
  double* F2 = (double*)malloc(sizeof(double) * ns * m);
  double* HF = (double*)malloc(sizeof(double) * ns * m);
  double* Hc = (double*)malloc(sizeof(double) * m * m);
  double* gc = (double*)malloc(sizeof(double) * m);
  double f[16], f2[16], H[256], h[16];
  int pidx[4];
  for (int a = 0; a < npc; ++a) pidx[a] = P->pose_idx[a];
  /* dyn_model 1: this scene's LTV at the current iterate, computed before the update */
  double* Lin = P->dyn_model ? (double*)malloc(sizeof(double) * N * (16 + 8 + 4)) : NULL;
  int rc = 0;
  for (int b = 0; b < P->n_scenes && rc == 0; ++b) {
    if (Lin)
      for (int t = 0; t < N; ++t)
        unicycle_ltv(P->dt, I->s + ((long long)b * (N + 1) + t) * ns, Lin + t * 28, Lin + t * 28 + 16,
                     Lin + t * 28 + 24);
#define DYN_A(b_, t_) (Lin ? Lin + (t_) * 28 : dyn_ptr(P, P->dyn_A, b_, t_, ns * ns))
#define DYN_B(b_, t_) (Lin ? Lin + (t_) * 28 + 16 : dyn_ptr(P, P->dyn_B, b_, t_, ns * nu))
#define DYN_C(b_, t_) (Lin ? Lin + (t_) * 28 + 24 : dyn_ptr(P, P->dyn_c, b_, t_, ns))
    scene_aggregates(P, I, b, S, g);
    memset(Hc, 0, sizeof(double) * m * m);
    memset(gc, 0, sizeof(double) * m);
    for (int t = 0; t < N; ++t)
      for (int a = 0; a < nu; ++a)
        for (int c = 0; c < nu; ++c) Hc[(t * nu + a) * m + t * nu + c] += 2.0 * P->Qu[a * nu + c];
    if (box) /* control part of (rho_b/2) ||u - w + l||^2: Hessian rho_b, gradient -rho_b (w - l) */
      for (int t = 0; t < N; ++t)
        for (int a = 0; a < nu; ++a)
          if (box_on(P->u_min, P->u_max, a)) {
            long long k = ((long long)b * N + t) * nu + a;
            Hc[(t * nu + a) * m + t * nu + a] += rb;
            gc[t * nu + a] += -rb * (I->wu[k] - I->lu[k]);
          }
    memset(F, 0, sizeof(double) * ns * m);
    for (int a = 0; a < ns; ++a) f[a] = P->s0[b * ns + a];
    for (int t = 0; t < N; ++t) {
      /* propagate: s_{t+1} = A_t s_t + B_t u_t + c_t */
      const double* At = DYN_A(b, t);
      const double* Bt = DYN_B(b, t);
      const double* ct = DYN_C(b, t);
      for (int a = 0; a < ns; ++a) {
        double acc = ct[a];
        for (int c = 0; c < ns; ++c) acc += At[a * ns + c] * f[c];
        f2[a] = acc;
        for (int col = 0; col < m; ++col) {
          double v = 0.0;
          for (int c = 0; c < ns; ++c) v += At[a * ns + c] * F[c * m + col];
          F2[a * m + col] = v;
        }
        for (int c = 0; c < nu; ++c) F2[a * m + t * nu + c] += Bt[a * nu + c];
      }
      memcpy(F, F2, sizeof(double) * ns * m);
      memcpy(f, f2, sizeof(double) * ns);
      /* stage t+1 cost: H = 2Qs + sigma P^T S P, h = -2 Qs sref + sigma P^T (g - S P s^k) */
      int tt = t + 1;
      const double* sref = P->s_ref + ((long long)b * (N + 1) + tt) * ns;
      const double* sk = I->s + ((long long)b * (N + 1) + tt) * ns;
      const double* St = S + t * npc * npc;
      const double* gt = g + t * npc;
      for (int a = 0; a < ns; ++a) {
        h[a] = 0.0;
        for (int c = 0; c < ns; ++c) {
          H[a * ns + c] = 2.0 * P->Qs[a * ns + c];
          h[a] += -2.0 * P->Qs[a * ns + c] * sref[c];
        }
      }
      for (int a = 0; a < npc; ++a) {
        double sp = gt[a];
        for (int c = 0; c < npc; ++c) {
          H[pidx[a] * ns + pidx[c]] += sig * St[a * npc + c];
          sp -= St[a * npc + c] * sk[pidx[c]];
        }
        h[pidx[a]] += sig * sp;
      }
      if (box) /* state part of (rho_b/2) ||s_t - w_t + l_t||^2 */
        for (int a = 0; a < ns; ++a)
          if (box_on(P->s_min, P->s_max, a)) {
            long long k = ((long long)b * (N + 1) + tt) * ns + a;
            H[a * ns + a] += rb;
            h[a] += -rb * (I->ws[k] - I->ls[k]);
          }
      /* Hc += F^T H F, gc += F^T (H f + h) */
      for (int a = 0; a < ns; ++a)
        for (int col = 0; col < m; ++col) {
          double v = 0.0;
          for (int c = 0; c < ns; ++c) v += H[a * ns + c] * F[c * m + col];
          HF[a * m + col] = v;
        }
      for (int r = 0; r < m; ++r)
        for (int col = 0; col < m; ++col) {
          double v = 0.0;
          for (int a = 0; a < ns; ++a) v += F[a * m + r] * HF[a * m + col];
          Hc[r * m + col] += v;
        }
      for (int a = 0; a < ns; ++a) {
        double hv = h[a];
        for (int c = 0; c < ns; ++c) hv += H[a * ns + c] * f[c];
        for (int r = 0; r < m; ++r) gc[r] += F[a * m + r] * hv;
      }
    }
    for (int r = 0; r < m; ++r) gc[r] = -gc[r];
    if (cholesky_solve(m, Hc, gc) != 0) { rc = -1; break; }
    /* controls, then roll the dynamics forward from s_0 (Eq. 13b holds exactly) */
    double* sb = I->s + (long long)b * (N + 1) * ns;
    for (int a = 0; a < ns; ++a) sb[a] = P->s0[b * ns + a];
    for (int t = 0; t < N; ++t) {
      double* ut = I->u + ((long long)b * N + t) * nu;
      for (int a = 0; a < nu; ++a) ut[a] = gc[t * nu + a];
      const double* At = DYN_A(b, t);
      const double* Bt = DYN_B(b, t);
      const double* ct = DYN_C(b, t);
      for (int a = 0; a < ns; ++a) {
        double acc = ct[a];
        for (int c = 0; c < ns; ++c) acc += At[a * ns + c] * sb[t * ns + c];
        for (int c = 0; c < nu; ++c) acc += Bt[a * nu + c] * ut[c];
        sb[(t + 1) * ns + a] = acc;
      }
    }
    if (box) { /* w^{k+1} = Pi_box(x^{k+1} + l^k), l^{k+1} = l^k + x^{k+1} - w^{k+1} */
      double res = 0.0;
      for (int t = 0; t < N; ++t) {
        for (int a = 0; a < nu; ++a) {
          if (!box_on(P->u_min, P->u_max, a)) continue;
          long long k = ((long long)b * N + t) * nu + a;
          double x = I->u[k];
          double w = clip(x + I->lu[k], box_lo(P->u_min, a), box_hi(P->u_max, a));
          I->lu[k] = I->lu[k] + (x - w);
          I->wu[k] = w;
          res += (x - w) * (x - w);
        }
        for (int a = 0; a < ns; ++a) {
          if (!box_on(P->s_min, P->s_max, a)) continue;
          long long k = ((long long)b * (N + 1) + t + 1) * ns + a;
          double x = I->s[k];
          double w = clip(x + I->ls[k], box_lo(P->s_min, a), box_hi(P->s_max, a));
          I->ls[k] = I->ls[k] + (x - w);
          I->ws[k] = w;
          res += (x - w) * (x - w);
        }
      }
      I->boxres[b] = res;
    }
  }
#undef DYN_A
#undef DYN_B
#undef DYN_C
  free(S); free(g); free(F); free(F2); free(HF); free(Hc); free(gc); free(Lin);
  return rc;
}

/* ---------------------------------------------------------------------------
 * ADMM step 3, Eq. 17 at s^{k+1}, y^{k+1} (reading #1, #21):
 *   T_p = 1 + (d_j - C_j rho)^T mu + gamma          (Eq. 10)
 *   R_p = A_i^T lambda + (C_j R)^T mu               (Eq. 11)
 *   zeta += T_p, xi += R_p;  rpri[b] = sum T_p^2 + ||R_p||^2  (Eq. 18a)
 * ------------------------------------------------------------------------- */
void orc_multiplier_update(const orc_problem* P, orc_iterate* I, double* rpri) {
  int d = P->dim, N = P->horizon, ns = P->n_state;
  long long np = n_pairs(P);
  for (int b = 0; b < P->n_scenes; ++b) rpri[b] = 0.0;
  for (long long p = 0; p < np; ++p) {
    int b, t, i, j;
    decode(P, p, &b, &t, &i, &j);
    if (!sensed(P, b, j)) continue;
    double R[9], rho[3];
    orc_pose(P->pose_model, P->pose_idx, d, I->s + ((long long)b * (N + 1) + t) * ns, R, rho);
    int r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
    int o = b * P->n_obs + j, l0 = P->obs_off[o], no = P->obs_off[o + 1] - l0;
    const double* y = I->y + p * P->ny;
    const double* lam = y;
    const double* mu = y + nr;
    double gam = y[nr + no];
    double T = 1.0, rj[3], bt[MAXN], rhoi[3];
    part_frame(P, i, R, rho, bt, rhoi);
    obstacle_frame(P, b, j, t, rhoi, rj);
    for (int l = 0; l < no; ++l) {
      double cr = 0.0;
      for (int a = 0; a < d; ++a) cr += P->obs_C[(long long)(l0 + l) * d + a] * rj[a];
      T += (P->obs_d[l0 + l] - cr) * mu[l];
    }
    T += gam;
    double Rr[MAXD];
    for (int a = 0; a < d; ++a) {
      double acc = 0.0;
      for (int k = 0; k < nr; ++k) acc += P->part_A[(long long)(r0 + k) * d + a] * lam[k];
      for (int l = 0; l < no; ++l) {
        double cR = 0.0; /* (C_j R)_{l,a} */
        for (int c = 0; c < d; ++c) cR += P->obs_C[(long long)(l0 + l) * d + c] * R[c * d + a];
        acc += cR * mu[l];
      }
      Rr[a] = acc;
    }
    I->zeta[p] += T;
    double r2 = T * T;
    for (int a = 0; a < d; ++a) {
      I->xi[p * d + a] += Rr[a];
      r2 += Rr[a] * Rr[a];
    }
    rpri[b] += r2;
  }
  /* box block (reading #7): its primal residual ||x - w||^2 joins Eq. 18a's sum */
  if (has_box(P))
    for (int b = 0; b < P->n_scenes; ++b) rpri[b] += I->boxres[b];
}

/* ---------------------------------------------------------------------------
 * K ADMM iterations, fixed count; per-iteration per-scene residual
 * histories hist_rpri[k*B + b], hist_rdual[k*B + b] (may be NULL).
 * Returns total failed pairs, or -1 if a primal solve failed.
 * ------------------------------------------------------------------------- */
long long orc_admm_iterate(const orc_problem* P, orc_iterate* I, int K, double* hist_rpri,
                           double* hist_rdual) {
  int B = P->n_scenes;
  double* rp = (double*)malloc(sizeof(double) * B);
  double* rd = (double*)malloc(sizeof(double) * B);
  long long fails = 0;
  for (int k = 0; k < K; ++k) {
    fails += orc_dual_sweep(P, I, rd);
    if (orc_primal_step(P, I) != 0) { fails = -1; break; }
    orc_multiplier_update(P, I, rp);
    for (int b = 0; b < B; ++b) {
      if (hist_rpri) hist_rpri[(long long)k * B + b] = rp[b];
      if (hist_rdual) hist_rdual[(long long)k * B + b] = rd[b];
    }
  }
  free(rp);
  free(rd);
  return fails;
}

/* alpha* (Eq. 3) for every pair at the states s; alpha[p].  Returns #infeasible. */
long long orc_scale_detect(const orc_problem* P, const double* s, double* alpha) {
  int d = P->dim, N = P->horizon, ns = P->n_state;
  long long np = n_pairs(P), bad = 0;
  for (long long p = 0; p < np; ++p) {
    int b, t, i, j;
    decode(P, p, &b, &t, &i, &j);
    if (!sensed(P, b, j)) {
      alpha[p] = INFINITY;
      continue;
    }
    double R[9], rho[3];
    orc_pose(P->pose_model, P->pose_idx, d, s + ((long long)b * (N + 1) + t) * ns, R, rho);
    int r0 = P->part_off[i], nr = P->part_off[i + 1] - r0;
    int o = b * P->n_obs + j, l0 = P->obs_off[o], no = P->obs_off[o + 1] - l0;
    double rj[3];
    double bt[MAXN], rhoi[3];
    part_frame(P, i, R, rho, bt, rhoi);
    obstacle_frame(P, b, j, t, rhoi, rj);
    if (orc_scale_lp(d, nr, P->part_A + (long long)r0 * d, bt, R, rj, no,
                     P->obs_C + (long long)l0 * d, P->obs_d + l0, alpha + p, NULL) != 0) {
      alpha[p] = NAN;
      ++bad;
    }
  }
  return bad;
}

/* ---------------------------------------------------------------------------
 * Eq. 18: the stopping criteria,
 *   r_pri  = sum_ijt ||zeta^{k+1} - zeta^k||^2 + ||xi^{k+1} - xi^k||^2  <= eps_pri   (18a)
 *   r_dual = sum_ijt ||lambda^{k+1} - lambda^k||^2 + ||mu^{k+1} - mu^k||^2 <= eps_dual (18b)
 * with '<=' as printed ("sum exactly eps -> true").  r_pri is what
 * orc_multiplier_update returns (zeta^{k+1} - zeta^k = T, Eq. 17; plus the box block's
 * ||x - w||^2, reading #7), r_dual what orc_dual_sweep returns (gamma excluded,
 * reading #19).
 * ------------------------------------------------------------------------- */
int orc_check_stopping(double r_pri, double r_dual, double eps_pri, double eps_dual) {
  return (r_pri <= eps_pri) && (r_dual <= eps_dual);
}

/* The problem and iterate of scene b alone (n_scenes = 1): every per-scene array is
 * offset to scene b; obs_off keeps absolute row indices into obs_C / obs_d, so the
 * view's obs_off = P->obs_off + b*M needs no rebasing.  Scenes share nothing in the
 * method (one robot, its own obstacles), so iterating the view = iterating
 * scene b of the batch. */
static void scene_view(const orc_problem* P, const orc_iterate* I, int b, orc_problem* Pb, orc_iterate* Ib) {
  const int N = P->horizon, ns = P->n_state, nu = P->n_ctrl, M = P->n_obs, d = P->dim;
  const long long pps = (long long)N * P->n_parts * M; /* pairs per scene */
  *Pb = *P;
  Pb->n_scenes = 1;
  Pb->obs_off = P->obs_off + (long long)b * M;
  if (P->dyn_per_scene) {
    const long long nt = P->dyn_per_time ? N : 1;
    Pb->dyn_A = P->dyn_A + (long long)b * nt * ns * ns;
    Pb->dyn_B = P->dyn_B + (long long)b * nt * ns * nu;
    Pb->dyn_c = P->dyn_c + (long long)b * nt * ns;
  }
  Pb->s0 = P->s0 + (long long)b * ns;
  Pb->s_ref = P->s_ref + (long long)b * (N + 1) * ns;
  if (P->obs_step) Pb->obs_step = P->obs_step + (long long)b * M * d;
  if (P->sensed) Pb->sensed = P->sensed + (long long)b * M;
  *Ib = *I;
  Ib->s = I->s + (long long)b * (N + 1) * ns;
  Ib->u = I->u + (long long)b * N * nu;
  Ib->y = I->y + b * pps * P->ny;
  Ib->zeta = I->zeta + b * pps;
  Ib->xi = I->xi + b * pps * d;
  if (I->pivots) Ib->pivots = I->pivots + b * pps;
  if (I->status) Ib->status = I->status + b * pps;
  if (I->zmask) Ib->zmask = I->zmask + b * pps;
  if (I->ws) {
    Ib->ws = I->ws + (long long)b * (N + 1) * ns;
    Ib->ls = I->ls + (long long)b * (N + 1) * ns;
    Ib->wu = I->wu + (long long)b * N * nu;
    Ib->lu = I->lu + (long long)b * N * nu;
    Ib->boxres = I->boxres + b;
  }
}

/* ADMM until Eq. 18: every scene of the batch is its own MPC problem and
 * stops at the first iteration k whose residuals meet Eq. 18 (orc_check_stopping),
 * its iterate left there; or after max_iters.  Per scene: iters[b] (iterations run),
 * conv[b] (0/1), rpri[b], rdual[b] (residuals of its last iteration).  Returns the
 * total number of failed pair solves, or -1 if a primal solve failed. */
long long orc_admm_solve(const orc_problem* P, orc_iterate* I, double eps_pri, double eps_dual, int max_iters,
                         int* iters, int* conv, double* rpri, double* rdual) {
  long long fails = 0;
  for (int b = 0; b < P->n_scenes; ++b) {
    orc_problem Pb;
    orc_iterate Ib;
    scene_view(P, I, b, &Pb, &Ib);
    double rp = 0.0, rd = 0.0;
    iters[b] = 0;
    conv[b] = 0;
    for (int k = 0; k < max_iters; ++k) {
      fails += orc_dual_sweep(&Pb, &Ib, &rd);        /* Eq. 15 */
      if (orc_primal_step(&Pb, &Ib) != 0) return -1; /* Eq. 16 */
      orc_multiplier_update(&Pb, &Ib, &rp);          /* Eq. 17 */
      iters[b] = k + 1;
      if (orc_check_stopping(rp, rd, eps_pri, eps_dual)) { /* Eq. 18 */
        conv[b] = 1;
        break;
      }
    }
    rpri[b] = rp;
    rdual[b] = rd;
  }
  return fails;
}

/* ---------------------------------------------------------------------------
 * Timing helper for the all-core CPU baseline: the same K fixed
 * iterations as orc_admm_iterate, fanned out over nthreads POSIX threads.
 *  - n_scenes >= nthreads: scenes are distributed over the threads, each scene iterated
 *    alone (scene_view) -- bitwise the sequential result (per-scene order unchanged).
 *  - fewer scenes: per iteration the pairs of the dual step (Eq. 15) are split into
 *    nthreads contiguous ranges, each with its own residual partial summed in range
 *    order (rounding-level differences in r_dual only); the primal step and the
 *    multiplier update stay sequential.
 * ------------------------------------------------------------------------- */
typedef struct {
  const orc_problem* P;
  orc_iterate* I;
  int K, b0, b1, B;
  long long p0, p1;
  double *hist_rpri, *hist_rdual, *rd;
  long long fails;
  int rc;
} mt_job;

static void* mt_scenes(void* arg) {
  mt_job* J = (mt_job*)arg;
  for (int b = J->b0; b < J->b1; ++b) {
    orc_problem Pb;
    orc_iterate Ib;
    scene_view(J->P, J->I, b, &Pb, &Ib);
    for (int k = 0; k < J->K; ++k) {
      double rd = 0.0, rp = 0.0;
      J->fails += orc_dual_sweep(&Pb, &Ib, &rd);
      if (orc_primal_step(&Pb, &Ib) != 0) { J->rc = -1; return NULL; }
      orc_multiplier_update(&Pb, &Ib, &rp);
      if (J->hist_rpri) J->hist_rpri[(long long)k * J->B + b] = rp;
      if (J->hist_rdual) J->hist_rdual[(long long)k * J->B + b] = rd;
    }
  }
  return NULL;
}

static void* mt_pairs(void* arg) {
  mt_job* J = (mt_job*)arg;
  J->fails += dual_sweep_range(J->P, J->I, J->p0, J->p1, J->rd);
  return NULL;
}

long long orc_admm_iterate_mt(const orc_problem* P, orc_iterate* I, int K, double* hist_rpri, double* hist_rdual,
                              int nthreads) {
  const int B = P->n_scenes;
  if (nthreads < 1) nthreads = 1;
  mt_job* J = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  long long fails = 0;
  if (B >= nthreads) {
    for (int t = 0; t < nthreads; ++t) {
      J[t] = (mt_job){P, I, K, (int)((long long)B * t / nthreads), (int)((long long)B * (t + 1) / nthreads), B,
                      0, 0, hist_rpri, hist_rdual, NULL, 0, 0};
      pthread_create(&th[t], NULL, mt_scenes, &J[t]);
    }
    for (int t = 0; t < nthreads; ++t) {
      pthread_join(th[t], NULL);
      fails += J[t].fails;
      if (J[t].rc) fails = -1;
    }
  } else {
    const long long np = n_pairs(P);
    double* rd = (double*)calloc((size_t)nthreads * B, sizeof(double));
    double* rp = (double*)calloc((size_t)B, sizeof(double));
    for (int k = 0; k < K && fails >= 0; ++k) {
      for (int t = 0; t < nthreads; ++t) {
        for (int b = 0; b < B; ++b) rd[(long long)t * B + b] = 0.0;
        J[t] = (mt_job){P, I, K, 0, 0, B, np * t / nthreads, np * (t + 1) / nthreads, NULL, NULL,
                        rd + (long long)t * B, 0, 0};
        pthread_create(&th[t], NULL, mt_pairs, &J[t]);
      }
      for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        fails += J[t].fails;
      }
      if (orc_primal_step(P, I) != 0) { fails = -1; break; }
      orc_multiplier_update(P, I, rp);
      for (int b = 0; b < B; ++b) {
        double s = 0.0;
        for (int t = 0; t < nthreads; ++t) s += rd[(long long)t * B + b];
        if (hist_rpri) hist_rpri[(long long)k * B + b] = rp[b];
        if (hist_rdual) hist_rdual[(long long)k * B + b] = s;
      }
    }
    free(rd);
    free(rp);
  }
  free(J);
  free(th);
  return fails;
}
