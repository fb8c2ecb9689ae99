/* orc.h -- CPU ORACLE for arXiv 2406.07048's ADMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the product (paper_2406_07048_b200/, include/).
 *
 * Citation key: P:n = /root/reference/PAPER.md line n (the LaTeX source);
 * "reading #k" = DESIGN.md "Readings of the paper" item k.
 *
 * Pair index p = ((b*N + (t-1))*n_parts + i)*n_obs + j, t = 1..N (reading #5).
 * y is stored padded: y[p*ny + k], k < n_p = n_r(i) + n_o(b,j) + 1,
 * rows ordered (lambda_1..lambda_nr, mu_1..mu_no, gamma) as in P:368-371.
 */
#ifndef ORC_H
#define ORC_H

enum { ORC_POSE_TRANSLATION = 0, ORC_POSE_SE2 = 1, ORC_POSE_TRANS_YAW = 2 };
enum { ORC_OK = 0, ORC_RAY = 1, ORC_ITER_LIMIT = 2, ORC_NEG_YE = 3 };

typedef struct {
  int dim, n_scenes, horizon, n_state, n_ctrl;
  int pose_model;
  int pose_idx[4];
  int n_parts;
  const int* part_off;
  const double* part_A;
  const double* part_b;
  int n_obs;
  const int* obs_off;
  const double* obs_C;
  const double* obs_d;
  int dyn_per_scene, dyn_per_time;
  const double* dyn_A;
  const double* dyn_B;
  const double* dyn_c;
  const double* Qs;
  const double* Qu;
  const double* s0;
  const double* s_ref;
  double sigma;
  double pivot_tol;
  double tie_tol;
  int max_pivot_factor;
  int ny;
  double prox_eps; /* 0 = paper-exact Eq. 19 (reading #2) */
  /* NULL = static obstacles (reading #15).  Else [n_scenes*n_obs][dim]:
   * per-timestep displacement of each obstacle (NEXT f3, moving traffic): obstacle j
   * at timestep t is O_j + t*step_j, i.e. C_j x <= d_j + t C_j step_j. */
  const double* obs_step;
  /* 0: the LTV model dyn_A/B/c as given (reading #8).  1: the SE2 unicycle of the car
   * scenes, s = (x, y, th, v), u = (a, om), s' = s + dt (v cos th, v sin th, om, a),
   * relinearised at the current iterate (s^k, u^k) in every primal step -- the SQP
   * step of P:272, P:349-351 (NEXT f2). */
  int dyn_model;
  double dt;
  /* State / control boxes of Eq. 13c-d, part of IC_0 -- NEXT f1.
   * NULL = unbounded in that direction; else [n_state] / [n_ctrl], shared by every scene
   * and timestep (s_0 is given, so the state box applies to t = 1..N).  Handled by an
   * extra ADMM block (reading #7): consensus x = w with w in the box, scaled multiplier
   * l, penalty box_rho > 0. */
  const double* s_min;
  const double* s_max;
  const double* u_min;
  const double* u_max;
  double box_rho;
  /* Sensing ("can only sense the obstacles within 20m x 20m x 6m"; NEXT
   * f3): NULL = every obstacle, else [n_scenes*n_obs] 0/1 -- pairs of an unsensed
   * obstacle leave the (i, j, t) table (no dual step, no aggregate, no multiplier
   * update, alpha = +inf).  orc_sense() fills it from the sensing box. */
  const unsigned char* sensed;
  /* Per-part scaling centres (NEXT f3; reading #22): NULL = every part scales about the
   * body origin, else [n_parts][dim] body-frame points o_i strictly inside their parts.
   * Part i is then the polytope A_i (x - o_i) <= b~_i, b~_i = b_i - A_i o_i, scaled about
   * o_i: its pairs use b~_i and the origin rho_i(s) = rho(s) + R(s) o_i. */
  const double* part_ctr;
} orc_problem;

typedef struct {
  double* s;    /* [B][N+1][ns] */
  double* u;    /* [B][N][nu]   */
  double* y;    /* [P][ny]      */
  double* zeta; /* [P]          */
  double* xi;   /* [P][d]       */
  int* pivots;  /* [P] pivots of the last dual sweep */
  int* status;  /* [P] ORC_* of the last dual sweep */
  /* box block (reading #7), used only when the problem has a box: */
  double* ws;     /* [B][N+1][ns] w for the states (t = 0 unused) */
  double* ls;     /* [B][N+1][ns] scaled multiplier l for the states */
  double* wu;     /* [B][N][nu]  w for the controls */
  double* lu;     /* [B][N][nu]  l for the controls */
  double* boxres; /* [B] sum ||x - w||^2 after the last primal step */
  /* nullable: [P] final Lemke basis of the last dual sweep, bit j = z_j basic (LCP
   * index j), bit 31 = z0 basic (ITER_LIMIT); 0 for q >= 0 (L1) */
  unsigned* zmask;
} orc_iterate;

#endif
