/* ca.h -- C ABI of the B200 (sm_100a) FP64 implementation of the ADMM hot path of
 * arXiv 2406.07048 (scale-based collision avoidance; ADMM over per-pair dual QPs).
 *
 * Citation key: P:n = line n of the paper's LaTeX source; DESIGN.md
 * "reading #k" = how this library resolves a point the paper leaves open.
 *
 * Conventions for every entry point
 *  - All pointers passed IN are HOST pointers unless stated; the library copies
 *    what it needs before returning (the caller keeps ownership).  Outputs are
 *    written to caller-allocated HOST buffers.  Device state is owned by the handle.
 *  - Row-major FP64 arrays; int32 offsets.  Scene b, timestep t = 1..N, robot
 *    part i, obstacle j form pair p = ((b*N + (t-1))*n_parts + i)*n_obs + j
 *    (reading #5: collision pairs exist for t = 1..N only).
 *  - All device work is ordered on the CUDA stream given at create.  A handle is
 *    not thread-safe; distinct handles are independent.
 *  - Return value: CA_OK (0), an error (< 0; details in ca_last_error()) or a
 *    warning (> 0).  Validation errors create no handle.  A CUDA error is sticky:
 *    the handle must be destroyed.  Per-pair Lemke failures are not fatal: the
 *    pair keeps its previous certificate, the failure is counted and
 *    CA_W_PAIR_FAILURES is returned.  No exception crosses the ABI.
 *  - No CPU fallback: without a usable sm_100 device every call that needs the
 *    GPU returns CA_E_CUDA.
 */
#ifndef CA_H
#define CA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ca_status;
enum {
  CA_OK = 0,
  CA_E_INVALID = -1,     /* null pointer, non-positive size, bad parameter */
  CA_E_DIM = -2,         /* d not in {2,3}; n = n_r + n_o + 1 > 32; pose index out of range */
  CA_E_GEOMETRY = -3,    /* robot part with b_i (b~_i with part_ctr) not > 0 (reading #22) or < d+1 rows */
  CA_E_UNSUPPORTED = -4, /* unknown pose model, n_state > 8, n_ctrl > 4 */
  CA_E_CUDA = -5,        /* CUDA error / no sm_100 device */
  CA_E_NCCL = -6,
  CA_E_OOM = -7,
  CA_W_NOT_CONVERGED = 1, /* ca_admm_solve hit max_iters */
  CA_W_PAIR_FAILURES = 2  /* >= 1 pair hit RAY / ITER_LIMIT / y_e < -1e-6 */
};

/* pose models R(s), rho(s) (reading #9) */
enum {
  CA_POSE_TRANSLATION = 0, /* rho = s[idx[0..d-1]], R = I */
  CA_POSE_SE2 = 1,         /* d = 2: rho = (s[idx0], s[idx1]), R = Rot(s[idx2]) */
  CA_POSE_TRANS_YAW = 2    /* d = 3: rho = s[idx0..2], R = Rot_z(s[idx3]) */
};

/* per-pair Lemke status (reading #4) */
enum { CA_PAIR_OK = 0, CA_PAIR_RAY = 1, CA_PAIR_ITER_LIMIT = 2, CA_PAIR_NEG_YE = 3 };

typedef struct ca_problem ca_problem;

/* Problem description.  All arrays are HOST arrays, copied at create/load.
 *  robot parts: part_off[n_parts+1]; part_A[rows*d] body-frame face
 *                normals a_k; part_b[rows] > 0.  A_i x <= b_i.
 *  obstacles: obs_off[n_scenes*n_obs+1]; obs_C[rows*d]; obs_d[rows];
 *                C_j y <= d_j in world coordinates; obstacle (b, j) = b*n_obs + j.
 *  dynamics      (P:176-182 linearised): s_{t+1} = A_t s_t + B_t u_t + c_t;
 *                dyn_A[nd*ns*ns], dyn_B[nd*ns*nu], dyn_c[nd*ns] with
 *                nd = (dyn_per_scene ? n_scenes : 1) * (dyn_per_time ? horizon : 1).
 *  cost: sum_t ||s_t - s_ref_t||^2_Qs + ||u_t||^2_Qu (no 1/2);
 *                Qs[ns*ns], Qu[nu*nu] SPD.  s0[B*ns], s_ref[B*(N+1)*ns];
 *                s_init nullable (default: s_ref, reading #11).
 *  ADMM: sigma > 0 (paper: 300); eps_pri/eps_dual per scene
 *                (<= 0: default 1e-3 * pairs per scene); max_iters for ca_admm_solve.
 *  Lemke         (reading #4): pivot_tol (1e-11), tie_tol (1e-9), max pivots
 *                = lemke_max_pivot_factor * n (50).  <= 0 selects the default.
 *  prox_eps      (reading #2): 0 = paper-exact Eq. 19; > 0 adds eps/2 ||y - y^k||^2
 *                (strictly convex pair QPs with a unique minimiser, solved as
 *                prox_solver selects); < 0 or NaN -> CA_E_INVALID.
 */
typedef struct {
  int32_t dim, n_scenes, horizon, n_state, n_ctrl;
  int32_t pose_model;
  int32_t pose_idx[4];
  int32_t n_parts;
  const int32_t* part_off;
  const double* part_A;
  const double* part_b;
  int32_t n_obs;
  const int32_t* obs_off;
  const double* obs_C;
  const double* obs_d;
  int32_t dyn_per_scene, dyn_per_time;
  const double* dyn_A;
  const double* dyn_B;
  const double* dyn_c;
  const double* Qs;
  const double* Qu;
  const double* s0;
  const double* s_ref;
  const double* s_init;
  double sigma, eps_pri, eps_dual;
  int32_t max_iters;
  double lemke_pivot_tol, lemke_tie_tol;
  int32_t lemke_max_pivot_factor;
  double prox_eps;
  /* NEXT f3, moving obstacles (nullable: NULL = static, reading #15):
   * HOST [n_scenes*n_obs][dim], the displacement of each obstacle per timestep --
   * obstacle j of scene b at timestep t is {x : C_j x <= d_j + t C_j step_bj}. */
  const double* obs_step;
  /* Nullable caller-owned DEVICE workspace (e.g. a torch uint8 tensor) of
   * workspace_bytes >= ca_workspace_size(): every buffer of the handle is carved out of
   * it (256-byte aligned) instead of cudaMalloc; the caller keeps it alive until
   * ca_problem_destroy.  Buffers needed later beyond it (more iterations than
   * max_iters, tracing, basis recording) fall back to cudaMalloc. */
  void* workspace;
  size_t workspace_bytes;
  /* NEXT f2: 0 = the LTV model dyn_A/B/c as given (reading #8); 1 = the car's unicycle,
   * s = (x, y, th, v), u = (a, om), s' = s + dt (v cos th, v sin th, om, a), relinearised
   * at the current iterate (s^k, u^k) in every primal step (the SQP step of P:272,
   * P:349-351); requires n_state 4, n_ctrl 2, SE2 pose (0, 1, 2), dt > 0; dyn_A/B/c
   * are then ignored (may be NULL). */
  int32_t dyn_model;
  double dt;
  /* NEXT f1: the state / control boxes of Eq. 13c-d, part of IC_0 in the
   * primal step.  Each nullable HOST array (NULL = unbounded on that side):
   * s_min/s_max[n_state], u_min/u_max[n_ctrl], shared by every scene and timestep;
   * +-inf entries leave a component free.  The state box applies to t = 1..N (s_0 is
   * given).  Handled by an extra ADMM block (reading #7): a copy w of every bounded
   * component constrained to the box, consensus x = w with scaled multiplier l and
   * penalty box_rho (> 0 when any bound is finite); r_pri (Eq. 18a) then also sums
   * ||x - w||^2.  The cold-start iterate is projected into the box;
   * ca_set_iterate resets w = Pi_box(x), l = 0.  min > max or NaN -> CA_E_INVALID. */
  const double* s_min;
  const double* s_max;
  const double* u_min;
  const double* u_max;
  double box_rho;
  /* NEXT f3, sensing ("can only sense the obstacles within 20m x 20m x 6m";
   * S:553).  Nullable HOST [dim] half-extents h > 0: only obstacles meeting the
   * world-aligned box rho(s0_b) + [-h, h] around each scene's current position enter
   * the (i, j, t) table (static positions, t = 0); pairs of the others are skipped by
   * every step (certificates keep their values, alpha = +inf).  Re-evaluated at every
   * create/load (each MPC step).  NULL = every obstacle. */
  const double* sense_half;
  /* NEXT f3, per-part scaling centres (reading #22): nullable HOST [n_parts*dim]
   * body-frame points o_i strictly inside their parts (b~_i = b_i - A_i o_i > 0, else
   * CA_E_GEOMETRY).  Part i is scaled about o_i instead of the body origin: its pairs
   * use b~_i and the origin rho(s) + R(s) o_i (Eq. 3-11 unchanged otherwise), so parts
   * that do not contain the body origin (a trailer) are allowed.  NULL = origin. */
  const double* part_ctr;
  /* NEXT f4, used only when prox_eps > 0: the solver of the strictly
   * convex pair QP (reading #2).  0 = the dual semismooth Newton method on the
   * (d+1)-dimensional dual of Eq. 19 + prox (one pair per thread, warm-started at the
   * root of the affine piece of y^k's support; a pair that does not converge in 64
   * iterations is re-solved by the dense Lemke); 1 = the dense Lemke on every pair (one
   * pair per warp).  Both return the unique minimiser (to rounding), so results agree
   * to the QP's conditioning, not bitwise; pivot counts report Newton iterations for 0.
   * Other values -> CA_E_INVALID. */
  int32_t prox_solver;
} ca_problem_desc;

/* Residuals and statistics of one ADMM iteration (or one step), summed over the
 * handle's scenes -- over ALL scenes of a scene-sharded run in ca_admm_iterate's history
 * and ca_admm_solve's report (Eq. 18; r_dual excludes gamma, reading #19;
 * raw sums, reading #20).
 *   n_pairs      pair QPs of the handle (rank-local)
 *   n_fail       pairs that kept their previous certificate =
 *                n_ray + n_iterlimit + n_neg_ye:
 *   n_ray        Lemke ray termination
 *   n_iterlimit  more than lemke_max_pivot_factor * n pivots
 *   n_neg_ye     recovered y_e < -1e-6
 *   pivots       total Lemke pivots (Newton iterations for prox_solver 0);
 *   max_pivots   the largest pivot count of one pair
 *   ms_*         device milliseconds of the pair sweep, NCCL collectives, primal step
 *                (Riccati) and standalone multiplier update of that iteration / step --
 *                CUDA events on the handle's stream, only while ca_set_timing(h, 1), else 0. */
typedef struct {
  double r_pri, r_dual;
  int64_t n_pairs, n_fail, pivots;
  int64_t n_ray, n_iterlimit, n_neg_ye;
  int32_t max_pivots, reserved_;
  float ms_sweep, ms_comm, ms_riccati, ms_mult;
} ca_residuals;

/* ca_admm_solve's report: iterations = the most iterations any scene ran, converged = 1
 * iff every scene met Eq. 18; last = the statistics of each scene's final iteration,
 * combined over scenes (per scene: ca_get_scene_residuals, ca_get_solve_scenes). */
typedef struct {
  int32_t iterations, converged;
  ca_residuals last;
} ca_solve_report;

/* Device bytes a handle for `desc` (and, if dist is non-NULL, rank dist->rank of an
 * obstacle-sharded problem) takes from a caller workspace: every buffer allocated at
 * creation plus the scale factors and max_iters iterations of statistics.  Host only. */
struct ca_dist_desc_s;
ca_status ca_workspace_size(const ca_problem_desc* desc, const struct ca_dist_desc_s* dist, size_t* bytes);

/* Validate, allocate device state (~(2n_max + 2d + 8) * 8 bytes per pair), upload the
 * problem and initialise the iterate (reading #11).  device: CUDA ordinal; stream:
 * cudaStream_t (NULL = legacy default stream).  On error *out is NULL. */
ca_status ca_problem_create(const ca_problem_desc* desc, int device, void* stream, ca_problem** out);
void ca_problem_destroy(ca_problem* h);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink / NVSwitch) ----
 * The ranks form a scene_shards x obstacle_shards grid (world_size = product; rank r
 * has scene shard r / obstacle_shards and obstacle shard r % obstacle_shards; 0, 0 =
 * 1 x world_size, obstacle sharding only).
 *  - Scene shard s holds scenes [B s / Ws, B (s+1) / Ws) of the full problem (scenes are
 *    independent MPC problems).  Per iteration ONE ncclAllReduce over all ranks carries
 *    every scene's statistics (NSTAT doubles per scene: Eq. 18's r_pri, r_dual, pivot and
 *    failure counts), so every rank sees the global residuals: ca_admm_solve's stop
 *    decision (Eq. 18 per scene, until every scene of every rank has stopped) and
 *    ca_admm_iterate's history are global and identical on every rank.
 *  - Obstacle shard o owns obstacles [j0, j1) of its scenes (a contiguous block balanced
 *    by total face count, ca_obstacle_partition) and solves only those pairs; every rank
 *    of the group holds the full trajectory of its scenes.  Per iteration the per-(scene,
 *    t) aggregates of step 2 and the residual partials are summed by ONE
 *    ncclAllReduce over the group (ncclCommSplit of the world); the primal step then runs
 *    replicated on identical bytes.
 * Getters are rank-local: scenes counted from the shard's first scene, pair indices with
 * j counted from j0. */
typedef struct ca_dist_desc_s {
  int32_t world_size, rank;
  const uint8_t* nccl_id; /* 128 bytes from ca_nccl_unique_id on one rank, broadcast */
  int32_t scene_shards, obstacle_shards; /* grid; 0, 0 = 1 x world_size */
} ca_dist_desc;

ca_status ca_nccl_unique_id(uint8_t* out128);

/* Pure host function: the obstacle block [*j0, *j1) of `rank`. */
ca_status ca_obstacle_partition(int32_t n_scenes, int32_t n_obs, const int32_t* obs_off, int32_t world_size,
                                int32_t rank, int32_t* j0, int32_t* j1);

/* ca_problem_create for rank dist->rank of a sharded problem (desc is the FULL problem;
 * the rank keeps its scene and obstacle block).  world_size == 1 is allowed (the NCCL
 * path on one rank).  CA_E_INVALID if scene_shards * obstacle_shards != world_size or
 * scene_shards > n_scenes.  A rank whose obstacle block is empty still takes part in
 * every collective. */
ca_status ca_problem_create_dist(const ca_problem_desc* desc, const ca_dist_desc* dist, int device, void* stream,
                                 ca_problem** out);

/* Re-upload every per-batch input of a problem with the SAME shapes (n_scenes,
 * horizon, parts, per-obstacle row counts) and reset the iterate.  The end-to-end
 * path: load -> ca_admm_iterate -> ca_get_trajectory. */
ca_status ca_problem_load(ca_problem* h, const ca_problem_desc* desc);

/* Reset the iterate to the initial point (reading #11) from the device-resident
 * inputs: s = s_ref (s_0 = s0), u = 0, lambda = 1/sum(b_i), mu = gamma = zeta = xi = 0.
 * Device-only (no host transfer): starts a new solve on the same inputs. */
ca_status ca_reset_iterate(ca_problem* h);

/* n_pairs, ny (= n_max, the per-pair y stride of ca_get_pair_state), device bytes. */
ca_status ca_problem_info(const ca_problem* h, int64_t* n_pairs, int32_t* ny, int64_t* device_bytes);

/* Eq. 3: alpha*_p for every pair at the states `states` (HOST
 * [B*(N+1)*ns], NULL = current iterate).  alpha: HOST [n_pairs] or NULL;
 * min_alpha: HOST [n_scenes] (per-scene minimum) or NULL. */
ca_status ca_scale_detect(ca_problem* h, const double* states, double* alpha, double* min_alpha);

/* `iters` fixed ADMM iterations (Eqs. 15-17, reading #1 Gauss-Seidel), no
 * early stop.  hist: HOST [iters] per-iteration residuals or NULL. */
ca_status ca_admm_iterate(ca_problem* h, int32_t iters, ca_residuals* hist);

/* ADMM until Eq. 18: every scene is its own MPC problem and stops at the
 * first iteration with r_pri <= eps_pri and r_dual <= eps_dual ('<=' as printed; SPEC
 * S:528) -- its iterate stays there while the other scenes continue -- or after
 * max_iters.  eps <= 0 at create: 1e-3 * pairs per scene of the FULL problem (SPEC
 * S:551).  Scene-sharded: the loop ends when every scene of every rank has stopped (the
 * per-iteration allreduce makes that decision identical on every rank).  Each call
 * starts from the current iterate.  CA_W_NOT_CONVERGED if a scene hit max_iters. */
ca_status ca_admm_solve(ca_problem* h, ca_solve_report* out);

/* After ca_admm_solve: per local scene, the iterations it ran and whether it met Eq. 18
 * (HOST [n_scenes] int32 each, nullable).  CA_E_INVALID before any solve. */
ca_status ca_get_solve_scenes(ca_problem* h, int32_t* iterations, int32_t* converged);

/* The three ADMM steps one at a time (frozen-input parity): step 1 (Eq. 15),
 * step 2 (Eq. 16), step 3 (Eq. 17).  out may be NULL. */
ca_status ca_dual_sweep(ca_problem* h, ca_residuals* out);
ca_status ca_primal_step(ca_problem* h);
ca_status ca_multiplier_update(ca_problem* h, ca_residuals* out);

/* The obstacle-sharded exchange made observable on one GPU: the
 * per-(scene, t) records of the last dual sweep, each the fixed-order sum over this
 * handle's pairs of that (scene, t) -- exactly what an obstacle-sharded rank
 * contributes to the per-iteration ncclAllReduce -- into HOST rec[B*N][R] (R = 17 for
 * dim 2, 22 for dim 3: (d+1)(d+2)/2 + (d+1) Gauss-Newton terms, then r_dual, r_pri,
 * pivots, failures, rays, iteration limits, negative y_e, max pivots).
 * ca_primal_step_records runs Eq. 16 (the replicated Riccati step of the sharded path)
 * on given HOST records of the same layout (e.g. the sum of two obstacle halves). */
ca_status ca_get_stage_records(ca_problem* h, double* rec);
ca_status ca_primal_step_records(ca_problem* h, const double* rec);

/* Per-scene residuals of the last completed step (after ca_admm_solve: of each scene's
 * final iteration): HOST [n_scenes] each (nullable). */
ca_status ca_get_scene_residuals(ca_problem* h, double* r_pri, double* r_dual);

/* HOST s[B*(N+1)*ns], u[B*N*nu] (either may be NULL). */
ca_status ca_get_trajectory(ca_problem* h, double* s, double* u);

/* Pair state for pairs [p0, p0+count): y[count*ny] (padded with 0 beyond n_p),
 * zeta[count], xi[count*d], pivots[count], status[count] (CA_PAIR_*; | 0x100 if the
 * pair was re-solved by the dense-tableau fallback), zmask[count]
 * (bit j = z_j basic in the final Lemke basis, bit 31 = z0).  Any may be NULL. */
ca_status ca_get_pair_state(ca_problem* h, int64_t p0, int64_t count, double* y, double* zeta,
                            double* xi, int32_t* pivots, int32_t* status, uint32_t* zmask);

/* Overwrite the iterate (any pointer may be NULL = keep).  Layouts as the getters.
 * With boxes (NEXT f1) the box block restarts from w = Pi_box(s, u), l = 0. */
ca_status ca_set_iterate(ca_problem* h, const double* s, const double* u, const double* y,
                         const double* zeta, const double* xi);

/* Box block state (NEXT f1, reading #7) into HOST arrays (any may be NULL): w_s, l_s
 * [B][N+1][ns] (t = 0 entries are Pi_box(s_0), 0), w_u, l_u [B][N][nu], res[B] =
 * sum ||x - w||^2 after the last primal step.  CA_E_INVALID if the problem has no box. */
ca_status ca_get_box_state(ca_problem* h, double* w_s, double* l_s, double* w_u, double* l_u, double* res);

/* Device milliseconds accumulated per family since the last reset (CUDA events on
 * the handle's stream, only while ca_set_timing(h, 1)): ms[0] pair sweep, [1] primal,
 * [2] multiplier, [3] scale detect (+ per-scene min), [4] other small kernels (init,
 * collect, history; not timed, ms[4] = 0), [5] NCCL collectives; launches[0..4] the
 * matching counts of this library's kernel launches, launches[5] the collectives
 * (always counted).  Arrays have 6 entries; reset != 0 zeroes. */
ca_status ca_kernel_times(ca_problem* h, double* ms, int64_t* launches, int32_t reset);

/* Enable (1) / disable (0) per-launch event timing (default off). */
ca_status ca_set_timing(ca_problem* h, int32_t enable);

/* Enable (1) / disable (0) recording of each pair's final Lemke basis (zmask of
 * ca_get_pair_state; costs 4 bytes per pair per sweep of extra HBM writes). */
ca_status ca_set_record_basis(ca_problem* h, int32_t enable);

/* Measured FP64 FMA throughput of the device: a register-resident DFMA loop on all
 * SMs for ~`ms` milliseconds; *tflops = 2 * FMAs / s / 1e12. */
ca_status ca_fp64_peak(int device, double ms, double* tflops);

/* Diagnostics: trace the Lemke pivots of pair p (-1 = off) during subsequent sweeps
 * into an internal buffer; out (HOST [64*48] doubles, nullable) receives the trace
 * recorded so far (per pivot: entering kind/j, m, leaving, theta_min, #ties, pivot,
 * value, w-mask, z-mask, max|cbar|, slow-path flag, z0 value and coefficient, then
 * 16 entering coefficients and 16 values by pair index); the buffer is then cleared. */
ca_status ca_debug_trace(ca_problem* h, int64_t p, double* out);

const char* ca_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
