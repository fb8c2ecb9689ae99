// ca_sweep.cuh -- ADMM step 1 (Eq. 15) over all (scene, t, part,
// obstacle) pairs, one pair per thread, fused with step 3 of the previous
// iteration (Eq. 17) and the step-2 Gauss-Newton aggregates.
//
// Per pair: Eq. 19 rows at pose(s^k) -> Eqs. 20-21 elimination (index e =
// argmax b_i, reading #3) -> Eq. 24 LCP -> revised Lemke (ca_lemke.cuh) ->
// recovery y_e = (1 - sum_{k != e} b_k lambda_k)/b_e -> dual residual
// (Eq. 18b) and (v v^T, |g|^2, -eT v, g.eR) for the primal step, reduced per
// (scene, t) work-item records in a fixed order (no FP atomics).
//
// Scheduling: persistent, independent warps (WPC per CTA) pull work items -- 32
// slots of a scene's sort pool of TG timesteps, ordered by last pivot count -- from
// a counter.  Per-thread state that the pivot loop indexes at run time (basic-
// variable values, entering-column coefficients, reduced obstacle rows) lives in
// shared memory as [item][lane] (conflict-free); tableau-row labels are 4-bit
// fields of a register; the m x m structural system is in registers (m <= 3) or a
// shared-memory slot / local memory.  Rare cases (multi-way ties, an ineligible
// provisional minimum, failures, unverified answers) leave the pivot loop for the
// warp-cooperative dense Lemke, so the loop's instruction footprint and register
// pressure stay small; the pivot trace and the scaling-centre terms are a separate
// kernel variant (TRACE).
#pragma once
#include <cstdlib>
#include <mutex>

#include "ca_kernels.cuh"
#include "ca_lemke.cuh"

#ifndef CA_MAX_DEVICES
#define CA_MAX_DEVICES 64
#endif

#ifndef CA_EXP_M12
#define CA_EXP_M12 0  // 1: exact m = 1, 2 specialisations of the structural solve (-5 % instructions,
                      // +7 % time: the larger pivot loop misses the instruction cache, profiles/r02)
#endif
#ifndef CA_EXP_COLD
#define CA_EXP_COLD 1  // rare branches of the pivot loop marked unlikely (cold-code placement: -0.3..1 %)
#endif
#if CA_EXP_COLD
#define CA_RARE(c) __builtin_expect(!!(c), 0)
#else
#define CA_RARE(c) (c)
#endif
#ifndef CA_EXP_MU_PIPE
#define CA_EXP_MU_PIPE 0
#endif
#ifndef CA_EXP_P1MERGE
#define CA_EXP_P1MERGE 0
#endif
#ifndef CA_EXP_RESET
#define CA_EXP_RESET 0  // 1: drop tie candidates on a clearly lower new minimum (measured slower)
#endif
#ifndef CA_EXP_MU_UNROLL
#define CA_EXP_MU_UNROLL 1
#endif
#ifndef CA_SWEEP_PERSIST
#define CA_SWEEP_PERSIST 1  // persistent warps pulling work items (no per-CTA launch / retire gaps)
#endif
#ifndef CA_SWEEP_PREFETCH
#define CA_SWEEP_PREFETCH 0  // 1: claim the next work item one ahead, prefetch its pair data into L2 (C5: 23.16 -> 24.15 ms, dropped)
#endif
#ifndef CA_SWEEP_MINB
#define CA_SWEEP_MINB 16  // resident warps per SM the register budget targets
#endif
#ifndef CA_SWEEP_WPC
#define CA_SWEEP_WPC 2  // independent warps per CTA (halves the per-CTA shared-memory reserve)
#endif
#ifndef CA_SWEEP_GSLOTS
#define CA_SWEEP_GSLOTS 2  // per warp: lanes whose m > 3 system lives in shared memory
#endif

namespace ca {

constexpr int WPC = CA_SWEEP_WPC, GSLOTS = CA_SWEEP_GSLOTS;
constexpr int NPMAX = 8;   // robot parts per problem (validated)
constexpr int NRMAX = 16;  // faces per robot part (validated)
constexpr int MFAST = 3;   // m x m systems up to this size live in shared memory (99.7 % on C5)

// Tableau-row labels (L5.5 final tie-break): 4-bit fields of one register when
// they fit (NMAX <= 15: labels <= 14, slot NMAX holds z0's row), else bytes in smem.
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <int NMAX, bool REG = (NMAX <= 15)>
struct RowLab {
  uint64_t v;
  __device__ __forceinline__ void init(int) { v = 0xFEDCBA9876543210ull; }
  __device__ __forceinline__ int get(int i) const { return (int)((v >> (4 * i)) & 15u); }
  __device__ __forceinline__ void set(int i, int x) {
    v = (v & ~(0xFull << (4 * i))) | ((uint64_t)x << (4 * i));
  }
};
template <int NMAX>
struct RowLab<NMAX, false> {
  unsigned char* p;  // [item][thread] bytes
  __device__ __forceinline__ void init(int n) {
#pragma unroll 1
    for (int i = 0; i <= n; ++i) p[i * CTA] = (unsigned char)i;
  }
  __device__ __forceinline__ int get(int i) const { return p[i * CTA]; }
  __device__ __forceinline__ void set(int i, int x) { p[i * CTA] = (unsigned char)x; }
};

// Per-thread shared-memory column ([item][thread], conflict-free): the obstacle
// rows (sized by the problem's largest obstacle, `nomax`), basic values, entering-
// column coefficients, and the row labels when they do not fit a register; then the
// CTA-shared lambda-row table and the gamma / phi constant rows.
template <int D, int NMAX>
struct SweepSmem {
  static constexpr int VAL = NMAX, CB = NMAX;
  static constexpr int ROWB = (NMAX <= 15) ? 0 : (NMAX + 1 + 7) / 8;  // label bytes, in doubles
  static_assert(VAL + CB + (D + 1) * (D + 1) >= rec_n(D) + 1, "the record reduction reuses the per-thread columns");
  static __host__ __device__ int mu(int nomax) { return nomax * (D + 1); }
  static __host__ __device__ int rowb_off(int nomax) { return mu(nomax) + VAL + CB; }
  static __host__ __device__ int per_thread(int nomax) { return mu(nomax) + VAL + CB + ROWB; }
  static constexpr int GN = (D + 4) * (D + 5);  // one generic m x m system (m > 3)
  static size_t bytes(int np, int nrmax, int nomax) {
    return sizeof(double) * ((size_t)WPC * per_thread(nomax) * CTA + (size_t)np * (nrmax - 1) * (D + 2) +
                             2 * (D + 2) + (size_t)WPC * GSLOTS * GN);
  }
};

// One pivot of the diagnostic trace (ca_debug_trace); kept out of line so the
// pivot loop's instruction footprint does not carry it.
struct TraceRow {
  double v[14];
};
static __device__ __noinline__ void trace_pivot(double* dd, const TraceRow tr, const double* sval, const double* scb, int n) {
  for (int k = 0; k < 14; ++k) dd[k] = tr.v[k];
  for (int i = 0; i < n && i < 16; ++i) {
    dd[14 + i] = scb[i * CTA];
    dd[30 + i] = sval[i * CTA];
  }
}

// Textbook dense-tableau Lemke (rules L1-L7, FMA policy of reading #18) on the
// same reduced rows, solved by a whole warp for one pair: lane i owns tableau row
// i of [I | -M | -1 | q] (local memory), the pivot row is broadcast by shuffles,
// reductions (min / max / ballots) are exact, so the arithmetic is element for
// element that of a sequential dense Lemke.  The rare fallback when the revised
// path fails, meets a multi-way tie (lexicographic rule) or an ineligible
// provisional minimum, or its result does not verify.  Called by all 32 lanes;
// writes the basic z values of the pair into svalL (by LCP index, stride CTA).
// Proximal term of reading #2 (prox_eps > 0): (eps/2)||y - y^k||^2 added to Eq. 19a,
// through Eqs. 20-25: M_UU += eps (I + kt kt^T), q_U -= eps (y^k_U + kt (etatil - y^k_e)).
// y^k of the pair: y[k * PP + p], eliminated index e.
struct Prox {
  double eps;  // 0: off (paper-exact)
  const double* y;
  long long PP, p;
  int e;
};

template <int D, int NMAX>
__device__ __noinline__ int lemke_warp_lm(const PairRows<D> W, const double btil[D + 1], double be,  // @region lemke_dense
                                       LemkeParams LP, Prox X, double* svalL, int lane, uint32_t* zb_out, int* piv_out) {
  constexpr unsigned FULL = 0xffffffffu;
  const int n = W.n, l = n - 1;
  const int Wd = 2 * n + 2, Z0 = 2 * n, RHS = 2 * n + 1;
  const bool own = lane < n;
  double T[2 * NMAX + 2];
  int basis = lane;
  if (own) {
    const int i = lane;
    double fi[D + 1], ki;
    W.row(i, fi, ki);
    for (int j = 0; j < Wd; ++j) T[j] = 0.0;
    T[i] = 1.0;
    for (int j = 0; j < n; ++j) {
      double fj[D + 1], kj;
      W.row(j, fj, kj);
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) acc = __fma_rn(fi[c], fj[c], acc);
      if (j == l) acc = ki;
      if (i == l) acc = -kj;
      if (i == l && j == l) acc = 0.0;
      if (X.eps > 0.0 && i < l && j < l) acc = __fma_rn(X.eps, __fma_rn(ki, kj, (i == j) ? 1.0 : 0.0), acc);
      T[n + j] = -acc;
    }
    T[Z0] = -1.0;
    double q = 1.0 / be;
    if (i < l) {
      q = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) q = __fma_rn(fi[c], btil[c], q);
      if (X.eps > 0.0) {
        const double ye = X.y[(long long)X.e * X.PP + X.p], yu = X.y[(long long)(i + (i >= X.e)) * X.PP + X.p];
        q = __fma_rn(-X.eps, __fma_rn(ki, 1.0 / be - ye, yu), q);
      }
    }
    T[RHS] = q;
  }
  auto wmin = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
  };
  // L3 pivot on (row r, column c): row r / T[r][c]; other rows fma(-T_ic, T_rj, T_ij)
  auto pivot = [&](int r, int c) {
    const double inv = 1.0 / __shfl_sync(FULL, own ? T[c] : 0.0, r);
    if (lane == r)
      for (int j = 0; j < Wd; ++j)
        if (j != c) T[j] = T[j] * inv;
    const double f = own ? T[c] : 0.0;
    for (int j = 0; j < Wd; ++j) {
      const double rj = __shfl_sync(FULL, own ? T[j] : 0.0, r);
      if (own && lane != r && j != c) T[j] = __fma_rn(-f, rj, T[j]);
    }
    if (own) T[c] = (lane == r) ? 1.0 : 0.0;
  };
  const double tau = LP.tie_tol;
  int status = ST_OK, pivots = 0;
  const double qmin = wmin(own ? T[RHS] : 1e308);
  if (qmin < 0.0) {
    const double tl = qmin + tau * fmax(1.0, fabs(qmin));
    const int r = 31 - __clz(__ballot_sync(FULL, own && T[RHS] <= tl));  // ties -> largest index
    const int leaving = r;                                               // basis[r] = w_r
    pivot(r, Z0);
    if (lane == r) basis = Z0;
    ++pivots;
    int entering = leaving + n;
    const int maxpiv = LP.max_pivot_factor * n;
    for (;;) {
      if (pivots >= maxpiv) { status = ST_ITER; break; }
      const int col = entering;
      const double cmax = -wmin(own ? -fabs(T[col]) : 0.0);
      const double thr = LP.pivot_tol * fmax(1.0, cmax);
      const double ci = own ? T[col] : 0.0;
      const bool el = own && ci > thr;
      const double th = el ? fmax(T[RHS], 0.0) / ci : 1e308;
      const double thmin = wmin(th);
      if (!(thmin < 1e308)) { status = ST_RAY; break; }
      const double ttol = thmin + tau * fmax(1.0, thmin);
      uint32_t tie = __ballot_sync(FULL, el && th <= ttol);
      const uint32_t z0t = __ballot_sync(FULL, ((tie >> lane) & 1u) && basis == Z0);
      int r2;
      if (z0t) {
        r2 = __ffs(z0t) - 1;  // L5.3: z0 leaves whenever it is tied
      } else {
        for (int j = 0; j < n && __popc(tie) > 1; ++j) {  // L5.4: lexicographic on B^{-1}
          const bool in = (tie >> lane) & 1u;
          const double v = in ? T[j] / T[col] : 1e308;
          const double vmin = wmin(v);
          const double vt = vmin + tau * fmax(1.0, fabs(vmin));
          tie = __ballot_sync(FULL, in && v <= vt);
        }
        r2 = __ffs(tie) - 1;  // L5.5: smallest row
      }
      const int leaving2 = __shfl_sync(FULL, basis, r2);
      pivot(r2, col);
      if (lane == r2) basis = col;
      ++pivots;
      if (leaving2 == Z0) break;
      entering = (leaving2 < n) ? leaving2 + n : leaving2 - n;
    }
  }
  const bool zbas = own && basis >= n && basis < 2 * n;
  if (zbas) svalL[(basis - n) * CTA] = T[RHS];
  *zb_out = __reduce_or_sync(FULL, zbas ? (1u << (basis - n)) : 0u);
  *piv_out = pivots;
  return status;
}

template <int D, int NMAX>
__device__ __noinline__ int lemke_warp_reg(const PairRows<D> W, const double btil[D + 1], double be,  // @region lemke_dense
                                       LemkeParams LP, Prox X, double* svalL, int lane, uint32_t* zb_out, int* piv_out) {
  constexpr unsigned FULL = 0xffffffffu;
  // fixed column layout (every index compile-time, so the row stays in registers):
  // w_j at j, z_j at NMAX + j, z0 at Z0, q at RHS; columns of absent pairs j >= n
  // are skipped (they would stay zero)
  constexpr int Z0 = 2 * NMAX, RHS = 2 * NMAX + 1, WC = 2 * NMAX + 2;
  const int n = W.n, l = n - 1;
  const bool own = lane < n;
  auto used = [&](int j) { return (j < NMAX) ? (j < n) : (j < 2 * NMAX ? (j - NMAX < n) : true); };
  double T[WC];
  int basis = lane;  // w_lane
  {
    double fi[D + 1], ki = 0.0;
    if (own) W.row(lane, fi, ki);
#pragma unroll
    for (int j = 0; j < WC; ++j) T[j] = 0.0;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
      if (j >= n) continue;
      T[j] = (j == lane) ? 1.0 : 0.0;
      if (own) {
        double fj[D + 1], kj;
        W.row(j, fj, kj);
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c <= D; ++c) acc = __fma_rn(fi[c], fj[c], acc);
        if (j == l) acc = ki;
        if (lane == l) acc = -kj;
        if (lane == l && j == l) acc = 0.0;
        if (X.eps > 0.0 && lane < l && j < l) acc = __fma_rn(X.eps, __fma_rn(ki, kj, (lane == j) ? 1.0 : 0.0), acc);
        T[NMAX + j] = -acc;
      }
    }
    T[Z0] = -1.0;
    double q = 1.0 / be;
    if (lane < l) {
      q = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) q = __fma_rn(fi[c], btil[c], q);
      if (X.eps > 0.0) {
        const double ye = X.y[(long long)X.e * X.PP + X.p], yu = X.y[(long long)(lane + (lane >= X.e)) * X.PP + X.p];
        q = __fma_rn(-X.eps, __fma_rn(ki, 1.0 / be - ye, yu), q);
      }
    }
    T[RHS] = q;
    if (!own) {
#pragma unroll
      for (int j = 0; j < WC; ++j) T[j] = 0.0;
    }
  }
  auto wmin = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
  };
  // min / max over the warp of NON-NEGATIVE doubles, exactly, by two integer reductions
  // on the bit patterns (for x, y >= 0 the IEEE order is the unsigned (hi, lo) order)
  auto wmin_nn = [&](double v) {
    const unsigned long long u = __double_as_longlong(v == 0.0 ? 0.0 : v);  // -0 -> +0
    const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
    const unsigned mh = __reduce_min_sync(FULL, hi);
    const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  };
  auto wmax_nn = [&](double v) {
    const unsigned long long u = __double_as_longlong(v == 0.0 ? 0.0 : v);  // -0 -> +0
    const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
    const unsigned mh = __reduce_max_sync(FULL, hi);
    const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  };
  auto col = [&](int c) {  // T[c] for a run-time column c: four short select chains, then one
    constexpr int GS = (WC + 3) / 4;  // of them (dependent depth GS + 3 instead of WC)
    double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < WC; ++j) v[j / GS] = (j == c) ? T[j] : v[j / GS];
    return (c < GS) ? v[0] : (c < 2 * GS) ? v[1] : (c < 3 * GS) ? v[2] : v[3];
  };
  // L3 pivot on (row r, column c), tc = this lane's T[c] and rc = 1 / tc (formed by every
  // lane beforehand, off the chain; lane r's is the one division of the rule): row r
  // scaled by it, other rows fma(-T_ic, T_rj, T_ij)
  auto pivot = [&](int r, int c, double tc, double rc) {
    const double inv = __shfl_sync(FULL, own ? rc : 0.0, r);
    if (lane == r) {
#pragma unroll
      for (int j = 0; j < WC; ++j)
        if (used(j) && j != c) T[j] = T[j] * inv;
    }
    const double f = own ? tc : 0.0;
#pragma unroll
    for (int j = 0; j < WC; ++j) {
      if (!used(j)) continue;
      const double rj = __shfl_sync(FULL, own ? T[j] : 0.0, r);
      if (own && lane != r && j != c) T[j] = __fma_rn(-f, rj, T[j]);
    }
#pragma unroll
    for (int j = 0; j < WC; ++j)
      if (j == c && own) T[j] = (lane == r) ? 1.0 : 0.0;
  };
  const double tau = LP.tie_tol;
  int status = ST_OK, pivots = 0;
  const double qmin = wmin(own ? T[RHS] : 1e308);
  if (qmin < 0.0) {
    const double tl = qmin + tau * fmax(1.0, fabs(qmin));
    const int r = 31 - __clz(__ballot_sync(FULL, own && T[RHS] <= tl));  // ties -> largest index
    const int leaving = r;                                               // basis[r] = w_r
    pivot(r, Z0, T[Z0], 1.0 / T[Z0]);
    if (lane == r) basis = Z0;
    ++pivots;
    int entering = NMAX + leaving;  // z_r
    const int maxpiv = LP.max_pivot_factor * n;
    for (;;) {
      if (pivots >= maxpiv) { status = ST_ITER; break; }
      const double ci = own ? col(entering) : 0.0;
      const double cmax = wmax_nn(fabs(ci));
      const double thr = LP.pivot_tol * fmax(1.0, cmax);
      const bool el = own && ci > thr;
      const double th = el ? fmax(T[RHS], 0.0) / ci : 1e308;
      const double rci = 1.0 / ci;  // the pivot's reciprocal if this row leaves
      const double thmin = wmin_nn(th);
      if (!(thmin < 1e308)) { status = ST_RAY; break; }
      const double ttol = thmin + tau * fmax(1.0, thmin);
      uint32_t tie = __ballot_sync(FULL, el && th <= ttol);
      const uint32_t z0t = __ballot_sync(FULL, ((tie >> lane) & 1u) && basis == Z0);
      int r2;
      if (z0t) {
        r2 = __ffs(z0t) - 1;  // L5.3: z0 leaves whenever it is tied
      } else {
#pragma unroll
        for (int j = 0; j < NMAX; ++j) {  // L5.4: lexicographic on B^{-1} (the w columns)
          if (j >= n || __popc(tie) <= 1) break;
          const bool in = (tie >> lane) & 1u;
          const double v = in ? T[j] / ci : 1e308;
          const double vmin = wmin(v);
          const double vt = vmin + tau * fmax(1.0, fabs(vmin));
          tie = __ballot_sync(FULL, in && v <= vt);
        }
        r2 = __ffs(tie) - 1;  // L5.5: smallest row
      }
      const int leaving2 = __shfl_sync(FULL, basis, r2);
      pivot(r2, entering, ci, rci);
      if (lane == r2) basis = entering;
      ++pivots;
      if (leaving2 == Z0) break;
      entering = (leaving2 < NMAX) ? leaving2 + NMAX : leaving2 - NMAX;  // complement (L4)
    }
  }
  const bool zbas = own && basis >= NMAX && basis < 2 * NMAX;
  if (zbas) svalL[(basis - NMAX) * CTA] = T[RHS];
  *zb_out = __reduce_or_sync(FULL, zbas ? (1u << (basis - NMAX)) : 0u);
  *piv_out = pivots;
  return status;
}

// The two forms compute the same thing element for element.  The register-tableau
// form (every column index compile-time) is the faster one for a warp that does
// little else (the extended variant: latency mode, centres, tracing); the production
// kernel keeps the local-memory form, whose call site costs the hot loop no
// registers (the register form would make the sweep spill: +11 % on C5).
template <int D, int NMAX, bool REG>
__device__ __forceinline__ int lemke_warp(const PairRows<D> W, const double btil[D + 1], double be, LemkeParams LP,
                                          Prox X, double* svalL, int lane, uint32_t* zb_out, int* piv_out) {
  if constexpr (REG) return lemke_warp_reg<D, NMAX>(W, btil, be, LP, X, svalL, lane, zb_out, piv_out);
  else return lemke_warp_lm<D, NMAX>(W, btil, be, LP, X, svalL, lane, zb_out, piv_out);
}

// ---------------------------------------------------------------------------
// NEXT f4: the prox-regularised pair QP of reading #2,
//   min_y 1/2 ||K^T y + bvec||^2 + eps/2 ||y - y^k||^2   s.t. y >= 0, kappa^T y = 1
// (Eq. 19 with kappa = (b_i, 0, 0), eta = 1, plus the proximal term), solved
// through its dual in R^{d+1}.  With u = K^T y + bvec and 1/2||u||^2 = max_w w.u - 1/2||w||^2,
//   g(w) = w.bvec - 1/2||w||^2 + min_{y in Y} [(K w).y + eps/2 ||y - y^k||^2]
// is concave with gradient u(w) - w, where y(w) = Pi_Y(y^k - K w / eps) is a Euclidean
// projection onto Y = {y >= 0, kappa^T y = 1}: mu and gamma entries are clipped at 0,
// the lambda entries are y_k = max(0, c_k - tau b_k) with tau fixed by b^T y_lambda = 1
// (variable fixing: drop the entries that go non-positive, recompute tau, until
// stable).  The minimiser is y(w*) at the unique fixed point w* = u(w*) (= u*).
// Semismooth Newton on u(w) - w = 0: the projection's Jacobian on the current support
// S gives H = I + (1/eps) [sum_{k in S} K_k K_k^T - s s^T / (b_F . b_F)], s = sum_{k in F}
// b_k K_k (F = lambda support), a (d+1) x (d+1) SPD system; an Armijo line search on g
// (quadratic-interpolation backtracking) makes it global.  A full step that keeps the
// support lands on the affine piece's root, which ends the iteration (finite
// termination).  Warm start: w = u(y^k).
// The oracle solves the same strictly convex QP with the dense Lemke (orc_pair_solve
// with prox_eps), so the two agree to rounding only (no shared algorithm).
// Rows: lambda_k (0, a_k), b_k = prow[4k+3]; mu_l the per-lane smem rows (stride CTA);
// gamma (1, 0).  y^k in ykc (stride CTA); y(w) written to yout (stride CTA) by index k.
#ifndef CA_PROX_MAXIT
#define CA_PROX_MAXIT 64  // Newton iterations before the dense-Lemke re-solve (20: no gain, profiles)
#endif

template <int D>
struct ProxNt {
  double g, u[D + 1], H[(D + 1) * (D + 2) / 2];
  uint32_t sup;  // support of y(w) (bit k: y_k > 0)
};

template <int D>
__device__ __forceinline__ void prox_row(int k, int nr, int no, const double* prow, const double* mu,
                                         double f[D + 1]) {
  if (k < nr) {
    f[0] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) f[1 + a] = prow[4 * k + a];
  } else if (k < nr + no) {
    const double* m = mu + (k - nr) * (D + 1) * CTA;
#pragma unroll
    for (int c = 0; c <= D; ++c) f[c] = m[c * CTA];
  } else {
    f[0] = 1.0;
#pragma unroll
    for (int a = 0; a < D; ++a) f[1 + a] = 0.0;
  }
}

template <int D>
__device__ __forceinline__ void prox_eval(const double* prow, const double* mu, int nr, int no, const double bv[D + 1],
                                       double eps, double ie, const double* ykc, const double w[D + 1],
                                       double* yout, ProxNt<D>& E) {
  constexpr int L1 = D + 1;
  const int n = nr + no + 1;  // ie = 1 / eps (hoisted by the caller)
  // lambda block: variable fixing for tau (b^T y_lambda = 1)
  uint32_t F = (nr >= 32) ? 0xffffffffu : ((1u << nr) - 1u);
  double tau = 0.0, sbb = 0.0;
#pragma unroll 1
  for (int pass = 0; pass <= nr; ++pass) {
    double sb = 0.0;
    sbb = 0.0;
#pragma unroll 1
    for (uint32_t bb = F; bb; bb &= bb - 1) {
      const int k = __ffs(bb) - 1;
      double kw = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) kw = __fma_rn(prow[4 * k + a], w[1 + a], kw);
      const double c = __fma_rn(-ie, kw, ykc[k * CTA]), bk = prow[4 * k + 3];
      sb = __fma_rn(bk, c, sb);
      sbb = __fma_rn(bk, bk, sbb);
    }
    tau = (sb - 1.0) / sbb;
    uint32_t F2 = 0;
#pragma unroll 1
    for (uint32_t bb = F; bb; bb &= bb - 1) {
      const int k = __ffs(bb) - 1;
      double kw = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) kw = __fma_rn(prow[4 * k + a], w[1 + a], kw);
      const double c = __fma_rn(-ie, kw, ykc[k * CTA]);
      if (__fma_rn(-tau, prow[4 * k + 3], c) > 0.0) F2 |= 1u << k;
    }
    if (F2 == F || F2 == 0u) break;
    F = F2;
  }
  // one pass over every row: y(w), u = K^T y + bvec, g, the Newton matrix
  double u[L1], Hs[L1 * (L1 + 1) / 2], s[L1], gs = 0.0;
#pragma unroll
  for (int c = 0; c < L1; ++c) { u[c] = bv[c]; s[c] = 0.0; }
#pragma unroll
  for (int c = 0; c < L1 * (L1 + 1) / 2; ++c) Hs[c] = 0.0;
  uint32_t sup = 0;
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    double f[L1];
    prox_row<D>(k, nr, no, prow, mu, f);
    double kw = 0.0;
#pragma unroll
    for (int c = 0; c < L1; ++c) kw = __fma_rn(f[c], w[c], kw);
    const double yk = ykc[k * CTA], c0 = __fma_rn(-ie, kw, yk);
    double y = 0.0;
    if (k < nr) {
      if ((F >> k) & 1u) y = fmax(__fma_rn(-tau, prow[4 * k + 3], c0), 0.0);
    } else {
      y = fmax(c0, 0.0);
    }
    yout[k * CTA] = y;
    const double dy = y - yk;
    gs = __fma_rn(kw, y, gs);
    gs = __fma_rn(0.5 * eps, dy * dy, gs);
    if (y > 0.0) {
      sup |= 1u << k;
      int h = 0;
#pragma unroll
      for (int a = 0; a < L1; ++a) {
        u[a] = __fma_rn(y, f[a], u[a]);
#pragma unroll
        for (int c = a; c < L1; ++c, ++h) Hs[h] = __fma_rn(f[a], f[c], Hs[h]);
      }
      if (k < nr) {
        const double bk = prow[4 * k + 3];
#pragma unroll
        for (int a = 0; a < L1; ++a) s[a] = __fma_rn(bk, f[a], s[a]);
      }
    }
  }
  double sbF = 0.0;  // b_F . b_F over the final lambda support
#pragma unroll 1
  for (uint32_t bb = sup & ((nr >= 32) ? 0xffffffffu : ((1u << nr) - 1u)); bb; bb &= bb - 1) {
    const double bk = prow[4 * (__ffs(bb) - 1) + 3];
    sbF = __fma_rn(bk, bk, sbF);
  }
  const double isb = sbF > 0.0 ? 1.0 / sbF : 0.0;
  double gw = 0.0;
  int h = 0;
#pragma unroll
  for (int a = 0; a < L1; ++a) {
    gw = __fma_rn(w[a], bv[a] - 0.5 * w[a], gw);
    E.u[a] = u[a];
#pragma unroll
    for (int c = a; c < L1; ++c, ++h) {
      const double t = __fma_rn(-s[a] * isb, s[c], Hs[h]);
      E.H[h] = __fma_rn(ie, t, a == c ? 1.0 : 0.0);
    }
  }
  E.g = gw + gs;
  E.sup = sup;
}

// x = A^{-1} r for the packed (upper, row by row) SPD (d+1) x (d+1) matrix A: Cholesky
// with reciprocal diagonal, forward and back substitution.
template <int L1>
__device__ __forceinline__ void prox_chol_solve(const double* Ap, const double r[L1], double x[L1]) {
  double Lm[L1][L1], idg[L1];
  int h = 0;
#pragma unroll
  for (int a = 0; a < L1; ++a)
#pragma unroll
    for (int c = a; c < L1; ++c, ++h) Lm[c][a] = Ap[h];
#pragma unroll
  for (int j = 0; j < L1; ++j) {
    double dj = Lm[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) dj = __fma_rn(-Lm[j][k], Lm[j][k], dj);
    dj = sqrt(dj);
    const double idj = 1.0 / dj;
    idg[j] = idj;
#pragma unroll
    for (int i = j + 1; i < L1; ++i) {
      double v = Lm[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v = __fma_rn(-Lm[i][k], Lm[j][k], v);
      Lm[i][j] = v * idj;
    }
  }
#pragma unroll
  for (int i = 0; i < L1; ++i) {
    double v = r[i];
#pragma unroll
    for (int k = 0; k < i; ++k) v = __fma_rn(-Lm[i][k], x[k], v);
    x[i] = v * idg[i];
  }
#pragma unroll
  for (int i = L1 - 1; i >= 0; --i) {
    double v = x[i];
#pragma unroll
    for (int k = i + 1; k < L1; ++k) v = __fma_rn(-Lm[k][i], x[k], v);
    x[i] = v * idg[i];
  }
}

// Returns the Newton iteration count (>= 1) on success, -1 when the iteration did not
// converge (the caller re-solves the pair with the dense Lemke).  y in yout by index k.
// Warm start across ADMM iterations: the root of the affine piece of y^k's support S0,
// (I + K^T J_S0 K / eps) w = u(y^k) - s (b_F.y^k_F - 1) / (b_F.b_F) -- exact when the
// support has not changed since the previous iteration (then one evaluation confirms).
template <int D>
__device__ __noinline__ int prox_newton_pair(const double* prow, const double* mu, int nr, int no,
                                             const double bv[D + 1], double eps, const double* ykc, double* yout) {
  constexpr int L1 = D + 1;
  const int n = nr + no + 1;
  const double ie = 1.0 / eps;
  double w[L1];
#pragma unroll
  for (int c = 0; c < L1; ++c) w[c] = bv[c];
  {
    double Hs[L1 * (L1 + 1) / 2], s[L1], sbF = 0.0, bdy = 0.0;
#pragma unroll
    for (int c = 0; c < L1; ++c) s[c] = 0.0;
#pragma unroll
    for (int c = 0; c < L1 * (L1 + 1) / 2; ++c) Hs[c] = 0.0;
#pragma unroll 1
    for (int k = 0; k < n; ++k) {  // u(y^k) and the support's Newton matrix
      const double yk = ykc[k * CTA];
      if (yk > 0.0) {
        double f[L1];
        prox_row<D>(k, nr, no, prow, mu, f);
        int h = 0;
#pragma unroll
        for (int a = 0; a < L1; ++a) {
          w[a] = __fma_rn(yk, f[a], w[a]);
#pragma unroll
          for (int c = a; c < L1; ++c, ++h) Hs[h] = __fma_rn(f[a], f[c], Hs[h]);
        }
        if (k < nr) {
          const double bk = prow[4 * k + 3];
#pragma unroll
          for (int a = 0; a < L1; ++a) s[a] = __fma_rn(bk, f[a], s[a]);
          sbF = __fma_rn(bk, bk, sbF);
          bdy = __fma_rn(bk, yk, bdy);
        }
      }
    }
    if (sbF > 0.0) {
      const double isb = 1.0 / sbF, cr = (bdy - 1.0) * isb;
      double A[L1 * (L1 + 1) / 2], rhs[L1];
      int h = 0;
#pragma unroll
      for (int a = 0; a < L1; ++a) {
        rhs[a] = __fma_rn(-cr, s[a], w[a]);
#pragma unroll
        for (int c = a; c < L1; ++c, ++h) {
          const double t = __fma_rn(-s[a] * isb, s[c], Hs[h]);
          A[h] = __fma_rn(ie, t, a == c ? 1.0 : 0.0);
        }
      }
      prox_chol_solve<L1>(A, rhs, w);
    }
  }
  ProxNt<D> E, E2;
  prox_eval<D>(prow, mu, nr, no, bv, eps, ie, ykc, w, yout, E);
#pragma unroll 1
  for (int it = 1; it <= CA_PROX_MAXIT; ++it) {
    double r[L1], rn = 0.0, sc = 1.0;
#pragma unroll
    for (int c = 0; c < L1; ++c) {
      r[c] = E.u[c] - w[c];
      rn = fmax(rn, fabs(r[c]));
      sc = fmax(sc, fabs(w[c]));
    }
    if (rn <= 1e-15 * sc) return it;
    double dx[L1];
    prox_chol_solve<L1>(E.H, r, dx);
    double slope = 0.0;
#pragma unroll
    for (int c = 0; c < L1; ++c) slope = __fma_rn(r[c], dx[c], slope);
    double t = 1.0, wt[L1];
    int ls = 0;
#pragma unroll 1
    for (;; ++ls) {
#pragma unroll
      for (int c = 0; c < L1; ++c) wt[c] = __fma_rn(t, dx[c], w[c]);
      prox_eval<D>(prow, mu, nr, no, bv, eps, ie, ykc, wt, yout, E2);
      if (E2.g >= E.g + 1e-4 * t * slope - 1e-14 * (1.0 + fabs(E.g)) || ls >= 40) break;
      // backtrack to the maximiser of the quadratic through g(0), g'(0), g(t), in [t/10, t/2]
      const double den = 2.0 * (slope * t - (E2.g - E.g));
      const double tq = den > 0.0 ? slope * t * t / den : 0.5 * t;
      t = fmin(fmax(tq, 0.1 * t), 0.5 * t);
    }
    const bool same = (ls == 0 && E2.sup == E.sup);
#pragma unroll
    for (int c = 0; c < L1; ++c) w[c] = wt[c];
    E = E2;
    if (same) {  // full step inside one affine piece: the root (verify the residual)
      double rn2 = 0.0;
#pragma unroll
      for (int c = 0; c < L1; ++c) rn2 = fmax(rn2, fabs(E.u[c] - w[c]));
      return (rn2 <= 1e-9 * sc) ? it : -1;
    }
  }
  return -1;
}

template <int D, int NMAX, bool FUSED, bool TRACE>
__global__ void __launch_bounds__(CTA * WPC, CA_SWEEP_MINB / WPC) k_sweep(Dev P) {  // @region cta_setup
  using SM = SweepSmem<D, NMAX>;
  constexpr int L1 = D + 1;
  constexpr int RECD = rec_n(D), NAGG = rec_nagg(D);  // record: aggregates | statistics
  extern __shared__ double smem[];
  const int tid = threadIdx.x & 31, warp = threadIdx.x >> 5;  // lane; warps are independent
  const int PT = SM::per_thread(P.nomax);
  double* wcol = smem + (long long)warp * PT * CTA;  // this warp's [item][lane] columns
  double* mu = wcol + tid;
  double* sval = mu + SM::mu(P.nomax) * CTA;
  double* scb = sval + SM::VAL * CTA;
  RowLab<NMAX> rowb;
  if constexpr (NMAX > 15)  // tableau-row labels as bytes, [item][lane] from the region base
    rowb.p = reinterpret_cast<unsigned char*>(wcol + SM::rowb_off(P.nomax) * CTA) + tid;
  double* lamtab = smem + (long long)WPC * PT * CTA;  // [np][nrmax-1][D+2]
  const int LT = (P.nrmax - 1) * (D + 2);
  double* cst = lamtab + P.np * LT;  // gamma row (1, 0, .., 0), phi row 0
  double* gpool = cst + 2 * (D + 2) + (long long)warp * GSLOTS * SM::GN;  // m > 3 systems
  // the lambda-row table (k_lamtab) and the constant rows: plain copies
#pragma unroll 1
  for (int k = threadIdx.x; k < P.np * LT; k += CTA * WPC) lamtab[k] = P.lam[k];
  if (threadIdx.x < 2 * (D + 2)) cst[threadIdx.x] = (threadIdx.x == 0) ? 1.0 : 0.0;
  __syncthreads();
#ifdef CA_CHECKED
#define VAL(i) sval[(CA_CHECK((i) >= 0 && (i) < NMAX), (i)) * CTA]
#define CBV(i) scb[(CA_CHECK((i) >= 0 && (i) < NMAX), (i)) * CTA]
#define YK(i) P.y[(long long)(CA_CHECK((i) >= 0 && (i) < P.ny && p >= 0 && p < PP), (i)) * PP + p]
#else
#define VAL(i) sval[(i) * CTA]
#define CBV(i) scb[(i) * CTA]
#define YK(i) P.y[(long long)(i) * PP + p]  // y^k from HBM (L1-resident re-reads)
#endif
#if CA_SWEEP_PERSIST
  // persistent warps: every warp pulls (b, group, chunk) work items from a
  // counter (reset by k_sortpairs); results depend only on the item, not on which
  // warp ran it, so the order of the pulls does not change any output bit.  With
  // CA_SWEEP_PREFETCH the next item is claimed one ahead and its pairs' y^k, zeta, xi
  // and pose lines are prefetched into L2 while this item is solved.
  int nxt = 0;
  if (CA_SWEEP_PREFETCH) {
    if (tid == 0) nxt = atomicAdd(P.work, 1);
    nxt = __shfl_sync(0xffffffffu, nxt, 0);
  }
  for (;;) {
  int item = 0;
  if (CA_SWEEP_PREFETCH) {
    item = nxt;
    if (item >= P.nitems) break;
    int n2 = 0;
    if (tid == 0) n2 = atomicAdd(P.work, 1);
    nxt = __shfl_sync(0xffffffffu, n2, 0);
  } else {
    if (tid == 0) item = atomicAdd(P.work, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= P.nitems) break;
  }
#else
  for (int item = blockIdx.x * WPC + warp, once = 1; once && item < P.nitems; once = 0) {
#endif
  // item = (scene b, group of TG timesteps, chunk of 32 slots of its sort pool)
  const Item it = item_of(P, item);
  const int b = it.b;
  if (!scene_on(P, b)) continue;  // stopped scene (ca_admm_solve): frozen, no record
  // this pair's record: the double fields (aggregates, r_dual, r_pri) staged for the
  // lane-ordered reduction; the integer statistics (pivots, failure kinds) reduced
  // exactly by warp integer reductions
  constexpr int NDBL = NAGG + 2;
  double rec[NDBL];
#pragma unroll
  for (int f = 0; f < NDBL; ++f) rec[f] = 0.0;
  int ist[5] = {0, 0, 0, 0, 0};  // pivots, fail, ray, iter_limit, neg_ye
  const int gs = it.chunk * P.CHG + tid;  // slot in the group's execution order
  int tl = -1;                            // this lane's timestep within the group
  // pair state shared by the two halves of the pair's work (around the warp's
  // dense re-solves)
  const long long PP = P.P;
  long long p = 0;
  int ip = 0, nr = 0, no = 0, n = 0, e = 0, pivots = 0, status = ST_OK;
  double be = 1.0, zeta = 0.0, xi[D], bt_[D + 1];
  const double* po = P.pose;
  const double* prow = P.part_rows;
  uint32_t zb = 0;
  bool z0b = false, fallback = false;
  const uint32_t pk = (tid < P.CHG && gs < it.size) ? P.gperm2[((long long)b * P.NG + it.grp) * P.GG + gs]
                                                    : PAIR_UNSENSED;
  // the next item's pair of this lane (prefetch, CA_SWEEP_PREFETCH): its slot, loaded now
  uint32_t pk2 = PAIR_UNSENSED;
  int b2 = 0, grp2 = 0;
#if CA_SWEEP_PERSIST
  if (CA_SWEEP_PREFETCH && nxt < P.nitems) {
    const Item i2 = item_of(P, nxt);
    const int gs2 = i2.chunk * P.CHG + tid;
    b2 = i2.b;
    grp2 = i2.grp;
    if (tid < P.CHG && gs2 < i2.size) pk2 = P.gperm2[((long long)b2 * P.NG + grp2) * P.GG + gs2];
  }
#endif
#ifndef CA_EXP_NO_SENSE
  const bool act = !(pk & PAIR_UNSENSED);  // padding lane or unsensed obstacle (NEXT f3): idle
#else
  const bool act = tid < P.CHG && gs < it.size;
#endif
  if (act) {
    int j;
    unpack_pair(pk, tl, ip, j);
    CA_CHECK(ip < P.np && j < P.M && tl < it.nt && item < P.nitems);
    const int g = ip * P.M + j;
    const long long bt = (long long)b * P.N + it.grp * P.TG + tl;  // b*N + (t-1)
    po = P.pose + bt * 12;                                        // pose(s_t^k) (k_sortpairs)
    p = bt * P.G + g;
    const int r0 = P.part_off[ip];
    nr = P.part_off[ip + 1] - r0;
    const int o = b * P.M + j, l0 = P.obs_off[o];
    no = P.obs_off[o + 1] - l0;
    CA_CHECK(p < PP && no >= 1 && no <= P.nomax && nr <= P.nrmax && nr + no + 1 <= NMAX && nr + no + 1 <= P.ny);
    n = nr + no + 1;
    prow = P.part_rows + 4 * r0;
    const double* orow = P.obs_rows + 4 * (long long)l0;
    e = P.part_e[ip];
    be = P.part_be[ip];
    zeta = P.zeta[p];  // @region pair_setup
#pragma unroll
    for (int a = 0; a < D; ++a) xi[a] = P.xi[(long long)a * PP + p];
    // obstacle rows of K at pose(s^k) (Eq. 19b): (d_l - c_l.rho, R^T c_l)
    double sR[D * D], srho[D];
#pragma unroll
    for (int a = 0; a < D * D; ++a) sR[a] = po[a];
#pragma unroll
    for (int a = 0; a < D; ++a) srho[a] = po[9 + a];
    if constexpr (TRACE) part_origin<D>(P, ip, sR, srho);      // scaling centre (NEXT f3)
    obstacle_frame<D>(P, b, j, it.grp * P.TG + tl + 1, srho);  // moving obstacles (NEXT f3)
#pragma unroll 1
    for (int lo = 0; lo < no; ++lo) {
      const double4 cr = *reinterpret_cast<const double4*>(orow + 4 * lo);
      const double c[3] = {cr.x, cr.y, cr.z};
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) acc = __fma_rn(c[a], srho[a], acc);
      double* m = mu + lo * L1 * CTA;
      m[0] = cr.w - acc;
#pragma unroll
      for (int mm = 0; mm < D; ++mm) {
        double r = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) r = __fma_rn(c[a], sR[a * D + mm], r);
        m[(1 + mm) * CTA] = r;
      }
    }
    const PairRows<D> W{lamtab + ip * LT, cst, mu, CTA, nr, no, n, n - 1};
    if (FUSED) {  // @region fused_mult
      // Eq. 17 for the previous iteration at s^k with y^k (Eqs. 10-11); y^k is
      // staged in the (still unused) cbar scratch with batched loads
#pragma unroll 4
      for (int k = 0; k < n; ++k) CBV(k) = YK(k);
      double Tv = 1.0, Rv[D];
#pragma unroll
      for (int a = 0; a < D; ++a) Rv[a] = 0.0;
#pragma unroll 1
      for (int k = 0; k < nr; ++k) {
        const double yv = CBV(k);
#pragma unroll
        for (int a = 0; a < D; ++a) Rv[a] = __fma_rn(yv, prow[4 * k + a], Rv[a]);
      }
#pragma unroll 1
      for (int k = nr; k < nr + no; ++k) {
        const double yv = CBV(k);
        const double* m = mu + (k - nr) * L1 * CTA;
        Tv = __fma_rn(yv, m[0], Tv);
#pragma unroll
        for (int a = 0; a < D; ++a) Rv[a] = __fma_rn(yv, m[(1 + a) * CTA], Rv[a]);
      }
      Tv += CBV(nr + no);
      zeta += Tv;
      double r2 = Tv * Tv;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        xi[a] += Rv[a];
        r2 = __fma_rn(Rv[a], Rv[a], r2);
      }
      rec[NAGG + S_RPRI] = r2;
      P.zeta[p] = zeta;
#pragma unroll
      for (int a = 0; a < D; ++a) P.xi[(long long)a * PP + p] = xi[a];
    }
    // q = [Kt btil; etatil]  with btil = bvec + K_e / b_e, etatil = 1 / b_e (Eq. 25)  // @region q_build
    bt_[0] = (1.0 + zeta) + 0.0 / be;
#pragma unroll
    for (int a = 0; a < D; ++a) bt_[1 + a] = xi[a] + prow[4 * e + a] / be;
    double qmin = 1.0 / be;
    VAL(n - 1) = qmin;
#pragma unroll 1
    for (int i = 0; i < n - 1; ++i) {
      double f[D + 1], k;
      W.row(i, f, k);
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) acc = __fma_rn(f[c], bt_[c], acc);
      VAL(i) = acc;
      qmin = fmin(qmin, acc);
    }
    if (CA_SWEEP_PREFETCH && !(pk2 & PAIR_UNSENSED)) {  // the next item's pair data into L2
      int tl2, ip2, j2;
      unpack_pair(pk2, tl2, ip2, j2);
      const long long bt2 = (long long)b2 * P.N + grp2 * P.TG + tl2;
      const long long p2 = bt2 * P.G + ip2 * P.M + j2;
      prefetch_l2(P.zeta + p2);
#pragma unroll
      for (int a = 0; a < D; ++a) prefetch_l2(P.xi + (long long)a * PP + p2);
#pragma unroll 1
      for (int k = 0; k < P.ny; ++k) prefetch_l2(P.y + (long long)k * PP + p2);
      prefetch_l2(P.pose + bt2 * 12);
    }
    // ------------------------------------------------------------------ Lemke  // @region lemke_init
    const LemkeParams& LP = P.lp;
    const double tau = LP.tie_tol, ptol = LP.pivot_tol;
    const uint32_t nmask = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
    uint32_t wb = nmask;
    zb = 0;
    z0b = false;
    double val0 = 0.0;
    pivots = 0;
    status = ST_OK;
    rowb.init(n);
    bool nwt_fail = false;
    if (TRACE && P.prox_newton) {  // NEXT f4: prox_eps > 0 by the dual Newton method, one pair per lane
      if (!FUSED) {  // y^k staged in the cbar scratch (the fused multiplier step already did)
#pragma unroll 4
        for (int k = 0; k < n; ++k) CBV(k) = YK(k);
      }
      double bv[D + 1];
      bv[0] = 1.0 + zeta;
#pragma unroll
      for (int a = 0; a < D; ++a) bv[1 + a] = xi[a];
      const int its = prox_newton_pair<D>(prow, mu, nr, no, bv, P.prox_eps, &CBV(0), &VAL(0));
      nwt_fail = its < 0;
      pivots = its < 0 ? 0 : its;
      // y by index k -> the recovery's LCP layout (index u = k - (k > e), support bits)
#pragma unroll 1
      for (int k = 0; k < n; ++k) {
        if (k == e) continue;
        const int u = k - (k > e);
        const double yv = VAL(k);
        VAL(u) = yv;
        if (yv > 0.0) zb |= 1u << u;
      }
    } else if (qmin < 0.0 && !(TRACE && P.dense)) {  // L1: otherwise z = 0 (latency mode: dense solve below)
      // L2: z0 enters at row argmin q (ties -> largest index); its column is -1
      const double tl = qmin + tau * fmax(1.0, fabs(qmin));
      int r = 0;
#pragma unroll 1
      for (int i = 0; i < n; ++i)
        if (VAL(i) <= tl) r = i;
      const double ve = VAL(r) * -1.0;
#pragma unroll 1
      for (int i = 0; i < n; ++i)
        if (i != r) VAL(i) = __fma_rn(1.0, ve, VAL(i));
      wb &= ~(1u << r);
      z0b = true;
      val0 = ve;
      rowb.set(NMAX, r);
      pivots = 1;
      Var ent{1, r};
      const int maxpiv = LP.max_pivot_factor * n;
      double Gslow[(D + 4) * (D + 5)];
      const double kInf = __longlong_as_double(0x7ff0000000000000LL);
      const double tauS = tau + 1e-12;  // candidate band: tie tolerance + superset margin (filtered exactly)
      const double* lt = lamtab + ip * LT;
      const int nr1 = nr - 1;
      uint32_t pend = 0;  // rows still owing the previous pivot's value update
      double ve2p = 0.0;
      for (;;) {
        if (CA_RARE(pivots >= maxpiv)) { status = ST_ITER; break; }
        if (CA_RARE(n - __popc(wb) > D + 4)) { status = ST_ITER; break; }  // rank bound (cannot happen exactly)
        // structural m x m system: registers for m <= 3, generic solver otherwise
        SmallSol<D> ss;  // @region solve_call
        bool small = true;
#if CA_EXP_M12
        {
          const uint32_t Rm = ~wb & nmask;
          const int mr = __popc(Rm);
          if (mr == 1) solve_m1<D>(W, Rm, zb, z0b, ent, ss);
          else if (mr == 2) solve_m2<D>(W, Rm, zb, z0b, ent, ss);
          else small = solve_small<D>(W, wb, zb, z0b, ent, ss);
        }
#else
        small = solve_small<D>(W, wb, zb, z0b, ent, ss);
#endif
        double* Gp = Gslow;
        if (CA_RARE(!small)) {
          // the first GSLOTS lanes of the warp needing it use shared memory
          const unsigned am = __activemask();
          const int slot = __popc(am & ((1u << tid) - 1u));
          if (slot < GSLOTS) Gp = gpool + slot * SM::GN;
          const ColSol<D> cg = Lemke<D, NMAX, D + 4>::solve_column(W, Gp, 1, wb, zb, z0b, ent, Gp);
#pragma unroll
          for (int c = 0; c <= D; ++c) ss.uh[c] = cg.uh[c];
          ss.sl = cg.sl;
          ss.sk = cg.sk;
          ss.s0 = cg.s0;
        }
        auto xcol = [&](int s) -> double {
          if (small) return (s == 0) ? ss.x[0] : ((s == 1) ? ss.x[1] : ss.x[2]);
          return Gp[s * (D + 5) + D + 4];
        };
        const uint32_t basic = wb | zb;
        // pass 1 (one sweep over the rows, segment by segment so every row fetch is a  // @region pass1
        // fixed-stride load): apply the previous pivot's value update (deferred from
        // L3), store the entering-column coefficient cbar_i of row i, and run the
        // L5.2 ratio test on the fly -- provisional minimum over cbar > pivot_tol (a
        // superset of the eligible rows cbar > pivot_tol max(1, cmax)) plus a
        // superset `cand` of the final tie set (rows within the tie tolerance of
        // the running minimum, which only shrinks).
        double cmax = 0.0, bn = kInf, bd = 1.0, tn = kInf;
        uint32_t cand = 0;
        auto ratio = [&](bool el, double c, double v, uint32_t bit) {  // branch-free
          const double nu = (v > 0.0) ? v : 0.0;
          const double nbd = nu * bd;
          const bool lt = el && (nbd < bn * c);
          // a new minimum is its own candidate; otherwise compare with the band of the
          // running minimum: nu/c <= theta + tau' max(1, theta), tau' = tau + 1e-12 (superset)
          const bool cnd = el && nbd <= tn * c;
          const double tnn = __fma_rn(tauS, (c > nu) ? c : nu, nu);  // (theta + tau' max(1,theta)) c
#if CA_EXP_RESET
          // a new minimum whose band lies below the old minimum drops the old candidates
          // (they are all >= the old minimum): cand stays (nearly) exact, so the tie
          // filter below only runs on real near-ties
          const bool reset = lt && (tnn * bd < bn * c);
#else
          const bool reset = false;
#endif
          cand = reset ? bit : ((lt || cnd) ? (cand | bit) : cand);
          bn = lt ? nu : bn;
          bd = lt ? c : bd;
          tn = lt ? tnn : tn;
        };
        auto rowcv = [&](int i, double c, double vo, double co) {
          const uint32_t bit = 1u << i;
          const double vu = __fma_rn(-co, ve2p, vo);
          const double v = (pend & bit) ? vu : vo;
          VAL(i) = v;
          CBV(i) = c;
          const bool wbas = (wb & bit) != 0u;
          const double ac = fabs(c);
          cmax = (wbas && ac > cmax) ? ac : cmax;
          ratio(wbas && c > ptol, c, v, bit);
        };
        auto rowc = [&](int i, double c) { rowcv(i, c, VAL(i), CBV(i)); };
#if CA_EXP_P1MERGE
        // every row in one loop (one inlined copy of the row step: a smaller hot loop),
        // rows fetched through the branch-free table select; bitwise the segmented form
        // (the extra terms are exact zeros: f = 0 or k = 0)
#pragma unroll 1
        for (int i = 0; i < n; ++i) {
          double f[D + 1], k;
          W.row(i, f, k);
          double c = ss.s0;
#pragma unroll
          for (int cc = 0; cc <= D; ++cc) c = __fma_rn(f[cc], ss.uh[cc], c);
          c = __fma_rn(k, ss.sl, c);
          rowc(i, (i == n - 1) ? c - ss.sk : c);
        }
#else
        // lambda rows (0, at_u, kt_u): CTA-shared table of part ip
#pragma unroll 1
        for (int i = 0; i < nr1; ++i) {
          const double* r = lt + i * (D + 2);
          double c = ss.s0;
#pragma unroll
          for (int cc = 0; cc <= D; ++cc) c = __fma_rn(r[cc], ss.uh[cc], c);
          rowc(i, __fma_rn(r[D + 1], ss.sl, c));
        }
#if CA_EXP_MU_PIPE
        // mu rows (d_l - c_l.rho, R^T c_l): kt = 0; software-pipelined -- the next row's
        // data and its value / coefficient are loaded while this row is processed
        {
          double mr[D + 1], vo = VAL(nr1), co = CBV(nr1);
#pragma unroll
          for (int cc = 0; cc <= D; ++cc) mr[cc] = mu[cc * CTA];
#pragma unroll 1
          for (int l = 0; l < no; ++l) {
            const int ln = (l + 1 < no) ? l + 1 : l;
            const double* mn = mu + ln * L1 * CTA;
            double nx[D + 1];
#pragma unroll
            for (int cc = 0; cc <= D; ++cc) nx[cc] = mn[cc * CTA];
            const double vn = VAL(nr1 + ln), cn = CBV(nr1 + ln);
            double c = ss.s0;
#pragma unroll
            for (int cc = 0; cc <= D; ++cc) c = __fma_rn(mr[cc], ss.uh[cc], c);
            rowcv(nr1 + l, c, vo, co);
#pragma unroll
            for (int cc = 0; cc <= D; ++cc) mr[cc] = nx[cc];
            vo = vn;
            co = cn;
          }
        }
#else
        // mu rows (d_l - c_l.rho, R^T c_l): kt = 0
#if CA_EXP_MU_UNROLL == 2
#pragma unroll 2
#else
#pragma unroll 1
#endif
        for (int l = 0; l < no; ++l) {
          const double* m = mu + l * L1 * CTA;
          double c = ss.s0;
#pragma unroll
          for (int cc = 0; cc <= D; ++cc) c = __fma_rn(m[cc * CTA], ss.uh[cc], c);
          rowc(nr1 + l, c);
        }
#endif
        rowc(n - 2, __fma_rn(1.0, ss.uh[0], ss.s0));  // gamma row (1, 0)
        rowc(n - 1, ss.s0 - ss.sk);                    // phi row (0, 0)
#endif
        pend = 0;
        // basic z rows: cbar is the structural solution itself
        {
          int s = 0;
#pragma unroll 1
          for (uint32_t bb = zb; bb; bb &= bb - 1, ++s) {
            const int i = __ffs(bb) - 1;
            const double c = xcol(s);
            CBV(i) = c;
            const double ac = fabs(c);
            cmax = (ac > cmax) ? ac : cmax;
            ratio(c > ptol, c, VAL(i), 1u << i);
          }
        }
        double cb0 = 0.0;
        if (z0b) {
          cb0 = xcol(__popc(zb));
          cmax = fmax(cmax, fabs(cb0));
          ratio(cb0 > ptol, cb0, val0, 0u);  // z0 has no row bit (a new minimum at z0 resets the rows)
        }
        const double thr = ptol * fmax(1.0, cmax);
        // rare: the provisional minimiser is not eligible (pivot_tol < cbar <= thr):
        // the dense-tableau solve takes the exact L5 decision
        if (CA_RARE(bn < kInf && !(bd > thr))) { status = ST_TIE; break; }
        if (CA_RARE(!(bn < kInf))) { status = ST_RAY; break; }
        const double thmin = bn / bd;
        const double tt = thmin + tau * fmax(1.0, thmin);
        // tie set (L5.2): filter the candidates against the final minimum.  A lone
        // candidate is the minimising row itself (eligible: checked above), so the
        // filter only runs on real near-ties.
        uint32_t tiem = cand;
        if (CA_RARE(__popc(cand) > 1)) {
          tiem = 0;
#pragma unroll 1
          for (uint32_t bb = cand; bb; bb &= bb - 1) {
            const int i = __ffs(bb) - 1;
            const double c = CBV(i);
            if (c > thr && fmax(VAL(i), 0.0) <= tt * c) tiem |= 1u << i;
          }
        }
        int lm;
        double cr, vr;
        if (z0b && cb0 > thr && fmax(val0, 0.0) <= tt * cb0) {
          lm = -1;  // L5.3: z0 leaves whenever it is tied
          cr = cb0;
          vr = val0;
        } else if (tiem == 0) {
          status = ST_RAY;
          break;
        } else {
          // a multi-way tie (L5.4-5, lexicographic rule) is left to the dense-tableau
          // solve, which applies the oracle's rules verbatim; ties are rare (none in
          // 3000 sampled C5 pairs) and keeping the rule out of the pivot loop keeps
          // its register footprint small
          if (CA_RARE(__popc(tiem) > 1)) { status = ST_TIE; break; }
          lm = __ffs(tiem) - 1;
          cr = CBV(lm);
          vr = VAL(lm);
        }
        if (TRACE && p == P.dbg_p && pivots < 64) {  // diagnostics (ca_debug_trace) build only
          const TraceRow tr{{(double)ent.kind, (double)ent.j, (double)(n - __popc(wb)), (double)lm, thmin,
                             (double)__popc(tiem), cr, vr, (double)wb, (double)zb, cmax, small ? 0.0 : 1.0, val0, cb0}};
          trace_pivot(P.dbg + pivots * 48, tr, sval, scb, n);
        }
        // L3: pivot (values only: the structure is re-derived from the basis); the  // @region pivot_update
        // update of the other basic values is deferred to the next pass 1 (`pend`);
        // the entering variable takes the leaving one's tableau row
        const bool leave_w = (lm >= 0) && ((wb >> lm) & 1u);
        const double ve2 = vr * (1.0 / cr);
        const int je = ent.j;
        pend = basic & ~(lm >= 0 ? (1u << lm) : 0u);
        ve2p = ve2;
        if (z0b && lm >= 0) val0 = __fma_rn(-cb0, ve2, val0);
        VAL(je) = ve2;
        rowb.set(je, rowb.get(lm >= 0 ? lm : NMAX));
        if (ent.kind == 0) wb |= 1u << je;
        else zb |= 1u << je;
        ++pivots;
        if (lm < 0) { z0b = false; break; }  // L6: z0 left
        // leaving member lm (w or z of pair lm); next entering is its complement (L4)
        if (leave_w) {
          wb &= ~(1u << lm);
          ent = Var{1, lm};
        } else {
          zb &= ~(1u << lm);
          ent = Var{0, lm};
        }
      }
#pragma unroll 1
      for (uint32_t bb = pend; bb; bb &= bb - 1) {  // the last pivot's deferred update
        const int i = __ffs(bb) - 1;
        VAL(i) = __fma_rn(-CBV(i), ve2p, VAL(i));
      }
    }

    // ------------------------------------------------------- verification  // @region verify
    // The revised path never forms the tableau, so check its answer against the
    // LCP itself: w = M z + q (O(n d) with the low-rank M), w_i = value of basic
    // w_i or 0, w >= 0, z >= 0.  Failure or RAY / ITER_LIMIT -> dense fallback.
    fallback = (status != ST_OK) || (TRACE && (P.dense || nwt_fail));
    if (!fallback && qmin < 0.0 && !(TRACE && P.prox_newton)) {
      double uz[D + 1], zl = 0.0, skz = 0.0, zsc = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) uz[c] = 0.0;
#pragma unroll 1
      for (uint32_t bb = zb; bb; bb &= bb - 1) {
        const int jz = __ffs(bb) - 1;
        const double z = VAL(jz);
        zsc = fmax(zsc, fabs(z));
        if (z < -1e-9) fallback = true;
        double f[D + 1], k;
        W.row(jz, f, k);
#pragma unroll
        for (int c = 0; c <= D; ++c) uz[c] = __fma_rn(z, f[c], uz[c]);
        skz = __fma_rn(z, k, skz);
        if (jz == n - 1) zl = z;
      }
#pragma unroll 1
      for (int i = 0; i < n && !fallback; ++i) {
        double f[D + 1], k;
        W.row(i, f, k);
        double q = 1.0 / be, w = 0.0, mag = 1.0 + zsc;
        if (i < n - 1) {
          q = 0.0;
#pragma unroll
          for (int c = 0; c <= D; ++c) {
            q = __fma_rn(f[c], bt_[c], q);
            w = __fma_rn(f[c], uz[c], w);
          }
        }
        w = __fma_rn(k, zl, w);
        if (i == n - 1) w -= skz;
        w += q;
        mag += fabs(q);
        const double expect = ((wb >> i) & 1u) ? VAL(i) : 0.0;
        if (fabs(w - expect) > 1e-7 * mag || w < -1e-7 * mag) fallback = true;
      }
    }
  }
  // dense-tableau re-solves (rules L1-L7 verbatim, lexicographic ties included), one
  // pair at a time by the whole warp: lane i owns tableau row i
  for (uint32_t need = __ballot_sync(0xffffffffu, act && fallback); need; need &= need - 1) {  // @region fallback
    const int L = __ffs(need) - 1;
    const int nrL = __shfl_sync(0xffffffffu, nr, L), noL = __shfl_sync(0xffffffffu, no, L);
    const int ipL = __shfl_sync(0xffffffffu, ip, L);
    double btL[D + 1];
#pragma unroll
    for (int c = 0; c <= D; ++c) btL[c] = __shfl_sync(0xffffffffu, bt_[c], L);
    const double beL = __shfl_sync(0xffffffffu, be, L);
    const PairRows<D> WL{lamtab + ipL * LT, cst, wcol + L, CTA, nrL, noL, nrL + noL + 1, nrL + noL};
    uint32_t zbL;
    int pivL;
    Prox XL{0.0, nullptr, 0, 0, 0};
    if (TRACE && P.prox_eps > 0.0)  // reading #2 (the latency-mode kernel only)
      XL = Prox{P.prox_eps, P.y, PP, __shfl_sync(0xffffffffu, p, L), P.part_e[ipL]};
    const int stL = lemke_warp<D, NMAX, TRACE>(WL, btL, beL, P.lp, XL, sval - tid + L, tid, &zbL, &pivL);
    if (tid == L) {
      status = stL;
      zb = zbL;
      pivots = pivL;  // the returned solution's own path
      z0b = false;
    }
  }
  if (act) {
    // ------------------------------------------------------------ recovery  // @region recover
    // z_j = value of basic z_j (LCP index j);  y_U = z[0..n-2] in original order
    // without e;  y_e = (1 - sum_{k != e} b_k y_k) / b_e
    const int st0 = status;
    double acc = 0.0;
#pragma unroll 1
    for (int k = 0; k < nr; ++k) {
      if (k == e) continue;
      const int u = k - (k > e);
      const double yv = ((zb >> u) & 1u) ? VAL(u) : 0.0;
      acc = __fma_rn(prow[4 * k + 3], yv, acc);
    }
    const double ye = (1.0 - acc) / be;
    int st = st0;
    if (st == ST_OK && ye < -1e-6) st = ST_NEGYE;
    const bool solved = (st == ST_OK);
    // y used by the aggregates: y^{k+1}, or y^k for a failed pair;
    // y^k re-staged in the cbar scratch (free again) with batched loads; the Newton
    // path (NEXT f4) only reads it, so it is still there
    if (!(TRACE && P.prox_newton && !fallback)) {
#pragma unroll 4
      for (int k = 0; k < n; ++k) CBV(k) = YK(k);
    }
    double rd = 0.0;
    double eT = 1.0 + zeta, eR[D], vb[D];  // vb = R^T v = sum_l mu_l R^T c_l (body frame)
#pragma unroll
    for (int a = 0; a < D; ++a) { eR[a] = xi[a]; vb[a] = 0.0; }
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      double yv;
      if (solved) {
        const int u = k - (k > e);
        yv = (k == e) ? ye : (((zb >> u) & 1u) ? VAL(u) : 0.0);
        if (k < nr + no) {
          const double df = yv - CBV(k);
          rd = __fma_rn(df, df, rd);
        }
        P.y[(long long)k * PP + p] = yv;
      } else {
        yv = CBV(k);
      }
      // Gauss-Newton aggregates at pose(s^k): u* = K^T y + bvec = (eT, eR); v = C_j^T mu  // @region aggregates
      if (k < nr) {
#pragma unroll
        for (int a = 0; a < D; ++a) eR[a] = __fma_rn(yv, prow[4 * k + a], eR[a]);
      } else if (k < nr + no) {
        const double* m = mu + (k - nr) * L1 * CTA;
        eT = __fma_rn(yv, m[0], eT);
#pragma unroll
        for (int a = 0; a < D; ++a) eR[a] = __fma_rn(yv, m[(1 + a) * CTA], eR[a]);
#pragma unroll
        for (int a = 0; a < D; ++a) vb[a] = __fma_rn(yv, m[(1 + a) * CTA], vb[a]);
      } else {
        eT += yv;
      }
    }
    double v[D];  // v = C_j^T mu = R vb (world frame)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) acc = __fma_rn(po[c * D + a], vb[a], acc);
      v[c] = acc;
    }
    if (solved) rec[NAGG + S_RDUAL] = rd;
    // failure kinds: RAY, ITER_LIMIT, y_e < -1e-6
    ist[0] = pivots;
    ist[1] = solved ? 0 : 1;
    ist[2] = (st == ST_RAY) ? 1 : 0;
    ist[3] = (st == ST_ITER) ? 1 : 0;
    ist[4] = (st == ST_NEGYE) ? 1 : 0;
    P.pst[p] = (uint32_t)min(pivots, 65535) | ((uint32_t)st << 16) | (fallback ? (1u << 20) : 0u);
    if (P.zmask) P.zmask[p] = zb | (z0b ? 0x80000000u : 0u);
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int c = a; c < D; ++c) rec[sym_idx(a, c, L1)] = v[a] * v[c];
      rec[L1 * (L1 + 1) / 2 + a] = -eT * v[a];
    }
    if (P.pose_model != 0) {
      // g = J^T R^T v = J^T vb with J the rotation generator (SE2 / yaw): (vb_1, -vb_0, 0)
      const double g0 = vb[1], g1 = -vb[0];
      rec[sym_idx(D, D, L1)] = g0 * g0 + g1 * g1;
      rec[L1 * (L1 + 1) / 2 + D] = g0 * eR[0] + g1 * eR[1];
      if (TRACE && P.part_ctr) {  // scaling centre: dT/dtheta = vb_0 o_1 - vb_1 o_0 (reading #22)
        const double* oc = P.part_ctr + 3 * ip;
        const double tau = vb[0] * oc[1] - vb[1] * oc[0];
#pragma unroll
        for (int a = 0; a < D; ++a) rec[sym_idx(a, D, L1)] = -v[a] * tau;
        rec[sym_idx(D, D, L1)] += tau * tau;
        rec[L1 * (L1 + 1) / 2 + D] += tau * eT;
      }
    }
  }
#undef VAL
#undef CBV
#undef YK
  {  // @region cta_reduce
    // deterministic grouped reduction: one record per timestep of the group, lanes
    // summed in lane order, staged through the (now free) per-thread columns
    double* out = P.agg + (long long)item * P.TG * RECD;
    group_reduce<NDBL>(wcol, tid, tl, P.TG, out, RECD, rec, 0, -1);
    group_reduce_int(tid, tl, P.TG, out + NAGG, RECD, ist);
  }
  }  // work item
}

// host-side launcher; explicitly instantiated in ca_sweep_*.cu (parallel build).
// The extended variant (TRACE) is a separate kernel, launched only while a
// ca_debug_trace request is armed, the problem has per-part scaling centres or runs
// in the small-problem latency mode, so the production kernel carries none of the
// diagnostic code, the centre terms (2 % of the C5 sweep when compiled in) or the
// latency-mode switch.
template <int D, int NM, bool F, bool T>
cudaError_t sweep_launch_v(const Dev& P, unsigned grid, cudaStream_t stream) {
#ifndef CA_EXP_SMEM_PAD
#define CA_EXP_SMEM_PAD 0
#endif
  const size_t sm = SweepSmem<D, NM>::bytes(P.np, P.nrmax, P.nomax) + CA_EXP_SMEM_PAD;
  // the dynamic-smem attribute and the residency are per device (and per instantiation):
  // cached per device ordinal under a lock (handles may live on several devices / threads)
  static std::mutex mu;
  static size_t configured[CA_MAX_DEVICES] = {};
  static int resident[CA_MAX_DEVICES] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= CA_MAX_DEVICES) return cudaErrorInvalidDevice;
  int res_dev = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (configured[dev] < sm) {
      resident[dev] = 0;
      e = cudaFuncSetAttribute(k_sweep<D, NM, F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      // all of the unified L1/shared array as shared memory: residency is smem-bound
      e = cudaFuncSetAttribute(k_sweep<D, NM, F, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      configured[dev] = sm;
    }
#if CA_SWEEP_PERSIST
    if (!resident[dev]) {
      int nsm = 0, per = 0;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sweep<D, NM, F, T>, CTA * WPC, sm);
      resident[dev] = nsm * (per > 0 ? per : 1) * WPC;  // in warps
    }
#endif
    res_dev = resident[dev];
  }
#if CA_SWEEP_PERSIST
  unsigned warps = (unsigned)res_dev < grid ? (unsigned)res_dev : grid;
  // diagnostics: CA_SWEEP_WARPS caps the persistent grid (a different item-to-warp
  // interleaving; results must not change -- tests/test_gpu_checked.py)
  static const int cap = std::getenv("CA_SWEEP_WARPS") ? std::atoi(std::getenv("CA_SWEEP_WARPS")) : 0;
  if (cap > 0 && (unsigned)cap < warps) warps = (unsigned)cap;
#else
  unsigned warps = grid;
#endif
  k_sweep<D, NM, F, T><<<(warps + WPC - 1) / WPC, CTA * WPC, sm, stream>>>(P);
  return cudaGetLastError();
}

template <int D, int NM, bool F>
cudaError_t sweep_launch(const Dev& P, unsigned grid, cudaStream_t stream) {
  return (P.dbg_p >= 0 || P.part_ctr || P.dense || P.prox_newton) ? sweep_launch_v<D, NM, F, true>(P, grid, stream)
                                                 : sweep_launch_v<D, NM, F, false>(P, grid, stream);
}

#define CA_SWEEP_NMAX_LIST(X, D, F) X(D, 9, F) X(D, 11, F) X(D, 13, F) X(D, 15, F) X(D, 20, F) X(D, 32, F)

}  // namespace ca
