// ca_lemke.cuh -- one-thread-per-pair revised Lemke for the LCP of Eq. 24
// built from the equality-eliminated pair QP.
//
// Why revised, not a dense tableau: the LCP matrix
//     M = [[Kt Kt^T, kt], [-kt^T, 0]]
// is  M = F F^T + k e_l^T - e_l k^T  with F = [Kt; 0] (n x (d+1)), k = [kt; 0],
// l = n-1: rank <= d+3.  A basis B of Lemke's tableau B^{-1}[I | -M | -1 | q]
// therefore holds at most d+4 structural columns (basic z_j / z0); with R the
// equations whose w is nonbasic (|R| = m), B^{-1} a reduces to the m x m system
//     G x = a_R,   G[p][s] = a(zb_s)_{R_p},
// and every basic w_i's coefficient is  a_i + F_i.u + k_i sl - [i=l] sk + s0
// (u, sl, sk, s0 linear in x).  A pivot costs O(n (d+2) + m^3) FP64 (m <= 3 in
// 99.7 % of bases on C5) instead of the O(n^2) dense tableau update -- in ONE
// thread, so a warp solves 32 pairs with no cross-lane traffic.
//
// Register discipline: per-variable state is indexed by the complementary PAIR
// index i (exactly one of w_i, z_i is basic, except the missing pair) and only
// ever with compile-time indices (unrolled loops); sets are bitmasks.  Anything
// indexed at run time (reduced rows, the m x m system, tableau-row labels) lives
// in per-thread shared memory, layout [item][thread] (conflict-free).
//
// Selection rules = DESIGN.md reading #4 (L1-L7), the oracle's textbook
// full-tableau rules, except that ratios are compared by cross multiplication
// (one division per pivot): decisions coincide with the oracle except at
// near-ties closer than rounding (the parity tests count and validate those).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef CA_EXP_INLINE_GEN
#define CA_EXP_INLINE_GEN 1  // generic m > 3 solve inlined (no call-site register saves)
#endif

namespace ca {

enum { ST_OK = 0, ST_RAY = 1, ST_ITER = 2, ST_NEGYE = 3, ST_TIE = 4 /* internal: re-solve densely */ };

// Reduced rows (Kt_i, kt_i) of one pair, i = 0..n-1 in LCP order:
//   i <  nr-1      lambda rows: (0, at_i), kt_i = b_k / b_e  [CTA-shared, per part, D+2 doubles]
//   i <  n-2       mu rows:     (d_l - c_l.rho, R^T c_l), 0  [per-thread table, D+1 doubles]
//   i == n-2       gamma row:   (1, 0), 0                    [CTA-shared constant row]
//   i == n-1       phi row:     0                            [CTA-shared constant row]
// row() is branch-free: a pointer/stride select between the tables.
template <int D>
struct PairRows {  // @region row_fetch
  const double* lam;  // [(nr-1)][D+2] = (0, at_1..at_D, kt)  (CTA smem)
  const double* cst;  // [2][D+2]: gamma row, phi row            (CTA smem)
  const double* mu;   // [no][D+1], stride `ms` between doubles (thread smem)
  int ms;
  int nr, no, n, l;
  __device__ __forceinline__ void row(int i, double f[D + 1], double& k) const {
    const bool isl = i < nr - 1;
    const bool sh = isl || i >= n - 2;
    const double* sb = isl ? lam + i * (D + 2) : cst + (i - (n - 2)) * (D + 2);
    const double* base = sh ? sb : mu + (i - (nr - 1)) * (D + 1) * ms;
    const int st = sh ? 1 : ms;
#pragma unroll
    for (int c = 0; c <= D; ++c) f[c] = base[c * st];
    const double ks = sb[D + 1];
    k = sh ? ks : 0.0;
  }
};

// M_ij of Eq. 24 from two reduced rows (row/col l = n-1 is the phi row)
template <int D>
__device__ __forceinline__ double m_entry(const double fi[D + 1], double ki, int i, const double fj[D + 1],  // @region m_entry
                                          double kj, int j, int l) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c <= D; ++c) acc = __fma_rn(fi[c], fj[c], acc);
  if (j == l) acc = ki;
  if (i == l) acc = -kj;
  if (i == l && j == l) acc = 0.0;
  return acc;
}

// Gauss-Jordan with partial pivoting (rows physically swapped) on an m x (m+1)
// system stored with element stride `es`: A[(p*(mm+1)+c)*es], mm = row capacity.
// Solution left in column m: x_s = A[s][m].
__device__ __forceinline__ void gj_solve(double* A, int es, int mm, int m) {  // @region gj_solve
#define GA(p_, c_) A[((p_) * (mm + 1) + (c_)) * es]
  for (int c = 0; c < m; ++c) {
    int pb = c;
    double best = fabs(GA(c, c));
    for (int p = c + 1; p < m; ++p) {
      const double a = fabs(GA(p, c));
      if (a > best) { best = a; pb = p; }
    }
    if (pb != c) {
      for (int cc = c; cc < m; ++cc) { const double t = GA(c, cc); GA(c, cc) = GA(pb, cc); GA(pb, cc) = t; }
      const double t = GA(c, mm); GA(c, mm) = GA(pb, mm); GA(pb, mm) = t;
    }
    const double inv = 1.0 / GA(c, c);
    for (int cc = c + 1; cc < m; ++cc) GA(c, cc) = GA(c, cc) * inv;
    GA(c, mm) = GA(c, mm) * inv;
    for (int p = 0; p < m; ++p) {
      if (p == c) continue;
      const double f = GA(p, c);
      if (f == 0.0) continue;
      for (int cc = c + 1; cc < m; ++cc) GA(p, cc) = __fma_rn(-f, GA(c, cc), GA(p, cc));
      GA(p, mm) = __fma_rn(-f, GA(c, mm), GA(p, mm));
    }
  }
#undef GA
}

// Entering-variable encoding: kind 0 = w_j, 1 = z_j, 2 = z0
struct Var {
  int kind, j;
};

template <int D>
struct ColSol {
  double uh[D + 1];
  double sl, sk, s0;
  int slow;
};

template <int D, int NMAX, int MFAST>
struct Lemke {
  static constexpr int MMAX = D + 4;  // rank bound of the structural block
  // Build and solve G x = a(e)_R; returns the low-rank coefficients
  //   coef(w_i) = F_i.uh + kt_i sl - [i=l] sk + s0
  // and writes x_s for the structural columns into xcol (smem, stride es).
  // Columns: basic z_j in increasing j, then z0 if basic.  Rows: R increasing.
#if CA_EXP_INLINE_GEN
  __device__ __forceinline__ static ColSol<D> solve_column(
#else
  __device__ __noinline__ static ColSol<D> solve_column(
#endif
      const PairRows<D> W, double* Gs, int gs, uint32_t wb,  // @region solve_column
                                                       uint32_t zb, bool z0b, Var e, double* Gslow) {
    ColSol<D> out;
    double* uh = out.uh;
    double& sl = out.sl;
    double& sk = out.sk;
    double& s0 = out.s0;
    const uint32_t nmask = (W.n >= 32) ? 0xffffffffu : ((1u << W.n) - 1u);
    const uint32_t Rm = ~wb & nmask;
    const int m = __popc(Rm);
    double* A = Gs;
    int es = gs, mm = MFAST;
    if (m > MFAST) { A = Gslow; es = 1; mm = MMAX; }
#define GA(p_, c_) A[((p_) * (mm + 1) + (c_)) * es]
    double fe[D + 1], ke = 0.0;
    if (e.kind == 1) W.row(e.j, fe, ke);
    int p = 0;
    for (uint32_t rb = Rm; rb; rb &= rb - 1, ++p) {
      const int i = __ffs(rb) - 1;
      double fi[D + 1], ki;
      W.row(i, fi, ki);
      int s = 0;
      for (uint32_t cb = zb; cb; cb &= cb - 1, ++s) {
        const int j = __ffs(cb) - 1;
        double fj[D + 1], kj;
        W.row(j, fj, kj);
        GA(p, s) = -m_entry<D>(fi, ki, i, fj, kj, j, W.l);
      }
      if (z0b) GA(p, s) = -1.0;
      double a;
      if (e.kind == 0) {
        a = (i == e.j) ? 1.0 : 0.0;
      } else if (e.kind == 2) {
        a = -1.0;
      } else {
        a = -m_entry<D>(fi, ki, i, fe, ke, e.j, W.l);
      }
      GA(p, mm) = a;
    }
    gj_solve(A, es, mm, m);
    // low-rank coefficients
#pragma unroll
    for (int c = 0; c <= D; ++c) uh[c] = 0.0;
    sl = sk = s0 = 0.0;
    int s = 0;
    for (uint32_t cb = zb; cb; cb &= cb - 1, ++s) {
      const int j = __ffs(cb) - 1;
      double fj[D + 1], kj;
      W.row(j, fj, kj);
      const double x = GA(s, mm);
#pragma unroll
      for (int c = 0; c <= D; ++c) uh[c] = __fma_rn(x, fj[c], uh[c]);
      sk = __fma_rn(x, kj, sk);
      if (j == W.l) sl += x;
    }
    if (z0b) s0 += GA(s, mm);
    if (e.kind == 2) {
      s0 -= 1.0;
    } else if (e.kind == 1) {
#pragma unroll
      for (int c = 0; c <= D; ++c) uh[c] -= fe[c];
      sk -= ke;
      if (e.j == W.l) sl -= 1.0;
    }
#undef GA
    out.slow = (m > MFAST) ? 1 : 0;
    return out;
  }
};

// Fast path of solve_column for m <= 3 (99.7 % of bases on C5): the m x m
// structural system lives in registers (padded to 3 x 3 with identity rows).
template <int D>
struct SmallSol {
  double x[3];  // columns: basic z_j in increasing j, then z0
  double uh[D + 1];
  double sl, sk, s0;
};

template <int D>
__device__ __forceinline__ bool solve_small(const PairRows<D>& W, uint32_t wb, uint32_t zb, bool z0b, Var e,
                                            SmallSol<D>& out) {  // @region small_build
  const uint32_t nmask = (W.n >= 32) ? 0xffffffffu : ((1u << W.n) - 1u);
  const uint32_t Rm = ~wb & nmask;
  const int m = __popc(Rm);
  if (m > 3) return false;
  const int mz = __popc(zb);
  const int l = W.l;
  // Branch-free: every row fetch uses a valid index (clamped), the results of the
  // padding slots are discarded by selects.
  double fc[3][D + 1], kc[3];
  int jc[3];
  uint32_t zbits = zb;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int j = __ffs(zbits) - 1;  // -1 when exhausted
    zbits &= zbits - 1;
    W.row(j < 0 ? 0 : j, fc[s], kc[s]);
    jc[s] = j;
  }
  double fe[D + 1], ke;
  W.row(e.kind == 1 ? e.j : 0, fe, ke);
  double G[3][4];
  uint32_t rbits = Rm;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int i = __ffs(rbits) - 1;
    rbits &= rbits - 1;
    double fi[D + 1], ki;
    W.row(i < 0 ? 0 : i, fi, ki);
    const bool real = p < m;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double me = -m_entry<D>(fi, ki, i, fc[s], kc[s], jc[s], l);
      const double v = (s < mz) ? me : ((s == mz && z0b) ? -1.0 : 0.0);
      G[p][s] = real ? v : ((p == s) ? 1.0 : 0.0);
    }
    const double me = -m_entry<D>(fi, ki, i, fe, ke, e.j, l);
    const double a = (e.kind == 0) ? ((i == e.j) ? 1.0 : 0.0) : ((e.kind == 2) ? -1.0 : me);
    G[p][3] = real ? a : 0.0;
  }
  // Gauss-Jordan with partial pivoting, compile-time indices  // @region small_gj
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int r = c + 1; r < 3; ++r) {
      const bool sw = fabs(G[r][c]) > fabs(G[c][c]);
#pragma unroll
      for (int cc = c; cc < 4; ++cc) {
        const double t = G[c][cc];
        G[c][cc] = sw ? G[r][cc] : t;
        G[r][cc] = sw ? t : G[r][cc];
      }
    }
    const double inv = 1.0 / G[c][c];
#pragma unroll
    for (int cc = c + 1; cc < 4; ++cc) G[c][cc] = G[c][cc] * inv;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      if (r == c) continue;
      const double f = G[r][c];
#pragma unroll
      for (int cc = c + 1; cc < 4; ++cc) G[r][cc] = __fma_rn(-f, G[c][cc], G[r][cc]);
    }
  }
  double uh[D + 1], sl = 0.0, sk = 0.0, s0 = 0.0;
#pragma unroll
  for (int c = 0; c <= D; ++c) uh[c] = 0.0;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const double x = G[s][3];
    out.x[s] = x;
    const bool col = s < mz;
    const double xz = col ? x : 0.0;  // contributes exact zeros otherwise
#pragma unroll
    for (int c = 0; c <= D; ++c) uh[c] = col ? __fma_rn(x, fc[s][c], uh[c]) : uh[c];
    sk = col ? __fma_rn(x, kc[s], sk) : sk;
    sl = (col && jc[s] == l) ? sl + xz : sl;
    s0 = (s == mz && z0b) ? s0 + x : s0;
  }
  if (e.kind == 2) s0 -= 1.0;
  const bool ez = e.kind == 1;
#pragma unroll
  for (int c = 0; c <= D; ++c) out.uh[c] = ez ? uh[c] - fe[c] : uh[c];
  out.sk = ez ? sk - ke : sk;
  out.sl = (ez && e.j == l) ? sl - 1.0 : sl;
  out.s0 = s0;
  return true;
}

// Exact replicas of solve_small for m = 1 and m = 2 structural columns (the first
// pivots of almost every pair: z0 alone, then z0 and one z_j): the identity-padded 3 x 3
// Gauss-Jordan of solve_small reduces on the real rows to the operations below (padding
// rows and columns only ever contribute exact zeros and unit pivots), so the results
// are bitwise those of solve_small, for a fraction of the work.
template <int D>
__device__ __forceinline__ void solve_m1(const PairRows<D>& W, uint32_t Rm, uint32_t zb, bool z0b, Var e,
                                         SmallSol<D>& out) {
  const int l = W.l, mz = __popc(zb);
  const int i = __ffs(Rm) - 1;
  double fi[D + 1], ki;
  W.row(i, fi, ki);
  double fe[D + 1], ke;
  W.row(e.kind == 1 ? e.j : 0, fe, ke);
  const int j = __ffs(zb) - 1;  // the column is z_j (mz = 1) or z0
  double fc[D + 1], kc;
  W.row(j < 0 ? 0 : j, fc, kc);
  const double g = (mz == 1) ? -m_entry<D>(fi, ki, i, fc, kc, j, l) : -1.0;
  const double me = -m_entry<D>(fi, ki, i, fe, ke, e.j, l);
  const double a = (e.kind == 0) ? ((i == e.j) ? 1.0 : 0.0) : ((e.kind == 2) ? -1.0 : me);
  const double x = a * (1.0 / g);
  out.x[0] = x;
  out.x[1] = out.x[2] = 0.0;
  const bool col = mz == 1;
  double uh[D + 1];
#pragma unroll
  for (int c = 0; c <= D; ++c) uh[c] = col ? __fma_rn(x, fc[c], 0.0) : 0.0;
  const double sk = col ? __fma_rn(x, kc, 0.0) : 0.0;
  const double sl = (col && j == l) ? 0.0 + x : 0.0;
  double s0 = (!col && z0b) ? 0.0 + x : 0.0;
  if (e.kind == 2) s0 -= 1.0;
  const bool ez = e.kind == 1;
#pragma unroll
  for (int c = 0; c <= D; ++c) out.uh[c] = ez ? uh[c] - fe[c] : uh[c];
  out.sk = ez ? sk - ke : sk;
  out.sl = (ez && e.j == l) ? sl - 1.0 : sl;
  out.s0 = s0;
}

template <int D>
__device__ __forceinline__ void solve_m2(const PairRows<D>& W, uint32_t Rm, uint32_t zb, bool z0b, Var e,
                                         SmallSol<D>& out) {
  const int l = W.l, mz = __popc(zb);
  const int i0 = __ffs(Rm) - 1;
  const int i1 = __ffs(Rm & (Rm - 1)) - 1;
  const int j0 = __ffs(zb) - 1;              // column 0: z_j0 (mz >= 1) or z0
  const int j1 = __ffs(zb & (zb - 1)) - 1;   // column 1: z_j1 (mz = 2) or z0
  double f0[D + 1], k0, f1[D + 1], k1, fe[D + 1], ke, fa[D + 1], ka, fb[D + 1], kb;
  W.row(i0, f0, k0);
  W.row(i1, f1, k1);
  W.row(e.kind == 1 ? e.j : 0, fe, ke);
  W.row(j0 < 0 ? 0 : j0, fa, ka);
  W.row(j1 < 0 ? 0 : j1, fb, kb);
  // G = [[g00 g01 | a0], [g10 g11 | a1]] as solve_small builds it
  auto gcol = [&](const double* fi, double ki, int i, int s) -> double {
    const double me = (s == 0) ? -m_entry<D>(fi, ki, i, fa, ka, j0, l) : -m_entry<D>(fi, ki, i, fb, kb, j1, l);
    return (s < mz) ? me : ((s == mz && z0b) ? -1.0 : 0.0);
  };
  auto rhs = [&](const double* fi, double ki, int i) -> double {
    const double me = -m_entry<D>(fi, ki, i, fe, ke, e.j, l);
    return (e.kind == 0) ? ((i == e.j) ? 1.0 : 0.0) : ((e.kind == 2) ? -1.0 : me);
  };
  double g00 = gcol(f0, k0, i0, 0), g01 = gcol(f0, k0, i0, 1), a0 = rhs(f0, k0, i0);
  double g10 = gcol(f1, k1, i1, 0), g11 = gcol(f1, k1, i1, 1), a1 = rhs(f1, k1, i1);
  // column 0: partial pivoting between the two real rows, one reciprocal
  const bool sw = fabs(g10) > fabs(g00);
  {
    const double t0 = g00, t1 = g01, t3 = a0;
    g00 = sw ? g10 : g00; g01 = sw ? g11 : g01; a0 = sw ? a1 : a0;
    g10 = sw ? t0 : g10; g11 = sw ? t1 : g11; a1 = sw ? t3 : a1;
  }
  const double inv0 = 1.0 / g00;
  g01 = g01 * inv0;
  a0 = a0 * inv0;
  g11 = __fma_rn(-g10, g01, g11);
  a1 = __fma_rn(-g10, a0, a1);
  // column 1
  const double inv1 = 1.0 / g11;
  a1 = a1 * inv1;
  a0 = __fma_rn(-g01, a1, a0);
  out.x[0] = a0;
  out.x[1] = a1;
  out.x[2] = 0.0;
  double uh[D + 1], sl = 0.0, sk = 0.0, s0 = 0.0;
#pragma unroll
  for (int c = 0; c <= D; ++c) uh[c] = 0.0;
  const bool c0 = 0 < mz, c1 = 1 < mz;
#pragma unroll
  for (int c = 0; c <= D; ++c) uh[c] = c0 ? __fma_rn(a0, fa[c], uh[c]) : uh[c];
  sk = c0 ? __fma_rn(a0, ka, sk) : sk;
  sl = (c0 && j0 == l) ? sl + a0 : sl;
  s0 = (mz == 0 && z0b) ? s0 + a0 : s0;
#pragma unroll
  for (int c = 0; c <= D; ++c) uh[c] = c1 ? __fma_rn(a1, fb[c], uh[c]) : uh[c];
  sk = c1 ? __fma_rn(a1, kb, sk) : sk;
  sl = (c1 && j1 == l) ? sl + a1 : sl;
  s0 = (mz == 1 && z0b) ? s0 + a1 : s0;
  if (e.kind == 2) s0 -= 1.0;
  const bool ez = e.kind == 1;
#pragma unroll
  for (int c = 0; c <= D; ++c) out.uh[c] = ez ? uh[c] - fe[c] : uh[c];
  out.sk = ez ? sk - ke : sk;
  out.sl = (ez && e.j == l) ? sl - 1.0 : sl;
  out.s0 = s0;
}

}  // namespace ca
