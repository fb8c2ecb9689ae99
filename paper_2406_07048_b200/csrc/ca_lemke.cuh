// ca_lemke.cuh -- one-thread-per-pair revised Lemke for the LCP of Eq. 24
// built from the equality-eliminated pair QP.
//
// Why revised, not a dense tableau: the LCP matrix
//     M = [[Kt Kt^T, kt], [-kt^T, 0]]
// is  M = F F^T + k e_l^T - e_l k^T  with F = [Kt; 0] (n x (d+1)), k = [kt; 0],
// l = n-1: rank <= d+3.  A basis B of Lemke's tableau B^{-1}[I | -M | -1 | q]
// therefore holds at most d+4 "structural" columns (basic z_j / z0); with R the
// equations whose w is nonbasic (|R| = m), B^{-1} a reduces to the m x m system
//     G x = a_R,  G[p][s] = a(zb_s)_{R_p},
// and every basic w_i's coefficient is  a_i + F_i.u + k_i sl - [i=l] sk + s0
// (u, sl, sk, s0 linear in x).  One pivot costs O(n (d+2) + m^3) FP64 instead of
// the O(n^2) dense tableau update, in registers of ONE thread, so a warp solves
// 32 pairs at once with no cross-lane traffic.
//
// Selection rules are DESIGN.md reading #4 (L1-L7), identical to the oracle's
// textbook full-tableau Lemke, except that ratios are compared by cross
// multiplication (one division per pivot): decisions coincide with the oracle
// except at near-ties closer than rounding (parity tests count those).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ca {

enum { ST_OK = 0, ST_RAY = 1, ST_ITER = 2, ST_NEGYE = 3 };
// variable labels: w_j -> j, z_j -> ZL + j, z0 -> Z0L
constexpr int ZL = 32;
constexpr int Z0L = 64;

struct LemkeParams {
  double pivot_tol, tie_tol;
  int max_pivot_factor;
};

// Thread-private rows of the reduced problem, in shared memory, layout
// [row][col][thread] (stride = threads per CTA) so a warp's accesses hit 32
// consecutive 8-byte words.  Row i < n-1: (Kt_i[0..D], kt_i); row n-1 (phi): 0.
template <int D>
struct Rows {
  double* p;
  int stride;
  __device__ __forceinline__ double F(int i, int c) const { return p[(i * (D + 2) + c) * stride]; }
  __device__ __forceinline__ double k(int i) const { return p[(i * (D + 2) + D + 1) * stride]; }
  __device__ __forceinline__ void setF(int i, int c, double v) const { p[(i * (D + 2) + c) * stride] = v; }
  __device__ __forceinline__ void setk(int i, double v) const { p[(i * (D + 2) + D + 1) * stride] = v; }
  // M_ij of Eq. 24 (i, j < n); row/col l = n-1 is stored as zeros
  __device__ __forceinline__ double M(int i, int j, int l) const {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c <= D; ++c) acc = __fma_rn(F(i, c), F(j, c), acc);
    if (j == l) acc = k(i);
    if (i == l) acc = -k(j);
    if (i == l && j == l) acc = 0.0;
    return acc;
  }
};

// a(v)_i: column of variable v in [I | -M | -1]
template <int D>
__device__ __forceinline__ double colval(const Rows<D>& W, int v, int i, int l) {
  if (v < ZL) return (v == i) ? 1.0 : 0.0;
  if (v == Z0L) return -1.0;
  return -W.M(i, v - ZL, l);
}

template <int D, int NMAX>
struct Lemke {
  static constexpr int MMAX = D + 4;
  // basic w_i: bit i of wmask; value rw[i]; tableau row roww[i]
  double rw[NMAX];
  int roww[NMAX];
  uint32_t wmask;
  // basic structural variables (z_j / z0): slots 0..m-1
  int m;
  int zl[MMAX], zr[MMAX];
  double rz[MMAX];
  // equations whose w is nonbasic: Rr[0..m-1]
  int Rr[MMAX];
  int n, l;
  int pivots, status;

  // Solve G x = a(e)_R and return the low-rank coefficients of the column
  // of entering variable e:  coef(w_i) = F_i.uh + k_i sl - [i=l] sk + s0.
  __device__ __forceinline__ void column(const Rows<D>& W, double* Gs, int gstride, int e,
                                         double x[MMAX], double uh[D + 1], double& sl, double& sk,
                                         double& s0) const {
#define GS(p_, c_) Gs[((p_) * (MMAX + 1) + (c_)) * gstride]
#pragma unroll
    for (int p = 0; p < MMAX; ++p) {
      if (p < m) {
        const int i = Rr[p];
#pragma unroll
        for (int s = 0; s < MMAX; ++s)
          if (s < m) GS(p, s) = colval<D>(W, zl[s], i, l);
        GS(p, MMAX) = colval<D>(W, e, i, l);
      }
    }
    // Gauss-Jordan with partial pivoting on [G | a] (m <= d+4, usually <= 3);
    // the right-hand side lives in column MMAX.
    int prow[MMAX];
    uint32_t used = 0;
#pragma unroll
    for (int c = 0; c < MMAX; ++c) {
      prow[c] = 0;
      if (c < m) {
        int pb = 0;
        double best = -1.0;
#pragma unroll
        for (int p = 0; p < MMAX; ++p) {
          if (p < m && !((used >> p) & 1u)) {
            double a = fabs(GS(p, c));
            if (a > best) { best = a; pb = p; }
          }
        }
        used |= 1u << pb;
        prow[c] = pb;
        const double inv = 1.0 / GS(pb, c);
#pragma unroll
        for (int cc = c; cc <= MMAX; ++cc)
          if (cc < m || cc == MMAX) GS(pb, cc) = GS(pb, cc) * inv;
#pragma unroll
        for (int p = 0; p < MMAX; ++p) {
          if (p < m && p != pb) {
            const double f = GS(p, c);
#pragma unroll
            for (int cc = c; cc <= MMAX; ++cc)
              if (cc < m || cc == MMAX) GS(p, cc) = __fma_rn(-f, GS(pb, cc), GS(p, cc));
          }
        }
      }
    }
#pragma unroll
    for (int s = 0; s < MMAX; ++s) x[s] = (s < m) ? GS(prow[s], MMAX) : 0.0;
#undef GS
#pragma unroll
    for (int c = 0; c <= D; ++c) uh[c] = 0.0;
    sl = sk = s0 = 0.0;
#pragma unroll
    for (int s = 0; s < MMAX; ++s) {
      if (s < m) {
        const int v = zl[s];
        if (v == Z0L) {
          s0 += x[s];
        } else {
          const int j = v - ZL;
#pragma unroll
          for (int c = 0; c <= D; ++c) uh[c] = __fma_rn(x[s], W.F(j, c), uh[c]);
          sk = __fma_rn(x[s], W.k(j), sk);
          if (j == l) sl += x[s];
        }
      }
    }
    if (e == Z0L) {
      s0 -= 1.0;
    } else if (e >= ZL) {
      const int j = e - ZL;
#pragma unroll
      for (int c = 0; c <= D; ++c) uh[c] -= W.F(j, c);
      sk -= W.k(j);
      if (j == l) sl -= 1.0;
    }
  }

  __device__ __forceinline__ double wcoef(const Rows<D>& W, int i, const double uh[D + 1], double sl,
                                          double sk, double s0) const {
    double c = s0;
#pragma unroll
    for (int cc = 0; cc <= D; ++cc) c = __fma_rn(W.F(i, cc), uh[cc], c);
    c = __fma_rn(W.k(i), sl, c);
    if (i == l) c -= sk;
    return c;
  }

  // Lexicographic tie-break (rare path): `tie` has bit r for each tied tableau
  // row; compares T[row][w_j] / cbar_row over j = 0..n-1, keeps the minimisers
  // (within tau), and returns the smallest surviving row (L5.4-5).
  __device__ __forceinline__ int lexico(const Rows<D>& W, double* Gs, int gstride, uint32_t tie,
                                        const double cw[NMAX], const double xe[MMAX], double tau) const {
    for (int j = 0; j < n && __popc(tie) > 1; ++j) {
      const bool basic_w = (wmask >> j) & 1u;
      double xj[MMAX], uh[D + 1], sl = 0.0, sk = 0.0, s0 = 0.0;
#pragma unroll
      for (int s = 0; s < MMAX; ++s) xj[s] = 0.0;
#pragma unroll
      for (int c = 0; c <= D; ++c) uh[c] = 0.0;
      if (!basic_w) column(W, Gs, gstride, j, xj, uh, sl, sk, s0);
      double vmin = 1e308;
      double vr[NMAX];
#pragma unroll
      for (int i = 0; i < NMAX; ++i) {
        vr[i] = 1e308;
        if (i < n && ((wmask >> i) & 1u) && ((tie >> roww[i]) & 1u)) {
          const double num = basic_w ? ((i == j) ? 1.0 : 0.0) : wcoef(W, i, uh, sl, sk, s0);
          vr[i] = num / cw[i];
          vmin = fmin(vmin, vr[i]);
        }
      }
      double vz[MMAX];
#pragma unroll
      for (int s = 0; s < MMAX; ++s) {
        vz[s] = 1e308;
        if (s < m && ((tie >> zr[s]) & 1u)) {
          vz[s] = (basic_w ? 0.0 : xj[s]) / xe[s];
          vmin = fmin(vmin, vz[s]);
        }
      }
      const double vt = vmin + tau * fmax(1.0, fabs(vmin));
      uint32_t keep = 0;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n && ((wmask >> i) & 1u) && ((tie >> roww[i]) & 1u) && vr[i] <= vt) keep |= 1u << roww[i];
#pragma unroll
      for (int s = 0; s < MMAX; ++s)
        if (s < m && ((tie >> zr[s]) & 1u) && vz[s] <= vt) keep |= 1u << zr[s];
      tie = keep;
    }
    return __ffs(tie) - 1;
  }

  // Run Lemke on q (registers), rows W.  Returns final status; z values in zU.
  __device__ __forceinline__ void solve(const Rows<D>& W, double* Gs, int gstride, const double q[NMAX], int n_,
                        const LemkeParams& P) {
    n = n_;
    l = n - 1;
    pivots = 0;
    status = ST_OK;
    m = 0;
    wmask = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
    double qmin = 1e308;
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
      rw[i] = q[i];
      roww[i] = i;
      if (i < n && q[i] < qmin) qmin = q[i];
    }
    if (!(qmin < 0.0)) return;  // L1
    // L2: z0 enters, leaving row = argmin q, ties -> largest index
    const double tau = P.tie_tol;
    double tl = qmin + tau * fmax(1.0, fabs(qmin));
    int r = 0;
#pragma unroll
    for (int i = 0; i < NMAX; ++i)
      if (i < n && q[i] <= tl) r = i;
    {
      // column of z0 is -1 everywhere (B = I): inv = -1
      double ve = 0.0;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i == r) ve = rw[i] * -1.0;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n && i != r) rw[i] = __fma_rn(1.0, ve, rw[i]);
      wmask &= ~(1u << r);
      Rr[0] = r;
      zl[0] = Z0L;
      zr[0] = r;
      rz[0] = ve;
      m = 1;
      pivots = 1;
    }
    int entering = ZL + r;  // complement of w_r
    const int maxpiv = P.max_pivot_factor * n;
    double cw[NMAX];
    for (;;) {
      if (pivots >= maxpiv) { status = ST_ITER; return; }
      double xe[MMAX], uh[D + 1], sl, sk, s0;
      column(W, Gs, gstride, entering, xe, uh, sl, sk, s0);
      // coefficients of basic w's and max |cbar|
      double cmax = 0.0;
#pragma unroll
      for (int i = 0; i < NMAX; ++i) {
        cw[i] = 0.0;
        if (i < n && ((wmask >> i) & 1u)) {
          cw[i] = wcoef(W, i, uh, sl, sk, s0);
          cmax = fmax(cmax, fabs(cw[i]));
        }
      }
#pragma unroll
      for (int s = 0; s < MMAX; ++s)
        if (s < m) cmax = fmax(cmax, fabs(xe[s]));
      const double thr = P.pivot_tol * fmax(1.0, cmax);
      // L5.2: minimum ratio max(rhs,0)/cbar over eligible rows (cross-multiplied)
      double bn = -1.0, bd = 1.0;  // best numerator / denominator
#pragma unroll
      for (int i = 0; i < NMAX; ++i) {
        if (i < n && ((wmask >> i) & 1u) && cw[i] > thr) {
          double nu = fmax(rw[i], 0.0);
          if (bn < 0.0 || nu * bd < bn * cw[i]) { bn = nu; bd = cw[i]; }
        }
      }
#pragma unroll
      for (int s = 0; s < MMAX; ++s) {
        if (s < m && xe[s] > thr) {
          double nu = fmax(rz[s], 0.0);
          if (bn < 0.0 || nu * bd < bn * xe[s]) { bn = nu; bd = xe[s]; }
        }
      }
      if (bn < 0.0) { status = ST_RAY; return; }
      const double thmin = bn / bd;
      const double tt = thmin + tau * fmax(1.0, thmin);
      uint32_t tie = 0;
      int z0row = -1;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n && ((wmask >> i) & 1u) && cw[i] > thr && fmax(rw[i], 0.0) <= tt * cw[i])
          tie |= 1u << roww[i];
#pragma unroll
      for (int s = 0; s < MMAX; ++s)
        if (s < m && xe[s] > thr && fmax(rz[s], 0.0) <= tt * xe[s]) {
          tie |= 1u << zr[s];
          if (zl[s] == Z0L) z0row = zr[s];
        }
      if (tie == 0) { status = ST_RAY; return; }  // cannot happen: the argmin is in
      int row;
      if (z0row >= 0) row = z0row;                     // L5.3
      else if (__popc(tie) == 1) row = __ffs(tie) - 1;
      else row = lexico(W, Gs, gstride, tie, cw, xe, tau);  // L5.4-5
      // identify the leaving variable at `row` and its coefficient / value
      int lw = -1, lzs = -1, lzl = 0;
      double cr = 0.0, vr = 0.0;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n && ((wmask >> i) & 1u) && roww[i] == row) { lw = i; cr = cw[i]; vr = rw[i]; }
#pragma unroll
      for (int s = 0; s < MMAX; ++s)
        if (s < m && zr[s] == row) { lzs = s; lzl = zl[s]; cr = xe[s]; vr = rz[s]; }
      // L3: pivot (rhs only; the structure is re-derived each pivot)
      const double inv = 1.0 / cr;
      const double ve = vr * inv;
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n && ((wmask >> i) & 1u) && i != lw) rw[i] = __fma_rn(-cw[i], ve, rw[i]);
#pragma unroll
      for (int s = 0; s < MMAX; ++s)
        if (s < m && s != lzs) rz[s] = __fma_rn(-xe[s], ve, rz[s]);
      ++pivots;
      const int leaving = (lw >= 0) ? lw : lzl;
      if (entering >= ZL && lw >= 0 && m >= MMAX) { status = ST_ITER; return; }  // rank bound d+4
      // basis bookkeeping
      if (entering < ZL) {  // w_j enters: leaves R
        const int j = entering;
        wmask |= 1u << j;
#pragma unroll
        for (int i = 0; i < NMAX; ++i)
          if (i == j) { rw[i] = ve; roww[i] = row; }
        int pj = 0;
#pragma unroll
        for (int p = 0; p < MMAX; ++p)
          if (p < m && Rr[p] == j) pj = p;
        if (lw >= 0) {  // w_i leaves: R swaps j -> i
          wmask &= ~(1u << lw);
#pragma unroll
          for (int p = 0; p < MMAX; ++p)
            if (p == pj) Rr[p] = lw;
        } else {  // z leaves (slot lzs): both sets shrink (swap-with-last)
          const int last = m - 1;
          int zlL = 0, zrL = 0, RrL = 0;
          double rzL = 0.0;
#pragma unroll
          for (int s = 0; s < MMAX; ++s)
            if (s == last) { zlL = zl[s]; zrL = zr[s]; rzL = rz[s]; RrL = Rr[s]; }
#pragma unroll
          for (int s = 0; s < MMAX; ++s) {
            if (s == lzs) { zl[s] = zlL; zr[s] = zrL; rz[s] = rzL; }
            if (s == pj) Rr[s] = RrL;
          }
          m = last;
        }
      } else {  // z_j / z0 enters
        if (lw >= 0) {  // w_i leaves: both sets grow
          wmask &= ~(1u << lw);
#pragma unroll
          for (int s = 0; s < MMAX; ++s)
            if (s == m) { zl[s] = entering; zr[s] = row; rz[s] = ve; Rr[s] = lw; }
          ++m;
        } else {  // z leaves: replace its slot
#pragma unroll
          for (int s = 0; s < MMAX; ++s)
            if (s == lzs) { zl[s] = entering; zr[s] = row; rz[s] = ve; }
        }
      }
      if (leaving == Z0L) return;  // L6
      entering = (leaving < ZL) ? ZL + leaving : leaving - ZL;  // L4
    }
  }

  // z_j values (LCP solution) into zU[0..n-1]
  __device__ __forceinline__ void solution(double zU[NMAX]) const {
#pragma unroll
    for (int j = 0; j < NMAX; ++j) zU[j] = 0.0;
#pragma unroll
    for (int s = 0; s < MMAX; ++s) {
      if (s < m && zl[s] != Z0L) {
        int j = zl[s] - ZL;
#pragma unroll
        for (int jj = 0; jj < NMAX; ++jj)
          if (jj == j) zU[jj] = rz[s];
      }
    }
  }

  __device__ __forceinline__ uint32_t zmask() const {
    uint32_t mk = 0;
#pragma unroll
    for (int s = 0; s < MMAX; ++s)
      if (s < m) mk |= (zl[s] == Z0L) ? 0x80000000u : (1u << (zl[s] - ZL));
    return mk;
  }
};

}  // namespace ca
