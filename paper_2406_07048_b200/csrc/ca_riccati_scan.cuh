// ca_riccati_scan.cuh -- ADMM step 2 (Eq. 16; one SQP QP per iteration,
// P:349-351) for small batches by a PARALLEL-IN-TIME LQ solve: the backward Riccati
// recursion of k_riccati (O(N) dependent steps on one warp) is replaced by an
// associative scan over the N+1 stages (log2(N+1) levels), one thread per stage.
//
// Stage t of the LQ (the same data as k_riccati: stage blocks H_t, h_t from the sweep's
// Gauss-Newton aggregates, dynamics s_{t+1} = A_t s_t + B_t u_t + c_t, control cost
// 1/2 u^T R_t u + r_t^T u with R_t = 2 Qu (+ rho_b on bounded controls), r_t the box
// block's linear term) is the element
//     e_t = (A, b, C, eta, J) = (A_t, c_t + B_t u0_t, B_t R_t^-1 B_t^T, -h_t, H_t),
//     u0_t = -R_t^-1 r_t   (t = 0: J = 0, eta = 0 -- s_0 is fixed; t = N: A = b = C = 0)
// of the conditional value function V_{t->t+1}(s_t | s_{t+1}) (Sarkka & Garcia-Fernandez,
// temporal parallelization of LQ control); the associative combination
//     T = (I + C_ij J_jk)^-1
//     A_ik = A_jk T A_ij          b_ik = A_jk T (b_ij + C_ij eta_jk) + b_jk
//     C_ik = A_jk T C_ij A_jk^T + C_jk
//     eta_ik = A_ij^T T^T (eta_jk - J_jk b_ij) + eta_ij
//     J_ik = A_ij^T T^T J_jk A_ij + J_ij
// composed over [t, N] (a suffix scan, Hillis-Steele, double-buffered in shared memory)
// gives the value function V_t(s) = 1/2 s^T J s - eta^T s, i.e. the Riccati P_t = J,
// p_t = -eta.  The gains then follow per stage in parallel with k_riccati's own formula
// (QuuSolve), and one thread rolls the dynamics forward exactly (riccati_forward).
// Different association order from the serial recursion: agreement to rounding of the
// LQ's conditioning (the T1 / T2 tests against the oracle's condensed Cholesky hold).
#pragma once
#include "ca_kernels.cuh"

namespace ca {

// A scan element / scratch record: one stage's fields contiguous, consecutive stages
// scan_pad doubles apart -- every field offset is then an immediate (no per-access
// stride arithmetic) and the threads of a warp, on consecutive stages, hit distinct
// shared-memory banks.
struct ElRef {
  double* p;
  __device__ __forceinline__ double& operator[](int k) const { return p[k]; }
};
// record stride: >= n, = 2 (mod 4) doubles -- 16-byte aligned records (vector loads of
// rows) whose 16-byte halves of consecutive stages fall on distinct bank groups
__host__ __device__ constexpr int scan_pad(int n) { return (n + 1) / 4 * 4 + 2; }
// rows of NS contiguous doubles to / from registers (16-byte vector accesses for even NS:
// every row offset of the element and scratch records is then even)
template <int NS>
__device__ __forceinline__ void ldrow(const double* p, double (&d)[NS]) {
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int i = 0; i < NS / 2; ++i) {
      const double2 v = reinterpret_cast<const double2*>(p)[i];
      d[2 * i] = v.x;
      d[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NS; ++i) d[i] = p[i];
  }
}
template <int NS>
__device__ __forceinline__ void strow(double* p, const double (&d)[NS]) {
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int i = 0; i < NS / 2; ++i) reinterpret_cast<double2*>(p)[i] = make_double2(d[2 * i], d[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < NS; ++i) p[i] = d[i];
  }
}
template <int NS>
__device__ __forceinline__ void ldmat(const double* p, double (&d)[NS][NS]) {
#pragma unroll
  for (int r = 0; r < NS; ++r) ldrow<NS>(p + r * NS, d[r]);
}

template <int NS>
struct ScanEl {
  static constexpr int A = 0, B = NS * NS, C = B + NS, ETA = C + NS * NS, J = ETA + NS, SIZE = J + NS * NS;
};

// T = M^-1 of a small matrix (NS <= 4) in closed form: the adjugate over one reciprocal
// of the determinant (2 x 2 minors for NS = 4) -- no pivoting, no data-dependent control,
// every entry independent.  M = I + C_ij J_jk has real eigenvalues >= 1 (C, J symmetric
// positive semidefinite), so det M >= 1.  CA_SCAN_INV_GE=1 selects Gauss-Jordan with
// partial pivoting instead (C4 primal step 42.8 vs 39.9 us with the adjugate; kept for A/B).
template <int NS>
__device__ __forceinline__ void scan_inverse(const double (&m)[NS][NS], double (&t)[NS][NS]) {
#if defined(CA_SCAN_INV_GE) && CA_SCAN_INV_GE
  double M[NS][NS];
#pragma unroll
  for (int r = 0; r < NS; ++r)
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      M[r][c] = m[r][c];
      t[r][c] = (r == c) ? 1.0 : 0.0;
    }
#pragma unroll
  for (int c = 0; c < NS; ++c) {
#pragma unroll
    for (int r = c + 1; r < NS; ++r) {
      const bool sw = fabs(M[r][c]) > fabs(M[c][c]);
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        const double t0 = M[c][q], t1 = t[c][q];
        M[c][q] = sw ? M[r][q] : t0;
        M[r][q] = sw ? t0 : M[r][q];
        t[c][q] = sw ? t[r][q] : t1;
        t[r][q] = sw ? t1 : t[r][q];
      }
    }
    const double inv = 1.0 / M[c][c];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      M[c][q] = M[c][q] * inv;
      t[c][q] = t[c][q] * inv;
    }
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      if (r == c) continue;
      const double f = M[r][c];
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        M[r][q] = __fma_rn(-f, M[c][q], M[r][q]);
        t[r][q] = __fma_rn(-f, t[c][q], t[r][q]);
      }
    }
  }
#else
  if constexpr (NS == 1) {
    t[0][0] = 1.0 / m[0][0];
  } else if constexpr (NS == 2) {
    const double inv = 1.0 / __fma_rn(m[0][0], m[1][1], -m[0][1] * m[1][0]);
    t[0][0] = m[1][1] * inv;
    t[0][1] = -m[0][1] * inv;
    t[1][0] = -m[1][0] * inv;
    t[1][1] = m[0][0] * inv;
  } else if constexpr (NS == 3) {
    double a[3][3];  // adjugate
    a[0][0] = __fma_rn(m[1][1], m[2][2], -m[1][2] * m[2][1]);
    a[0][1] = __fma_rn(m[0][2], m[2][1], -m[0][1] * m[2][2]);
    a[0][2] = __fma_rn(m[0][1], m[1][2], -m[0][2] * m[1][1]);
    a[1][0] = __fma_rn(m[1][2], m[2][0], -m[1][0] * m[2][2]);
    a[1][1] = __fma_rn(m[0][0], m[2][2], -m[0][2] * m[2][0]);
    a[1][2] = __fma_rn(m[0][2], m[1][0], -m[0][0] * m[1][2]);
    a[2][0] = __fma_rn(m[1][0], m[2][1], -m[1][1] * m[2][0]);
    a[2][1] = __fma_rn(m[0][1], m[2][0], -m[0][0] * m[2][1]);
    a[2][2] = __fma_rn(m[0][0], m[1][1], -m[0][1] * m[1][0]);
    const double det = __fma_rn(m[0][0], a[0][0], __fma_rn(m[0][1], a[1][0], m[0][2] * a[2][0]));
    const double inv = 1.0 / det;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) t[r][c] = a[r][c] * inv;
  } else {
    static_assert(NS == 4, "scan_inverse: NS <= 4");
    const double s0 = __fma_rn(m[0][0], m[1][1], -m[1][0] * m[0][1]);
    const double s1 = __fma_rn(m[0][0], m[1][2], -m[1][0] * m[0][2]);
    const double s2 = __fma_rn(m[0][0], m[1][3], -m[1][0] * m[0][3]);
    const double s3 = __fma_rn(m[0][1], m[1][2], -m[1][1] * m[0][2]);
    const double s4 = __fma_rn(m[0][1], m[1][3], -m[1][1] * m[0][3]);
    const double s5 = __fma_rn(m[0][2], m[1][3], -m[1][2] * m[0][3]);
    const double c5 = __fma_rn(m[2][2], m[3][3], -m[3][2] * m[2][3]);
    const double c4 = __fma_rn(m[2][1], m[3][3], -m[3][1] * m[2][3]);
    const double c3 = __fma_rn(m[2][1], m[3][2], -m[3][1] * m[2][2]);
    const double c2 = __fma_rn(m[2][0], m[3][3], -m[3][0] * m[2][3]);
    const double c1 = __fma_rn(m[2][0], m[3][2], -m[3][0] * m[2][2]);
    const double c0 = __fma_rn(m[2][0], m[3][1], -m[3][0] * m[2][1]);
    const double det = (s0 * c5 - s1 * c4) + (s2 * c3 + s3 * c2) + (s5 * c0 - s4 * c1);
    const double inv = 1.0 / det;
    auto e3 = [](double x0, double y0, double x1, double y1, double x2, double y2) {
      return __fma_rn(x2, y2, __fma_rn(x1, y1, x0 * y0));
    };
    t[0][0] = e3(m[1][1], c5, -m[1][2], c4, m[1][3], c3) * inv;
    t[0][1] = e3(-m[0][1], c5, m[0][2], c4, -m[0][3], c3) * inv;
    t[0][2] = e3(m[3][1], s5, -m[3][2], s4, m[3][3], s3) * inv;
    t[0][3] = e3(-m[2][1], s5, m[2][2], s4, -m[2][3], s3) * inv;
    t[1][0] = e3(-m[1][0], c5, m[1][2], c2, -m[1][3], c1) * inv;
    t[1][1] = e3(m[0][0], c5, -m[0][2], c2, m[0][3], c1) * inv;
    t[1][2] = e3(-m[3][0], s5, m[3][2], s2, -m[3][3], s1) * inv;
    t[1][3] = e3(m[2][0], s5, -m[2][2], s2, m[2][3], s1) * inv;
    t[2][0] = e3(m[1][0], c4, -m[1][1], c2, m[1][3], c0) * inv;
    t[2][1] = e3(-m[0][0], c4, m[0][1], c2, -m[0][3], c0) * inv;
    t[2][2] = e3(m[3][0], s4, -m[3][1], s2, m[3][3], s0) * inv;
    t[2][3] = e3(-m[2][0], s4, m[2][1], s2, -m[2][3], s0) * inv;
    t[3][0] = e3(-m[1][0], c3, m[1][1], c1, -m[1][2], c0) * inv;
    t[3][1] = e3(m[0][0], c3, -m[0][1], c1, m[0][2], c0) * inv;
    t[3][2] = e3(-m[3][0], s3, m[3][1], s1, -m[3][2], s0) * inv;
    t[3][3] = e3(m[2][0], s3, -m[2][1], s1, m[2][2], s0) * inv;
  }
#endif
}

// eo = ei (x) ej (ei covers stages [i, j), ej covers [j, k)), operands in shared memory:
// computed by a group of GS = 4 threads (row a of every output on thread a;
// rows a >= NS idle), the intermediates exchanged through the group's scratch `sh`
// (SCR doubles) -- the per-level latency of the scan is then a few short dependent
// chains instead of one thread's ~700 FP64 operations.  Each phase first loads all of
// its shared-memory operands into registers, then computes, then stores: operands and
// results live in one shared array, so interleaved loads and stores would be serialised
// by possible aliasing.  Every thread of the warp calls it (`on`: this group has a
// combination at this level) so the warp barriers match.  (One thread per matrix entry,
// 16 per element, measured slower: on the one SM of a single scene the 16-fold
// redundant inverse and operand loads saturate the FP64 pipe and shared-memory
// bandwidth -- profiles/README.md.)
template <int NS>
struct ScanScr {
  static constexpr int M = 0, G = NS * NS, H = G + NS, V = H + NS, X = V + NS * NS, Z = X + NS * NS, Y = Z + NS * NS,
                       W = Y + NS, SIZE = W + NS * NS;
};
template <int NS>
__device__ __forceinline__ void scan_comb_g(ElRef ei, ElRef ej, ElRef eo, int a, bool on, ElRef sh,
                                            long long* ts = nullptr) {
#ifdef CA_RIC_PROFILE
#define CG_TS(k) if (ts) ts[k] = clock64()
#else
#define CG_TS(k)
#endif
  CG_TS(0);
  using L = ScanEl<NS>;
  using S = ScanScr<NS>;
  const bool row = on && a < NS;
  // P1: row a of M = I + Ci Jj, g = bi + Ci nj, h = nj - Jj bi, V = Jj Ai
  if (row) {
    double ca_[NS], ja[NS], bi_[NS], nj_[NS], Jj_[NS][NS], Ai_[NS][NS];
    double gs = ei[L::B + a], hs = ej[L::ETA + a];
    ldrow<NS>(&ei[L::C + a * NS], ca_);
    ldrow<NS>(&ej[L::J + a * NS], ja);
    ldrow<NS>(&ei[L::B], bi_);
    ldrow<NS>(&ej[L::ETA], nj_);
    ldmat<NS>(&ej[L::J], Jj_);
    ldmat<NS>(&ei[L::A], Ai_);
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      gs = __fma_rn(ca_[q], nj_[q], gs);
      hs = __fma_rn(-ja[q], bi_[q], hs);
    }
    double m_[NS], v_[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double m = (a == c) ? 1.0 : 0.0, v = 0.0;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        m = __fma_rn(ca_[q], Jj_[q][c], m);
        v = __fma_rn(ja[q], Ai_[q][c], v);
      }
      m_[c] = m;
      v_[c] = v;
    }
    sh[S::G + a] = gs;
    sh[S::H + a] = hs;
    strow<NS>(&sh[S::M + a * NS], m_);
    strow<NS>(&sh[S::V + a * NS], v_);
  }
  CG_TS(1);
  __syncwarp();
  CG_TS(2);
  // P2: T = M^-1 (redundantly per thread, scan_inverse); row a of X = T Ai, Z = T Ci, y = T g
  if (row) {
    double M[NS][NS], T[NS][NS], Ai_[NS][NS], Ci_[NS][NS], g_[NS];
    ldrow<NS>(&sh[S::G], g_);
    ldmat<NS>(&sh[S::M], M);
    ldmat<NS>(&ei[L::A], Ai_);
    ldmat<NS>(&ei[L::C], Ci_);
    scan_inverse<NS>(M, T);
    double Ta[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {  // row a of T (a run-time index: select, no local array)
      double v = T[0][q];
#pragma unroll
      for (int r = 1; r < NS; ++r) v = (r == a) ? T[r][q] : v;
      Ta[q] = v;
    }
    double sy = 0.0, sx_[NS], sz_[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) sy = __fma_rn(Ta[q], g_[q], sy);
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double sx = 0.0, sz = 0.0;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        sx = __fma_rn(Ta[q], Ai_[q][c], sx);
        sz = __fma_rn(Ta[q], Ci_[q][c], sz);
      }
      sx_[c] = sx;
      sz_[c] = sz;
    }
    sh[S::Y + a] = sy;
    strow<NS>(&sh[S::X + a * NS], sx_);
    strow<NS>(&sh[S::Z + a * NS], sz_);
  }
  CG_TS(3);
  __syncwarp();
  // P3: rows a of A_ik = Aj X, b_ik = Aj y + bj, W = Aj Z, eta_ik = X^T h + ni,
  // J_ik = sym(X^T V) + Ji
  if (row) {
    double aj[NS], y_[NS], h_[NS], X_[NS][NS], Z_[NS][NS], V_[NS][NS], xa[NS], va[NS], ji[NS];
    double sb = ej[L::B + a], se = ei[L::ETA + a];
    ldrow<NS>(&ej[L::A + a * NS], aj);
    ldrow<NS>(&sh[S::Y], y_);
    ldrow<NS>(&sh[S::H], h_);
    ldrow<NS>(&ei[L::J + a * NS], ji);
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      xa[q] = sh[S::X + q * NS + a];
      va[q] = sh[S::V + q * NS + a];
    }
    ldmat<NS>(&sh[S::X], X_);
    ldmat<NS>(&sh[S::Z], Z_);
    ldmat<NS>(&sh[S::V], V_);
#pragma unroll
    for (int q = 0; q < NS; ++q) sb = __fma_rn(aj[q], y_[q], sb);
#pragma unroll
    for (int q = 0; q < NS; ++q) se = __fma_rn(xa[q], h_[q], se);
    double oa[NS], ow[NS], oj[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double sa = 0.0, sw = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        sa = __fma_rn(aj[q], X_[q][c], sa);
        sw = __fma_rn(aj[q], Z_[q][c], sw);
        s1 = __fma_rn(xa[q], V_[q][c], s1);
        s2 = __fma_rn(X_[q][c], va[q], s2);
      }
      oa[c] = sa;
      ow[c] = sw;
      oj[c] = 0.5 * (s1 + s2) + ji[c];
    }
    eo[L::B + a] = sb;
    eo[L::ETA + a] = se;
    strow<NS>(&eo[L::A + a * NS], oa);
    strow<NS>(&sh[S::W + a * NS], ow);
    strow<NS>(&eo[L::J + a * NS], oj);
  }
  CG_TS(4);
  __syncwarp();
  // P4: row a of C_ik = sym(W Aj^T) + Cj
  if (row) {
    double W_[NS][NS], Aj_[NS][NS], wa[NS], aa[NS], cj[NS];
    ldrow<NS>(&sh[S::W + a * NS], wa);
    ldrow<NS>(&ej[L::A + a * NS], aa);
    ldrow<NS>(&ej[L::C + a * NS], cj);
    ldmat<NS>(&sh[S::W], W_);
    ldmat<NS>(&ej[L::A], Aj_);
    double oc[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        s1 = __fma_rn(wa[q], Aj_[c][q], s1);
        s2 = __fma_rn(W_[c][q], aa[q], s2);
      }
      oc[c] = 0.5 * (s1 + s2) + cj[c];
    }
    strow<NS>(&eo[L::C + a * NS], oc);
  }
  CG_TS(5);
#undef CG_TS
}

// Row r of stage_assemble (ca_kernels.cuh) for stage t of scene b: the same arithmetic in
// the same order per entry (H_t row r, h_t entry r; the statistics on row 0), so the stage
// blocks equal the serial path's bit for bit.  sref / sk: this stage's s_ref and s rows.
template <int NS>
__device__ __forceinline__ void stage_assemble_row(const Dev& P, int b, int t, int r, const double* rec, double* out,
                                                   double* so, const double* Qs, const double* sref,
                                                   const double* sk) {
  const int N = P.N, npc = P.npc, L1 = P.d + 1;
  const double sig = P.sigma;
  double* ho = out + NS * NS;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < NS; ++c) {
    out[r * NS + c] = 2.0 * Qs[r * NS + c];
    acc += Qs[r * NS + c] * sref[c];
  }
  ho[r] = -2.0 * acc;
  // the pose component a with pidx[a] = r (if any): S (Gauss-Newton block) and g terms
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    if (a >= npc || P.pidx[a] != r) continue;
    double spv = (a < L1) ? rec[L1 * (L1 + 1) / 2 + a] : 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= npc) continue;
      const int lo = (a <= c) ? a : c, hi = (a <= c) ? c : a;
      const double Sac = (hi < L1) ? rec[sym_idx(lo, hi, L1)] : 0.0;
      spv -= Sac * sk[P.pidx[c]];
      out[r * NS + P.pidx[c]] += sig * Sac;
    }
    ho[r] += sig * spv;
  }
  if (P.box && box_on(P.box_lim[r], P.box_lim[NS + r])) {  // (rho_b/2) ||s_t - w_t + l_t||^2 (reading #7)
    const long long k0 = ((long long)b * (N + 1) + t) * NS;
    out[r * NS + r] += P.box_rho;
    ho[r] += -P.box_rho * (P.box_ws[k0 + r] - P.box_ls[k0 + r]);
  }
  if (r == 0)
#pragma unroll
    for (int f = 0; f < NSTAT; ++f) so[f] = rec[P.nagg + f];
}

// asynchronous 8-byte global -> shared copy (cp.async, L1-allocating) and its wait
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// threads per scan element (rows of the combination)
constexpr int SCAN_GS = 4;
__host__ __device__ inline long long riccati_scan_smem_doubles(int N, int NS, int NU, bool dyn_pt) {
  // the kernel's layout (k_riccati_scan below); per-stage rows padded to an odd number of
  // doubles so that consecutive stages fall on distinct shared-memory banks
  const int EL = 3 * NS * NS + 2 * NS;
  const int SCR = NS * NS * 5 + 3 * NS;        // ScanScr<NS>::SIZE
  const int SBS = (NS * NS + NS) | 1, DBS = (NS * NS + NS * NU + NS) | 1, PHIS = (NS * NS + NS) | 1, XSS = NS | 1;
  return (long long)N * SBS + (long long)NSTAT * N + (long long)(dyn_pt ? N : 1) * DBS + (long long)N * NU * (NS + 1) +
         1 + (N + 1LL) * (2 * scan_pad(EL) + scan_pad(SCR)) + (long long)N * PHIS + (long long)(N + 1) * XSS + 2LL * N +
         NS * NS + 2LL * (N + 1) * NS;
}

// One CTA per scene, blockDim = SCAN_GS * (N + 1) rounded up to a multiple of 32.
// Shared memory: k_riccati's layout (stage blocks, statistics, dynamics, gains), then two
// element buffers, the combination scratch, the closed-loop maps, the states, and the
// per-stage box residuals.
template <int NS, int NU>
__global__ void k_riccati_scan(Dev P, const double* recs, int nchunk, double* dst_cur, double* dst_prev) {
  extern __shared__ double rsm[];
  const int b = blockIdx.x, tid = threadIdx.x, nth = blockDim.x;
  if (!scene_on(P, b)) return;  // stopped scene (ca_admm_solve)
  const int N = P.N;
  constexpr int SB = NS * NS + NS, DB = NS * NS + NS * NU + NS, EL = ScanEl<NS>::SIZE, SCR = ScanScr<NS>::SIZE,
                PHI = NS * NS + NS;
  // per-stage row strides, odd: consecutive stages on distinct banks (riccati_scan_smem_doubles)
  constexpr int SBS = SB | 1, DBS = DB | 1, PHIS = PHI | 1, XSS = NS | 1;
  using L = ScanEl<NS>;
  double* sstg = rsm;                         // [N][SB]
  double* sst = sstg + (long long)N * SBS;    // [N][NSTAT]
  double* sdyn = sst + (long long)NSTAT * N;  // [nd][DB]
  const int nd = P.dyn_pt ? N : 1;
  double* ric = sdyn + (long long)nd * DBS;   // [N][NU][NS+1]
  constexpr int ELP = scan_pad(EL), SCRP = scan_pad(SCR);  // element / scratch record strides
  // [N+1][ELP], 16-byte aligned (vector row accesses)
  double* E0 = ric + (((long long)N * NU * (NS + 1) + (ric - rsm) + 1) & ~1LL) - (ric - rsm);
  double* E1 = E0 + (N + 1LL) * ELP;
  double* scr = E1 + (N + 1LL) * ELP;            // [N+1][SCRP]
  double* phi = scr + (N + 1LL) * SCRP;          // [N][PHIS]: x_{t+1} = Phi_t x_t + phi_t
  double* xs = phi + (long long)N * PHIS;        // [N+1][XSS]
  double* rbx = xs + (long long)(N + 1) * XSS;   // [N] box residual of stage t
  double* sQs = rbx + 2LL * N;                   // Qs, this scene's s_ref and s rows
  double* ssref = sQs + NS * NS;
  double* ss_ = ssref + (long long)(N + 1) * NS;
  double* rsum = E0;  // [N][rec] per-(t, field) record sums (E0 is free until the elements are built)
#ifdef CA_RIC_PROFILE
  long long tp[10];
  int np_ = 0;
#define RIC_TS() (tp[np_++] = clock64())
#else
#define RIC_TS() ((void)0)
#endif
  RIC_TS();
  // (1) asynchronous 8-byte copies into shared memory (cp.async: every element in flight
  // at once, no register staging) of Qs, this scene's s_ref and s rows and the dynamics;
  // meanwhile the per-(t, field) sums of the chunk records straight from global memory
  // (entry k = (t, f): field f of timestep t+1 summed over the chunk records in chunk
  // order, the max for S_PMAX; the loads of up to RU entries per thread in flight together)
  auto bulk = [&](double* dst, const double* __restrict__ src, long long tot) {
    for (long long k = tid; k < tot; k += nth) cp_async8(dst + k, src + k);
  };
  bulk(sQs, P.Qs, NS * NS);
  bulk(ssref, P.sref + (long long)b * (N + 1) * NS, (long long)(N + 1) * NS);
  bulk(ss_, P.s + (long long)b * (N + 1) * NS, (long long)(N + 1) * NS);
  {
    const long long idx0 = P.dyn_ps ? (long long)b * nd : 0;
    auto stage_dyn = [&](const double* __restrict__ src, int blk, int off) {
      const int tot = nd * blk;
      for (int k = tid; k < tot; k += nth) cp_async8(sdyn + (k / blk) * DBS + off + k % blk, src + k);
    };
    stage_dyn(P.dynA + idx0 * NS * NS, NS * NS, 0);
    stage_dyn(P.dynB + idx0 * NS * NU, NS * NU, NS * NS);
    stage_dyn(P.dync + idx0 * NS, NS, NS * NS + NS * NU);
  }
  {
    const int RC = P.rec, fm = P.nagg + S_PMAX, nc = nchunk ? nchunk : 1, tot = N * RC;
    CA_CHECK(rsum + (long long)tot <= E0 + (N + 1LL) * ELP);
    constexpr int RU = 4, CU = 4;  // entries per thread in flight together; chunks per batch
    for (int k0 = tid; k0 < tot; k0 += RU * nth) {
      const double* src[RU];
      long long step = 0;
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int k = k0 + u * nth, kk = (k < tot) ? k : 0;
        const int t = kk / RC, f = kk - t * RC;
        // rec_index(P, b, t + 1, c) = base + c TG (the sweep's layout), else (scene, t)
        const long long base =
            nchunk ? (((long long)b * P.NG + t / P.TG) * P.nchunkG) * P.TG + t % P.TG : (long long)b * N + t;
        src[u] = recs + base * RC + f;
        step = (long long)P.TG * RC;
      }
      double acc[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) acc[u] = 0.0;
      for (int c0 = 0; c0 < nc; c0 += CU) {
        double v[RU][CU];
#pragma unroll
        for (int u = 0; u < RU; ++u)
#pragma unroll
          for (int cc = 0; cc < CU; ++cc)
            v[u][cc] = (k0 + u * nth < tot && c0 + cc < nc) ? __ldg(src[u] + (c0 + cc) * step) : 0.0;
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const bool mx = (k0 + u * nth) % RC == fm;
#pragma unroll
          for (int cc = 0; cc < CU; ++cc)
            if (c0 + cc < nc) acc[u] = mx ? fmax(acc[u], v[u][cc]) : acc[u] + v[u][cc];
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u)
        if (k0 + u * nth < tot) rsum[k0 + u * nth] = acc[u];
    }
  }
  cp_async_wait_all();
  __syncthreads();
  RIC_TS();
  {
    const int RC = P.rec;
    // stage_assemble's H_t, h_t and statistics, row r of stage t+1 on thread (t, r)
    for (int t0 = 0; t0 < N; t0 += nth / SCAN_GS) {
      const int t = t0 + tid / SCAN_GS, r = tid % SCAN_GS;
      if (t < N && r < NS)
        stage_assemble_row<NS>(P, b, t + 1, r, rsum + (long long)t * RC, sstg + (long long)t * SBS,
                               sst + (long long)NSTAT * t, sQs, ssref + (long long)(t + 1) * NS,
                               ss_ + (long long)(t + 1) * NS);
    }
  }
  __syncthreads();
  RIC_TS();
  // control weights R = 2 Qu + rho_b (bounded controls), shared by all stages
  double Rm[NU][NU], urho[NU];
#pragma unroll
  for (int a = 0; a < NU; ++a) {
    const double lo = P.box ? P.box_lim[2 * NS + a] : -INFINITY, hi = P.box ? P.box_lim[2 * NS + NU + a] : INFINITY;
    urho[a] = (P.box && box_on(lo, hi)) ? P.box_rho : 0.0;
  }
#pragma unroll
  for (int a = 0; a < NU; ++a)
#pragma unroll
    for (int c = 0; c < NU; ++c) Rm[a][c] = 2.0 * P.Qu[a * NU + c] + ((a == c) ? urho[a] : 0.0);
  QuuSolve<NU> rs;
  rs.factor(Rm);
  // (2) elements, SCAN_GS threads per stage (row a each): u0 = -R^-1 r_t (the box block's
  // linear control term, redundantly), column a of R^-1 B^T through the scratch, then
  // row a of A, b = c + B u0, C = B R^-1 B^T, J = H_t, eta = -h_t
  constexpr int RBF = 0;  // scratch field of (R^-1 B^T)[q][c]: RBF + q NS + c of the stage's record
  for (int t0 = 0; t0 <= N; t0 += nth / SCAN_GS) {
    const int t = t0 + tid / SCAN_GS, a = tid % SCAN_GS;
    const bool live = t < N && a < NS;
    const double* A = sdyn + (P.dyn_pt ? (long long)(t < N ? t : 0) * DBS : 0);
    const double* Bm = A + NS * NS;
    const double* cv = Bm + NS * NU;
    const ElRef sc{scr + (long long)t * SCRP};
    if (live) {
      double col[NU];
#pragma unroll
      for (int q = 0; q < NU; ++q) col[q] = Bm[a * NU + q];
      rs.apply(col);
#pragma unroll
      for (int q = 0; q < NU; ++q) sc[RBF + q * NS + a] = col[q];
    }
    __syncwarp();
    if (t <= N && a < NS) {
      const ElRef e{E0 + (long long)t * ELP};
      if (t < N) {
        double u0[NU];
#pragma unroll
        for (int q = 0; q < NU; ++q) {
          const long long ku = ((long long)b * N + t) * NU + q;
          u0[q] = (urho[q] != 0.0) ? urho[q] * (P.box_wu[ku] - P.box_lu[ku]) : 0.0;  // -r_t
        }
        rs.apply(u0);
        double s = cv[a];
#pragma unroll
        for (int q = 0; q < NU; ++q) s = __fma_rn(Bm[a * NU + q], u0[q], s);
        e[L::B + a] = s;
        double rb[NU][NS];
#pragma unroll
        for (int q = 0; q < NU; ++q)
#pragma unroll
          for (int c = 0; c < NS; ++c) rb[q][c] = sc[RBF + q * NS + c];
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          e[L::A + a * NS + c] = A[a * NS + c];
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < NU; ++q) v = __fma_rn(Bm[a * NU + q], rb[q][c], v);
          e[L::C + a * NS + c] = v;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NS; ++c) e[L::A + a * NS + c] = e[L::C + a * NS + c] = 0.0;
        e[L::B + a] = 0.0;
      }
      if (t >= 1) {  // stage cost 1/2 s^T H_t s + h_t^T s  ->  J = H_t, eta = -h_t
        const double* in = sstg + (long long)(t - 1) * SBS;
#pragma unroll
        for (int c = 0; c < NS; ++c) e[L::J + a * NS + c] = in[a * NS + c];
        e[L::ETA + a] = -in[NS * NS + a];
      } else {
#pragma unroll
        for (int c = 0; c < NS; ++c) e[L::J + a * NS + c] = 0.0;
        e[L::ETA + a] = 0.0;
      }
    }
    __syncwarp();
  }
  __syncthreads();
  RIC_TS();
  // (3) suffix scan: e_t <- e_t (x) e_{t+1} (x) ... (x) e_N, SCAN_GS threads per element
  double* cur = E0;
  double* nxt = E1;
  const int per = nth / SCAN_GS;
  const int gi = tid / SCAN_GS, ga = tid % SCAN_GS;
  for (int d = 1; d <= N; d <<= 1) {
    for (int e0 = 0; e0 <= N; e0 += per) {
      const int t = e0 + gi;
      const bool have = t <= N, on = have && t + d <= N;
      if (have && !on) {  // no partner: carried over
        const ElRef ei{cur + (long long)t * ELP}, eo{nxt + (long long)t * ELP};
        for (int k = ga; k < EL; k += SCAN_GS) eo[k] = ei[k];
      }
      const int tc = have ? t : 0;
      const int tj = on ? t + d : tc;
#ifdef CA_RIC_PROFILE
      long long cg[6] = {0, 0, 0, 0, 0, 0};
      scan_comb_g<NS>(ElRef{cur + tc * ELP}, ElRef{cur + tj * ELP}, ElRef{nxt + tc * ELP}, ga, on, ElRef{scr + tc * SCRP}, cg);
      if (tid == 0 && b == 0 && d == 1)
        printf("comb cycles: P1 %lld sync %lld P2 %lld P3 %lld P4 %lld\n", cg[1] - cg[0], cg[2] - cg[1], cg[3] - cg[2],
               cg[4] - cg[3], cg[5] - cg[4]);
#else
      scan_comb_g<NS>(ElRef{cur + tc * ELP}, ElRef{cur + tj * ELP}, ElRef{nxt + tc * ELP}, ga, on, ElRef{scr + tc * SCRP});
#endif
    }
    __syncthreads();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  RIC_TS();
  // (4) gains of every stage from P_{t+1} = J, p_{t+1} = -eta (k_riccati's formula, the
  // same sums in the same order), SCAN_GS threads per stage through the scratch:
  //   G1 row a < NS of PA = P A, PB = P B, w = P c - eta_{t+1}
  //   G2 row a < NU of Quu = R + B^T PB, Qux = B^T PA, qu = -r + B^T w
  //   G3 Quu factored (redundantly), columns a, a + GS, .. of K = -Quu^-1 [Qux | qu]
  //   G4 row a < NS of the closed-loop map x_{t+1} = (A + B K) x_t + (B k + c)
  {
    constexpr int FPA = 0, FPB = FPA + NS * NS, FW = FPB + NS * NU, FQUU = FW + NS, FQUX = FQUU + NU * NU,
                  FQU = FQUX + NU * NS;
    static_assert(FQU + NU <= ScanScr<NS>::SIZE, "gains scratch");
    for (int t0 = 0; t0 < N; t0 += nth / SCAN_GS) {
      const int t = t0 + tid / SCAN_GS, a = tid % SCAN_GS;
      const bool st = t < N;
      const int tt = st ? t : 0;
      const ElRef e{cur + (tt + 1LL) * ELP}, sc{scr + (long long)tt * SCRP};
      const double* A = sdyn + (P.dyn_pt ? (long long)tt * DBS : 0);
      const double* Bm = A + NS * NS;
      const double* cv = Bm + NS * NU;
      if (st && a < NS) {  // G1
        double jr[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) jr[k] = e[L::J + a * NS + k];
        double acc = -e[L::ETA + a];
#pragma unroll
        for (int c = 0; c < NS; ++c) acc = __fma_rn(jr[c], cv[c], acc);
        sc[FW + a] = acc;
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < NS; ++k) s = __fma_rn(jr[k], A[k * NS + c], s);
          sc[FPA + a * NS + c] = s;
        }
#pragma unroll
        for (int c = 0; c < NU; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < NS; ++k) s = __fma_rn(jr[k], Bm[k * NU + c], s);
          sc[FPB + a * NU + c] = s;
        }
      }
      __syncwarp();
      if (st && a < NU) {  // G2
        double bc[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) bc[k] = Bm[k * NU + a];
#pragma unroll
        for (int c = 0; c < NU; ++c) {
          double s = 2.0 * P.Qu[a * NU + c] + ((a == c) ? urho[a] : 0.0);
#pragma unroll
          for (int k = 0; k < NS; ++k) s = __fma_rn(bc[k], sc[FPB + k * NU + c], s);
          sc[FQUU + a * NU + c] = s;
        }
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < NS; ++k) s = __fma_rn(bc[k], sc[FPA + k * NS + c], s);
          sc[FQUX + a * NS + c] = s;
        }
        const long long ku = ((long long)b * N + t) * NU + a;
        double s = (urho[a] != 0.0) ? -urho[a] * (P.box_wu[ku] - P.box_lu[ku]) : 0.0;
#pragma unroll
        for (int k = 0; k < NS; ++k) s = __fma_rn(bc[k], sc[FW + k], s);
        sc[FQU + a] = s;
      }
      __syncwarp();
      if (st) {  // G3
        double Quu[NU][NU];
#pragma unroll
        for (int q = 0; q < NU; ++q)
#pragma unroll
          for (int c = 0; c < NU; ++c) Quu[q][c] = sc[FQUU + q * NU + c];
        QuuSolve<NU> qs;
        qs.factor(Quu);
        for (int c = a; c <= NS; c += SCAN_GS) {
          double rhs[NU];
#pragma unroll
          for (int q = 0; q < NU; ++q) rhs[q] = (c < NS) ? sc[FQUX + q * NS + c] : sc[FQU + q];
          qs.apply(rhs);
#pragma unroll
          for (int q = 0; q < NU; ++q) ric[((long long)t * NU + q) * (NS + 1) + c] = -rhs[q];
        }
      }
      __syncwarp();
      if (st && a < NS) {  // G4
        double kg[NU][NS + 1];
#pragma unroll
        for (int q = 0; q < NU; ++q)
#pragma unroll
          for (int c = 0; c <= NS; ++c) kg[q][c] = ric[((long long)t * NU + q) * (NS + 1) + c];
        double* ph = phi + (long long)t * PHIS;
        double s = cv[a];
#pragma unroll
        for (int q = 0; q < NU; ++q) s = __fma_rn(Bm[a * NU + q], kg[q][NS], s);
        ph[NS * NS + a] = s;
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          double v = A[a * NS + c];
#pragma unroll
          for (int q = 0; q < NU; ++q) v = __fma_rn(Bm[a * NU + q], kg[q][c], v);
          ph[a * NS + c] = v;
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  RIC_TS();
  // (5) forward x_{t+1} = Phi_t x_t + phi_t from s_0, in chunks of FC stages:
  //   F1 each chunk's composed map (Psi, psi), column c of it on thread (chunk, c)
  //      (column NS = the affine part), so no exchange is needed;
  //   F2 one thread: the chunk start states x_{jFC} = Psi x + psi, chunk after chunk;
  //   F3 each chunk rolls its own stages from its start state, one rounding per step
  //      (Eq. 13b holds to one rounding per step inside a chunk, and to the chunk map's
  //      rounding at a chunk's last step).
  {
    constexpr int FC = 7, CW = NS * NS + NS;  // stages per chunk (odd: chunk rows on distinct banks); map size
    const int nch = (N + FC - 1) / FC;
    double* cmap = scr;  // [nch][CW]: Psi (row-major), psi
    for (int k = tid; k < nch * (NS + 1); k += nth) {  // F1
      const int j = k / (NS + 1), c = k % (NS + 1);
      double v[NS];
#pragma unroll
      for (int a = 0; a < NS; ++a) v[a] = (c < NS && a == c) ? 1.0 : 0.0;
      const int t1 = min(N, (j + 1) * FC);
#pragma unroll
      for (int u = 0; u < FC; ++u) {
        const int t = j * FC + u;
        if (t >= t1) break;
        const double* ph = phi + (long long)t * PHIS;
        double w[NS];
#pragma unroll
        for (int a = 0; a < NS; ++a) {
          double s = (c == NS) ? ph[NS * NS + a] : 0.0;
#pragma unroll
          for (int q = 0; q < NS; ++q) s = __fma_rn(ph[a * NS + q], v[q], s);
          w[a] = s;
        }
#pragma unroll
        for (int a = 0; a < NS; ++a) v[a] = w[a];
      }
#pragma unroll
      for (int a = 0; a < NS; ++a) cmap[(long long)j * CW + ((c < NS) ? a * NS + c : NS * NS + a)] = v[a];
    }
    __syncthreads();
    if (tid == 0) {  // F2
      double x[NS];
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        x[a] = P.s0[b * NS + a];
        xs[a] = x[a];
      }
      for (int j = 0; j + 1 < nch; ++j) {
        const double* m = cmap + (long long)j * CW;
        double xn[NS];
#pragma unroll
        for (int a = 0; a < NS; ++a) {
          double s = m[NS * NS + a];
#pragma unroll
          for (int c = 0; c < NS; ++c) s = __fma_rn(m[a * NS + c], x[c], s);
          xn[a] = s;
        }
#pragma unroll
        for (int a = 0; a < NS; ++a) {
          x[a] = xn[a];
          xs[(long long)(j + 1) * FC * XSS + a] = xn[a];
        }
      }
    }
    __syncthreads();
    for (int j = tid; j < nch; j += nth) {  // F3
      double x[NS];
#pragma unroll
      for (int a = 0; a < NS; ++a) x[a] = xs[(long long)j * FC * XSS + a];
      const int t1 = min(N, (j + 1) * FC);
#pragma unroll
      for (int u = 0; u < FC; ++u) {
        const int t = j * FC + u;
        if (t >= t1) break;
        const double* ph = phi + (long long)t * PHIS;
        double xn[NS];
#pragma unroll
        for (int a = 0; a < NS; ++a) {
          double s = ph[NS * NS + a];
#pragma unroll
          for (int c = 0; c < NS; ++c) s = __fma_rn(ph[a * NS + c], x[c], s);
          xn[a] = s;
        }
#pragma unroll
        for (int a = 0; a < NS; ++a) x[a] = xn[a];
        if (t + 1 < t1 || t + 1 == N)
#pragma unroll
          for (int a = 0; a < NS; ++a) xs[(long long)(t + 1) * XSS + a] = xn[a];
      }
    }
  }
  __syncthreads();
  RIC_TS();
  // (6) every stage in parallel: u_t = K_t x_t + k_t, the trajectory, the box block's
  // w, l update (reading #7) and its residual terms
  const double box_res_prev = (P.box && tid == 0) ? P.box_res[b] : 0.0;
  for (int t = tid; t <= N; t += nth) {
    double* sb = P.s + ((long long)b * (N + 1) + t) * NS;
#pragma unroll
    for (int a = 0; a < NS; ++a) sb[a] = xs[(long long)t * XSS + a];
    if (t == N) continue;
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < NU; ++a) {
      double s = ric[((long long)t * NU + a) * (NS + 1) + NS];
#pragma unroll
      for (int c = 0; c < NS; ++c) s = __fma_rn(ric[((long long)t * NU + a) * (NS + 1) + c], xs[(long long)t * XSS + c], s);
      const long long ku = ((long long)b * N + t) * NU + a;
      P.u[ku] = s;
      if (P.box && urho[a] != 0.0) {
        const double lo = P.box_lim[2 * NS + a], hi = P.box_lim[2 * NS + NU + a];
        r += box_update(s, lo, hi, &P.box_wu[ku], &P.box_lu[ku]);
      }
    }
    if (P.box) {  // states of t + 1
      const long long k0 = ((long long)b * (N + 1) + t + 1) * NS;
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        const double lo = P.box_lim[a], hi = P.box_lim[NS + a];
        if (box_on(lo, hi)) r += box_update(xs[(long long)(t + 1) * XSS + a], lo, hi, &P.box_ws[k0 + a], &P.box_ls[k0 + a]);
      }
    }
    rbx[t] = r;
  }
  __syncthreads();
  // (7) per-scene statistics: thread f sums field f over the stages in order, thread
  // NSTAT the box residuals; thread 0 writes
  double* sred = xs;  // (states no longer needed: reuse)
  if (tid < NSTAT) {
    double a = 0.0;
#pragma unroll 8
    for (int t = 0; t < N; ++t) a = stat_comb(tid, a, sst[(long long)NSTAT * t + tid]);
    sred[tid] = a;
  } else if (tid == NSTAT && P.box) {
    double br = 0.0;
#pragma unroll 8
    for (int t = 0; t < N; ++t) br += rbx[t];
    P.box_res[b] = br;
  }
  __syncthreads();
  if (tid == 0) {
    if (dst_cur)
#pragma unroll
      for (int f = 0; f < NSTAT; ++f)
        if (f != S_RPRI) dst_cur[b * NSTAT + f] = sred[f];
    if (dst_prev) dst_prev[b * NSTAT + S_RPRI] = sred[S_RPRI] + box_res_prev;
  }
  RIC_TS();
#ifdef CA_RIC_PROFILE
  if (tid == 0 && b == 0)
    printf("ric_scan cycles: loads+sums %lld assemble %lld elements %lld scan %lld gains %lld forward %lld "
           "stages+stats %lld\n", tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5],
           tp[7] - tp[6]);
#endif
#undef RIC_TS
}

}  // namespace ca
