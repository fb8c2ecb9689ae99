// ca_api.cu -- C ABI (include/ca.h) and host orchestration of the sm_100a kernels.
// Every step of the method runs in the kernels of ca_kernels.cuh; this file only
// validates input, lays data out in HBM, launches, and copies results back.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ca.h"
#define CA_COMMON_KERNELS 1
#ifndef CA_SWEEP_POOL
#define CA_SWEEP_POOL 800  // pairs per sweep sort pool (whole timesteps of one scene)
#endif
#ifndef CA_SWEEP_POOL_MIN_ITEMS
#define CA_SWEEP_POOL_MIN_ITEMS 10000  // ~4 waves of resident warps on 148 SMs
#endif
#include "ca_kernels.cuh"
#include "ca_riccati_scan.cuh"
#include "ca_sweep.cuh"

// the pair-sweep instantiations live in ca_sweep_d2.cu / ca_sweep_d3.cu
#define CA_EXTERN_SWEEP(D, NM, F) extern template cudaError_t ca::sweep_launch<D, NM, F>(const ca::Dev&, unsigned, cudaStream_t);
CA_SWEEP_NMAX_LIST(CA_EXTERN_SWEEP, 2, false)
CA_SWEEP_NMAX_LIST(CA_EXTERN_SWEEP, 2, true)
CA_SWEEP_NMAX_LIST(CA_EXTERN_SWEEP, 3, false)
CA_SWEEP_NMAX_LIST(CA_EXTERN_SWEEP, 3, true)

namespace {

thread_local std::string g_err;

ca_status fail(ca_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define NCCL_TRY(expr)                                                                        \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) return fail(CA_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(CA_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    }                                                                                         \
  } while (0)

constexpr int NMAX_SET[] = {9, 11, 13, 15, 20, 32};

}  // namespace

constexpr int NST = ca::NSTAT;  // per-scene statistics per slot (ca::S_* order)
constexpr int NFAM = 6;          // timing families: sweep, primal, multiplier, scale, other, comm

struct ca_problem {
  int device = 0;
  cudaStream_t stream = nullptr;
  ca::Dev dev{};
  int d = 0, B = 0, N = 0, ns = 0, nu = 0, np = 0, M = 0, nmax = 0, nmax_t = 0, rows_max = 0;
  long long P = 0;
  int M_full = 0;  // obstacles per scene of the FULL problem (default Eq. 18 thresholds)
  std::vector<int> obs_counts;  // per obstacle row counts (shape check on load)
  std::vector<int> part_off;
  std::vector<void*> allocs;
  double* alpha = nullptr;
  double* slots = nullptr;
  int slots_cap = 0;
  double* scene_res = nullptr;  // [B][NST] statistics of the last step (ca::S_* order)
  double* hist_dev = nullptr;
  int hist_cap = 0;
  double eps_pri = 0, eps_dual = 0;
  int max_iters = 100;
  bool timing = false;
  double ms[NFAM] = {0, 0, 0, 0, 0, 0};
  long long launches[NFAM] = {0, 0, 0, 0, 0, 0};
  double* s_start = nullptr;  // initial state trajectory (reset point)
  struct Pending {
    int fam, iter;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  int cur_iter = -1;  // iteration index of the launches being enqueued (timing per iteration)
  std::vector<cudaEvent_t> event_pool;
  bool sticky = false;
  long long bytes = 0;
  // multi-GPU (include/ca.h ca_dist_desc): a scene_shards x obstacle_shards grid.
  // comm = the obstacle group of this rank (ranks holding the same scenes; NULL when
  // obstacle_shards == 1), comm_all = every rank (NULL when scene_shards == 1: comm is
  // then the world).  j0/j1: obstacle block; b0: first global scene; B_total: all scenes.
  ncclComm_t comm = nullptr, comm_all = nullptr;
  int world = 1, rank = 0, j0 = 0, j1 = 0, n_obs_full = 0;
  int Ws = 1, Wo = 1, rs = 0, ro = 0, b0 = 0, B_total = 0;
  // the per-iteration scene-statistics exchange is on (scene_shards > 1; at world 1 only with
  // CA_FORCE_SCENE_GRID=1, which runs the scene-sharded code path on one rank for testing)
  bool scene_xchg = false;
  double* glob = nullptr;  // scene-sharded: [slots_cap][B_total][NST] allreduced statistics
  double* pmx = nullptr;   // [max(B*N, B)] S_PMAX column for the max-allreduce
  // ca_admm_solve (Eq. 18 per scene)
  uint8_t* active = nullptr;
  int* s_iters = nullptr;
  int* d_remaining = nullptr;
  double* s_fin = nullptr;    // [B][NST] statistics of each scene's last iteration
  double* states_buf = nullptr;  // ca_scale_detect(states != NULL) staging
  bool dist_mode = false;        // created by ca_problem_create_dist
  bool solved = false;           // ca_admm_solve has run (ca_get_solve_scenes)
  double* obs_step_buf = nullptr;  // moving obstacles (allocated on first use)
  double* sense_half = nullptr;    // [3] sensing box half-extents (NEXT f3)
  // caller-provided device workspace (bump allocation, 256-B aligned); count_only:
  // ca_workspace_size's planning pass (no device calls)
  char* ws = nullptr;
  size_t ws_size = 0, ws_used = 0;
  bool count_only = false;
  // CUDA graph of one ca_admm_iterate(g_iters) call (single GPU, timing off)
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;  // private stream to capture on (the handle's may be legacy)
  int g_iters = 0;
  long long g_launches[NFAM] = {0, 0, 0, 0, 0, 0};
  bool use_graphs = std::getenv("CA_NO_GRAPHS") == nullptr;  // diagnostics: CA_NO_GRAPHS=1 disables
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    g_iters = 0;
  }
  double* rb = nullptr;    // [B*N][rec] reduced records (allreduced)
  size_t agg_n = 0;        // doubles of dev.agg
  double* tmpB = nullptr;  // [B][NST]

  ~ca_problem() {
    drop_graph();
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (comm && comm != comm_all) ncclCommDestroy(comm);
    if (comm_all) ncclCommDestroy(comm_all);
    for (void* p : allocs) cudaFree(p);
    for (auto& e : event_pool) cudaEventDestroy(e);
    for (auto& pe : pending) {
      cudaEventDestroy(pe.a);
      cudaEventDestroy(pe.b);
    }
  }
  template <class T>
  ca_status alloc(T** p, size_t count) {
    void* q = nullptr;
    size_t nb = std::max<size_t>(count, 1) * sizeof(T);
    const size_t na = (nb + 255) & ~size_t(255);
    if (count_only) {  // ca_workspace_size: plan only
      ws_used += na;
      *p = reinterpret_cast<T*>(uintptr_t(256));
      return CA_OK;
    }
    if (ws && ws_used + na <= ws_size) {  // the caller's workspace (e.g. a torch tensor)
      *p = reinterpret_cast<T*>(ws + ws_used);
      ws_used += na;
      bytes += (long long)na;
      return CA_OK;
    }
    cudaError_t e = cudaMalloc(&q, nb);
    if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? CA_E_OOM : CA_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    allocs.push_back(q);
    bytes += (long long)nb;
    *p = static_cast<T*>(q);
    return CA_OK;
  }
  cudaEvent_t ev() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {

// ------------------------------ validation --------------------------------
bool spd(const double* Q, int n) {
  std::vector<double> L(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s = Q[j * n + j];
    for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
    if (!(s > 0.0)) return false;
    L[j * n + j] = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double a = Q[i * n + j];
      for (int k = 0; k < j; ++k) a -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = a / L[j * n + j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (std::fabs(Q[i * n + j] - Q[j * n + i]) > 1e-12 * (1 + std::fabs(Q[i * n + j]))) return false;
  return true;
}

bool riccati_supported(int ns, int nu) {
  return (ns == 4 && nu == 2) || (ns == 7 && nu == 4) || (ns == 2 && nu == 1) || (ns == 4 && nu == 1) ||
         (ns == 6 && nu == 3) || (ns == 3 && nu == 2) || (ns == 4 && nu == 3) || (ns == 6 && nu == 2);
}

ca_status validate(const ca_problem_desc* D) {
  if (!D) return fail(CA_E_INVALID, "desc is NULL");
  if (D->dim != 2 && D->dim != 3) return fail(CA_E_DIM, "dim must be 2 or 3");
  if (D->n_scenes <= 0 || D->horizon <= 0 || D->n_state <= 0 || D->n_ctrl <= 0 || D->n_parts <= 0 ||
      D->n_obs < 0)
    return fail(CA_E_INVALID, "non-positive size");
  if (!D->part_off || !D->part_A || !D->part_b || !D->Qs || !D->Qu || !D->s0 || !D->s_ref)
    return fail(CA_E_INVALID, "NULL input array");
  if (D->dyn_model == 0 && (!D->dyn_A || !D->dyn_B || !D->dyn_c)) return fail(CA_E_INVALID, "NULL dynamics array");
  if (D->dyn_model != 0 && D->dyn_model != 1) return fail(CA_E_UNSUPPORTED, "unknown dyn_model");
  if (D->dyn_model == 1 &&
      (D->n_state != 4 || D->n_ctrl != 2 || D->pose_model != CA_POSE_SE2 || D->pose_idx[0] != 0 ||
       D->pose_idx[1] != 1 || D->pose_idx[2] != 2 || !(D->dt > 0.0)))
    return fail(CA_E_INVALID, "dyn_model 1 (unicycle): n_state 4, n_ctrl 2, SE2 pose (0, 1, 2), dt > 0");
  if (D->n_obs > 0 && (!D->obs_off || !D->obs_C || !D->obs_d)) return fail(CA_E_INVALID, "NULL obstacle array");
  if (!(D->sigma > 0.0)) return fail(CA_E_INVALID, "sigma must be > 0");
  if (!(D->prox_eps >= 0.0 && std::isfinite(D->prox_eps))) return fail(CA_E_INVALID, "prox_eps must be finite and >= 0");
  if (D->prox_solver != 0 && D->prox_solver != 1) return fail(CA_E_INVALID, "prox_solver must be 0 (dual Newton) or 1 (dense Lemke)");
  const int d = D->dim;
  const int pm = D->pose_model;
  if (pm < 0 || pm > 2) return fail(CA_E_UNSUPPORTED, "unknown pose model");
  if ((pm == CA_POSE_SE2 && d != 2) || (pm == CA_POSE_TRANS_YAW && d != 3))
    return fail(CA_E_DIM, "pose model does not match dim");
  const int npc = (pm == CA_POSE_TRANSLATION) ? d : d + 1;
  for (int a = 0; a < npc; ++a)
    if (D->pose_idx[a] < 0 || D->pose_idx[a] >= D->n_state) return fail(CA_E_DIM, "pose index out of range");
  if (!riccati_supported(D->n_state, D->n_ctrl))
    return fail(CA_E_UNSUPPORTED, "(n_state, n_ctrl) combination not instantiated");
  if (ca::riccati_k_smem_doubles(D->horizon, D->n_state, D->n_ctrl, D->dyn_per_time != 0) * 8 > 227 * 1024)
    return fail(CA_E_UNSUPPORTED, "horizon too long for the shared-memory Riccati step");
  if (D->n_parts > ca::NPMAX) return fail(CA_E_UNSUPPORTED, "more than 8 robot parts");
  if ((long long)D->n_parts * D->n_obs > 65535) return fail(CA_E_UNSUPPORTED, "more than 65535 pairs per (scene, t)");
  int nrmax = 0;
  for (int i = 0; i < D->n_parts; ++i) {
    if (D->part_off[i + 1] - D->part_off[i] > ca::NRMAX)
      return fail(CA_E_UNSUPPORTED, "robot part with more than 16 faces");
    const int r0 = D->part_off[i], nr = D->part_off[i + 1] - r0;
    if (nr < d + 1) return fail(CA_E_GEOMETRY, "robot part with fewer than d+1 faces");
    for (int k = 0; k < nr; ++k)
      {
        double bt = D->part_b[r0 + k];  // b~ = b - A o_i with a scaling centre (NEXT f3)
        if (D->part_ctr)
          for (int a = 0; a < d; ++a) bt -= D->part_A[(r0 + k) * d + a] * D->part_ctr[i * d + a];
        if (!(bt > 0.0))
          return fail(CA_E_GEOMETRY, D->part_ctr ? "robot part: its scaling centre must lie strictly inside"
                                                 : "robot part b_i must be > 0 (body origin inside)");
      }
    nrmax = std::max(nrmax, nr);
  }
  int nomax = 0;
  for (long long o = 0; o < (long long)D->n_scenes * D->n_obs; ++o) {
    const int no = D->obs_off[o + 1] - D->obs_off[o];
    if (no < d + 1) return fail(CA_E_GEOMETRY, "obstacle with fewer than d+1 faces");
    nomax = std::max(nomax, no);
  }
  if (nrmax + nomax + 1 > 32) return fail(CA_E_DIM, "n = n_r + n_o + 1 > 32");
  if (D->obs_step)
    for (long long k = 0; k < (long long)D->n_scenes * D->n_obs * d; ++k)
      if (!std::isfinite(D->obs_step[k])) return fail(CA_E_INVALID, "obs_step must be finite");
  if (!spd(D->Qs, D->n_state) || !spd(D->Qu, D->n_ctrl)) return fail(CA_E_INVALID, "Qs/Qu must be SPD");
  if (D->s_min || D->s_max || D->u_min || D->u_max) {  // NEXT f1 boxes
    bool finite = false;
    for (int pass = 0; pass < 2; ++pass) {
      const int n = pass ? D->n_ctrl : D->n_state;
      const double* lo = pass ? D->u_min : D->s_min;
      const double* hi = pass ? D->u_max : D->s_max;
      for (int a = 0; a < n; ++a) {
        const double l = lo ? lo[a] : -INFINITY, u = hi ? hi[a] : INFINITY;
        if (std::isnan(l) || std::isnan(u) || l > u || l == INFINITY || u == -INFINITY)
          return fail(CA_E_INVALID, "box bounds must satisfy min <= max (no NaN, no empty side)");
        finite = finite || std::isfinite(l) || std::isfinite(u);
      }
    }
    if (finite && !(D->box_rho > 0.0 && std::isfinite(D->box_rho)))
      return fail(CA_E_INVALID, "box_rho must be > 0 with finite bounds");
  }
  if (D->part_ctr)
    for (int k = 0; k < D->n_parts * d; ++k)
      if (!std::isfinite(D->part_ctr[k])) return fail(CA_E_INVALID, "part_ctr must be finite");
  if (D->sense_half)
    for (int a = 0; a < d; ++a)
      if (!(D->sense_half[a] > 0.0 && std::isfinite(D->sense_half[a])))
        return fail(CA_E_INVALID, "sense_half must be finite and > 0");
  return CA_OK;
}

template <class T>
ca_status h2d(ca_problem* h, T* dst, const T* src, size_t count) {
  if (count == 0) return CA_OK;
  CUDA_TRY(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, h->stream));
  return CA_OK;
}

// box block (reading #7): clip_iterate = project s (t >= 1), u into the box first
ca_status box_reset(ca_problem* h, int clip_iterate) {
  if (!h->dev.box) return CA_OK;
  const long long nq = (long long)h->B * (h->N + 1);
  ca::k_box_reset<<<(unsigned)((nq + 127) / 128), 128, 0, h->stream>>>(h->dev, clip_iterate);
  CUDA_TRY(cudaGetLastError());
  h->launches[4]++;
  return CA_OK;
}

// O1 initial iterate on the device (reading #11): s = s_start, u = 0,
// lambda = 1/sum(b_i) 1, mu = gamma = zeta = xi = 0
ca_status reset_iterate(ca_problem* h) {
  ca::Dev& v = h->dev;
  CUDA_TRY(cudaMemcpyAsync(v.s, h->s_start, sizeof(double) * (size_t)h->B * (h->N + 1) * h->ns,
                           cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaMemsetAsync(v.u, 0, sizeof(double) * (size_t)h->B * h->N * h->nu, h->stream));
  if (h->P == 0)  // no pair ever writes a record: the primal step then reads zero aggregates
    CUDA_TRY(cudaMemsetAsync(v.agg, 0, sizeof(double) * h->agg_n, h->stream));
  if (h->P > 0) {
    CUDA_TRY(cudaMemsetAsync(v.zeta, 0, sizeof(double) * (size_t)h->P, h->stream));
    CUDA_TRY(cudaMemsetAsync(v.xi, 0, sizeof(double) * (size_t)h->d * h->P, h->stream));
    CUDA_TRY(cudaMemsetAsync(v.pst, 0, sizeof(uint32_t) * (size_t)h->P, h->stream));
    const unsigned grid = (unsigned)((h->P + 255) / 256);
    ca::k_init_y<<<grid, 256, 0, h->stream>>>(h->dev);
    CUDA_TRY(cudaGetLastError());
    h->launches[4]++;
  }
  return box_reset(h, 1);
}

// upload all per-batch inputs and reset the iterate (reading #11)
ca_status upload(ca_problem* h, const ca_problem_desc* D) {
  const int d = h->d, B = h->B, N = h->N, ns = h->ns, nu = h->nu;
  ca::Dev& v = h->dev;
  // robot rows (a_0, a_1, a_2|0, b)
  const int prow = D->part_off[h->np];
  std::vector<double> pr(4 * (size_t)prow, 0.0);
  for (int r = 0; r < prow; ++r) {
    for (int a = 0; a < d; ++a) pr[4 * r + a] = D->part_A[r * d + a];
    pr[4 * r + 3] = D->part_b[r];
  }
  const long long orow = (h->M > 0) ? D->obs_off[(long long)B * h->M] : 0;
  ca_status st;
  if ((st = h2d(h, const_cast<double*>(v.part_rows), pr.data(), pr.size()))) return st;
  if ((st = h2d(h, const_cast<int*>(v.part_off), D->part_off, (size_t)h->np + 1))) return st;
  if (v.part_ctr) {  // scaling centres (NEXT f3): b~ = b - A o_i on the device
    std::vector<double> oc(3 * (size_t)h->np, 0.0);
    for (int i = 0; i < h->np; ++i)
      for (int a = 0; a < d; ++a) oc[3 * i + a] = D->part_ctr[i * d + a];
    if ((st = h2d(h, const_cast<double*>(v.part_ctr), oc.data(), oc.size()))) return st;
    ca::k_part_centre<<<1, 32, 0, h->stream>>>(v, const_cast<double*>(v.part_rows));
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(h->stream));  // oc is a stack vector
  }
  ca::k_lamtab<<<1, 32, 0, h->stream>>>(v);
  CUDA_TRY(cudaGetLastError());
  if (d == 2) {  // polygon vertices for the separating-axis scale detection
    ca::k_vertices2d<<<1, 32, 0, h->stream>>>(v.part_rows, v.part_off, h->np, v.part_vert, v.part_nv);
    CUDA_TRY(cudaGetLastError());
  }
  if (h->M > 0) {
    // obstacle rows: C and d straight from the caller's arrays into a staging area
    // (the certificate array y, rewritten by reset_iterate below), interleaved into
    // (c_0, c_1, c_2, d) rows on the device
    double* stg = h->dev.y;
    if ((st = h2d(h, stg, D->obs_C, (size_t)orow * d))) return st;
    if ((st = h2d(h, stg + (size_t)orow * d, D->obs_d, (size_t)orow))) return st;
    ca::k_pack_obs<<<(unsigned)((orow + 255) / 256), 256, 0, h->stream>>>(stg, orow, d, const_cast<double*>(v.obs_rows));
    CUDA_TRY(cudaGetLastError());
    if ((st = h2d(h, const_cast<int*>(v.obs_off), D->obs_off, (size_t)B * h->M + 1))) return st;
    if (D->obs_step) {  // moving obstacles (NEXT f3)
      if (!h->obs_step_buf && (st = h->alloc(&h->obs_step_buf, (size_t)B * h->M * d))) return st;
      if ((st = h2d(h, h->obs_step_buf, D->obs_step, (size_t)B * h->M * d))) return st;
    }
    v.obs_step = D->obs_step ? h->obs_step_buf : nullptr;
    if (d == 2) {
      const long long no = (long long)B * h->M;
      ca::k_vertices2d<<<(unsigned)((no + 127) / 128), 128, 0, h->stream>>>(v.obs_rows, v.obs_off, (int)no, v.obs_vert,
                                                                           v.obs_nv);
      CUDA_TRY(cudaGetLastError());
    }
  }
  const long long nd = (long long)(D->dyn_per_scene ? B : 1) * (D->dyn_per_time ? N : 1);
  if (!D->dyn_model) {  // dyn_model 1: written by k_relin_unicycle every primal step
    if ((st = h2d(h, const_cast<double*>(v.dynA), D->dyn_A, (size_t)nd * ns * ns))) return st;
    if ((st = h2d(h, const_cast<double*>(v.dynB), D->dyn_B, (size_t)nd * ns * nu))) return st;
    if ((st = h2d(h, const_cast<double*>(v.dync), D->dyn_c, (size_t)nd * ns))) return st;
  }
  if ((st = h2d(h, const_cast<double*>(v.Qs), D->Qs, (size_t)ns * ns))) return st;
  if ((st = h2d(h, const_cast<double*>(v.Qu), D->Qu, (size_t)nu * nu))) return st;
  if ((st = h2d(h, const_cast<double*>(v.s0), D->s0, (size_t)B * ns))) return st;
  if ((st = h2d(h, const_cast<double*>(v.sref), D->s_ref, (size_t)B * (N + 1) * ns))) return st;
  // iterate: s = s_init (default s_ref) with s_0 = s0 (set on the device); u = 0;
  // lambda = 1/sum(b) 1; rest 0
  if ((st = h2d(h, h->s_start, D->s_init ? D->s_init : D->s_ref, (size_t)B * (N + 1) * ns))) return st;
  ca::k_set_s0<<<(unsigned)((B * ns + 127) / 128), 128, 0, h->stream>>>(v, h->s_start);
  CUDA_TRY(cudaGetLastError());
  // execution order of each (b, t) group: pairs stably sorted by LCP size n so that a
  // warp's 32 threads mostly run the same-size Lemke (pure scheduling; results are
  // stored at the pair's own index p) -- one thread per scene on the device
  if (h->P > 0) {
    ca::k_gperm<<<(unsigned)((B + 63) / 64), 64, 0, h->stream>>>(v, const_cast<int*>(v.gperm));
    CUDA_TRY(cudaGetLastError());
  }
  if (v.box) {  // [s_min | s_max | u_min | u_max], +-inf where unbounded
    std::vector<double> lim(2 * (size_t)(ns + nu));
    for (int a = 0; a < ns; ++a) {
      lim[a] = D->s_min ? D->s_min[a] : -INFINITY;
      lim[ns + a] = D->s_max ? D->s_max[a] : INFINITY;
    }
    for (int a = 0; a < nu; ++a) {
      lim[2 * ns + a] = D->u_min ? D->u_min[a] : -INFINITY;
      lim[2 * ns + nu + a] = D->u_max ? D->u_max[a] : INFINITY;
    }
    v.box_rho = D->box_rho;
    if ((st = h2d(h, const_cast<double*>(v.box_lim), lim.data(), lim.size()))) return st;
    CUDA_TRY(cudaStreamSynchronize(h->stream));  // lim is a stack vector
  }
  if (v.sensed) {  // which obstacles enter the pair table (NEXT f3)
    if ((st = h2d(h, h->sense_half, D->sense_half, (size_t)d))) return st;
    const long long no = (long long)B * h->M;
    if (d == 2) ca::k_sense<2><<<(unsigned)((no + 127) / 128), 128, 0, h->stream>>>(v, h->sense_half, const_cast<uint8_t*>(v.sensed));
    else ca::k_sense<3><<<(unsigned)((no + 127) / 128), 128, 0, h->stream>>>(v, h->sense_half, const_cast<uint8_t*>(v.sensed));
    CUDA_TRY(cudaGetLastError());
    h->launches[4]++;
  }
  if ((st = reset_iterate(h))) return st;
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

// ------------------------------ launches -----------------------------------
void t_begin(ca_problem* h, cudaEvent_t* e) {
  if (h->timing) {
    *e = h->ev();
    cudaEventRecord(*e, h->stream);
  }
}
void t_end(ca_problem* h, int fam, cudaEvent_t e0) {
  h->launches[fam]++;
  if (h->timing) {
    cudaEvent_t e1 = h->ev();
    cudaEventRecord(e1, h->stream);
    h->pending.push_back({fam, h->cur_iter, e0, e1});
  }
}
// Accumulate the recorded launch times into h->ms; with per_iter (HOST [n_iter][NFAM])
// also per iteration of the enqueue that recorded them.
ca_status flush_timing(ca_problem* h, double* per_iter = nullptr, int n_iter = 0) {
  for (auto& pe : h->pending) {
    float ms = 0.f;
    CUDA_TRY(cudaEventSynchronize(pe.b));
    CUDA_TRY(cudaEventElapsedTime(&ms, pe.a, pe.b));
    h->ms[pe.fam] += ms;
    if (per_iter && pe.iter >= 0 && pe.iter < n_iter) per_iter[pe.iter * NFAM + pe.fam] += ms;
    h->event_pool.push_back(pe.a);
    h->event_pool.push_back(pe.b);
  }
  h->pending.clear();
  return CA_OK;
}

int nmax_template(int nmax) {
  for (int v : NMAX_SET)
    if (nmax <= v) return v;
  return 32;
}

template <int D, int NM, bool F>
ca_status launch_sweep_t(ca_problem* h) {
  const long long grid = (long long)h->dev.nitems;
  CUDA_TRY((ca::sweep_launch<D, NM, F>(h->dev, (unsigned)grid, h->stream)));
  return CA_OK;
}

template <int D, bool F>
ca_status launch_sweep_d(ca_problem* h) {
  switch (h->nmax_t) {
    case 9: return launch_sweep_t<D, 9, F>(h);
    case 11: return launch_sweep_t<D, 11, F>(h);
    case 13: return launch_sweep_t<D, 13, F>(h);
    case 15: return launch_sweep_t<D, 15, F>(h);
    case 20: return launch_sweep_t<D, 20, F>(h);
    default: return launch_sweep_t<D, 32, F>(h);
  }
}

ca_status launch_sweep(ca_problem* h, bool fused) {
  if (h->P == 0) return CA_OK;
  // each warp stages its group's status words and the n-order when they fit (48 KB per CTA)
  // -- on large batches, where the scattered 4-byte reads bound the kernel (C5: 338 -> 274
  // us per launch); a one-wave batch keeps the shorter unstaged chain (same output bits)
  const size_t sort_sm = sizeof(uint32_t) * ca::SORT_WPC * ((size_t)h->dev.GG + h->dev.G);
  const int sort_staged = (sort_sm <= 48 * 1024 && (long long)h->B * h->dev.NG >= 1024) ? 1 : 0;
  ca::k_sortpairs<<<(unsigned)(((long long)h->B * h->dev.NG + ca::SORT_WPC - 1) / ca::SORT_WPC), 32 * ca::SORT_WPC,
                     sort_staged ? sort_sm : 0, h->stream>>>(h->dev, sort_staged);
  CUDA_TRY(cudaGetLastError());
  h->launches[4]++;
  cudaEvent_t e0 = nullptr;
  t_begin(h, &e0);
  ca_status st;
  if (h->d == 2) st = fused ? launch_sweep_d<2, true>(h) : launch_sweep_d<2, false>(h);
  else st = fused ? launch_sweep_d<3, true>(h) : launch_sweep_d<3, false>(h);
  t_end(h, 0, e0);
  return st;
}

// Scenes per batch above which the thread-per-scene Riccati (throughput) beats the
// warp-per-scene one (latency): the warp version runs ~1 scene-recursion per resident
// CTA at a time, the thread version 32 per warp.
constexpr int RIC_THREAD_MIN_B = 1024;

template <int NS, int NU>
ca_status launch_riccati_t(ca_problem* h, const double* recs, int nchunk, double* cur, double* prev) {
  static const int thread_min_b =
      std::getenv("CA_RIC_THREAD_MIN_B") ? std::atoi(std::getenv("CA_RIC_THREAD_MIN_B")) : RIC_THREAD_MIN_B;
  if (h->B > thread_min_b) {
    const long long nq = (long long)h->B * h->N;
    if (nchunk) {
      const long long nbg = (long long)h->B * h->dev.NG;
      ca::k_stage_grouped<<<(unsigned)((nbg + 3) / 4), 128, 0, h->stream>>>(h->dev);
    } else {
      ca::k_stage<<<(unsigned)((nq + 127) / 128), 128, 0, h->stream>>>(h->dev, recs, nchunk);
    }
    CUDA_TRY(cudaGetLastError());
    ca::k_riccati_thread<NS, NU><<<(h->B + 63) / 64, 64, 0, h->stream>>>(h->dev, cur, prev);
    CUDA_TRY(cudaGetLastError());
    h->launches[1]++;
    return CA_OK;
  }
  // parallel-in-time LQ (ca_riccati_scan.cuh): log2(N+1) combination levels instead of N
  // dependent Riccati steps on one warp; n_s <= 4 (the element combination keeps its
  // matrices in registers), CA_RICCATI_SCAN=0 selects the serial recursion
  if constexpr (NS <= 4) {
    const size_t sms = sizeof(double) * (size_t)ca::riccati_scan_smem_doubles(h->N, NS, NU, h->dev.dyn_pt != 0);
    static const bool scan_on = !(std::getenv("CA_RICCATI_SCAN") && std::getenv("CA_RICCATI_SCAN")[0] == '0');
    // shortest horizon taking the scan (C1, N = 10: 35.8 vs 36.3 us per iteration serial)
    static const int scan_min_n = std::getenv("CA_RICCATI_SCAN_MIN_N") ? std::atoi(std::getenv("CA_RICCATI_SCAN_MIN_N")) : 8;
    if (scan_on && sms <= 200 * 1024 && ca::SCAN_GS * (h->N + 1) <= 1024 && h->N >= scan_min_n) {
      int tmax = 0;
      {
        static std::mutex mu;
        static size_t configured[CA_MAX_DEVICES] = {};
        // one group of SCAN_GS threads per stage, capped by what the kernel's register
        // count allows in one CTA (the kernel strides over the stages when fewer)
        static int max_threads[CA_MAX_DEVICES] = {};
        if (h->device >= CA_MAX_DEVICES) return fail(CA_E_CUDA, "device ordinal too large");
        std::lock_guard<std::mutex> lk(mu);
        if (sms > configured[h->device]) {
          if (sms > 48 * 1024)
            CUDA_TRY(cudaFuncSetAttribute(ca::k_riccati_scan<NS, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sms));
          // the same L1 / shared split as the sweep: no SM reconfiguration between the two
          // kernels of an iteration (C4 primal step 25.9 -> 24.2 us)
          CUDA_TRY(cudaFuncSetAttribute(ca::k_riccati_scan<NS, NU>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
          configured[h->device] = sms;
        }
        if (!max_threads[h->device]) {
          cudaFuncAttributes fa;
          CUDA_TRY(cudaFuncGetAttributes(&fa, ca::k_riccati_scan<NS, NU>));
          max_threads[h->device] = fa.maxThreadsPerBlock & ~31;
        }
        tmax = max_threads[h->device];
      }
      const int threads = std::min(tmax, 32 * ((ca::SCAN_GS * (h->N + 1) + 31) / 32));
      ca::k_riccati_scan<NS, NU><<<(unsigned)h->B, threads, sms, h->stream>>>(h->dev, recs, nchunk, cur, prev);
      CUDA_TRY(cudaGetLastError());
      return CA_OK;
    }
  }
  const size_t sm = sizeof(double) * (size_t)ca::riccati_k_smem_doubles(h->N, NS, NU, h->dev.dyn_pt != 0);
  if (sm > 48 * 1024) {  // the attribute is per device: cached per device ordinal under a lock
    static std::mutex mu;
    static size_t configured[CA_MAX_DEVICES] = {};
    if (h->device >= CA_MAX_DEVICES) return fail(CA_E_CUDA, "device ordinal too large");
    std::lock_guard<std::mutex> lk(mu);
    if (sm > configured[h->device]) {
      CUDA_TRY(cudaFuncSetAttribute(ca::k_riccati<NS, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      CUDA_TRY(cudaFuncSetAttribute(ca::k_riccati<NS, NU>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      configured[h->device] = sm;
    }
  }
  ca::k_riccati<NS, NU><<<(unsigned)h->B, 32 * ca::RIC_WARPS, sm, h->stream>>>(h->dev, recs, nchunk, cur, prev);
  CUDA_TRY(cudaGetLastError());
  return CA_OK;
}

ca_status launch_riccati(ca_problem* h, double* cur, double* prev, const double* given_recs = nullptr) {
  cudaEvent_t e0 = nullptr;
  t_begin(h, &e0);
  ca_status st;
  if (h->dev.dyn_model == 1) {  // SQP step: linearise the unicycle at the current iterate
    const long long nq = (long long)h->B * h->N;
    ca::k_relin_unicycle<<<(unsigned)((nq + 127) / 128), 128, 0, h->stream>>>(h->dev);
    CUDA_TRY(cudaGetLastError());
    h->launches[1]++;
  }
  const double* recs = h->dev.agg;
  int nchunk = h->dev.nchunkG;
  if (given_recs) {  // ca_primal_step_records: one record per (scene, t) given
    recs = given_recs;
    nchunk = 0;
  } else if (h->comm) {
    // a5: one allreduce of the per-(scene, t) aggregates + residual partials (the S_PMAX
    // column max-reduced in the same NCCL group: one fused collective)
    const long long nq = (long long)h->B * h->N;
    const unsigned gq = (unsigned)((nq + 127) / 128);
    ca::k_reduce_records<<<gq, 128, 0, h->stream>>>(h->dev, h->rb, h->pmx);
    CUDA_TRY(cudaGetLastError());
    h->launches[1]++;
    cudaEvent_t c0 = nullptr;
    t_begin(h, &c0);
    NCCL_TRY(ncclGroupStart());
    NCCL_TRY(ncclAllReduce(h->rb, h->rb, (size_t)nq * h->dev.rec, ncclDouble, ncclSum, h->comm, h->stream));
    NCCL_TRY(ncclAllReduce(h->pmx, h->pmx, (size_t)nq, ncclDouble, ncclMax, h->comm, h->stream));
    NCCL_TRY(ncclGroupEnd());
    t_end(h, 5, c0);
    ca::k_pmax_back<<<gq, 128, 0, h->stream>>>(h->dev, h->rb, h->pmx);
    CUDA_TRY(cudaGetLastError());
    h->launches[1]++;
    recs = h->rb;
    nchunk = 0;  // one reduced record per (scene, t)
  }
  const int ns = h->ns, nu = h->nu;
  if (ns == 4 && nu == 2) st = launch_riccati_t<4, 2>(h, recs, nchunk, cur, prev);
  else if (ns == 7 && nu == 4) st = launch_riccati_t<7, 4>(h, recs, nchunk, cur, prev);
  else if (ns == 2 && nu == 1) st = launch_riccati_t<2, 1>(h, recs, nchunk, cur, prev);
  else if (ns == 4 && nu == 1) st = launch_riccati_t<4, 1>(h, recs, nchunk, cur, prev);
  else if (ns == 6 && nu == 3) st = launch_riccati_t<6, 3>(h, recs, nchunk, cur, prev);
  else if (ns == 3 && nu == 2) st = launch_riccati_t<3, 2>(h, recs, nchunk, cur, prev);
  else if (ns == 4 && nu == 3) st = launch_riccati_t<4, 3>(h, recs, nchunk, cur, prev);
  else st = launch_riccati_t<6, 2>(h, recs, nchunk, cur, prev);
  t_end(h, 1, e0);
  return st;
}

ca_status launch_mult(ca_problem* h) {
  if (h->P == 0) return CA_OK;
  cudaEvent_t e0 = nullptr;
  t_begin(h, &e0);
  const long long grid = (long long)h->dev.nitems;
  if (h->d == 2) ca::k_mult<2><<<(unsigned)grid, ca::CTA, 0, h->stream>>>(h->dev);
  else ca::k_mult<3><<<(unsigned)grid, ca::CTA, 0, h->stream>>>(h->dev);
  CUDA_TRY(cudaGetLastError());
  t_end(h, 2, e0);
  return CA_OK;
}

ca_status launch_collect(ca_problem* h, double* dst, int mask) {
  if (h->P == 0) {
    CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(double) * NST * h->B, h->stream));
    return CA_OK;
  }
  // the box residual joins r_pri once (rank 0 of an obstacle-sharded run)
  const int add_box = ((mask & 2) && (!h->comm || h->rank == 0)) ? 1 : 0;
  ca::k_collect<<<(h->B + 3) / 4, 128, 0, h->stream>>>(h->dev, dst, mask, add_box);
  CUDA_TRY(cudaGetLastError());
  h->launches[4]++;
  return CA_OK;
}

// [n][NST] statistics summed over the ranks of `comm` (S_PMAX: max), one NCCL group
ca_status allreduce_stats(ca_problem* h, double* buf, int n, ncclComm_t comm) {
  const unsigned g = (unsigned)((n + 127) / 128);
  ca::k_stat_split<<<g, 128, 0, h->stream>>>(buf, h->pmx, n);
  CUDA_TRY(cudaGetLastError());
  cudaEvent_t c0 = nullptr;
  t_begin(h, &c0);
  NCCL_TRY(ncclGroupStart());
  NCCL_TRY(ncclAllReduce(buf, buf, (size_t)n * NST, ncclDouble, ncclSum, comm, h->stream));
  NCCL_TRY(ncclAllReduce(h->pmx, h->pmx, (size_t)n, ncclDouble, ncclMax, comm, h->stream));
  NCCL_TRY(ncclGroupEnd());
  t_end(h, 5, c0);
  ca::k_stat_join<<<g, 128, 0, h->stream>>>(buf, h->pmx, n);
  CUDA_TRY(cudaGetLastError());
  h->launches[4] += 2;
  return CA_OK;
}

// per-scene statistics of the local pairs -> fields `mask` of dst; in obstacle-sharded
// runs combined over the obstacle group (one small allreduce).  Other fields are left
// untouched.
ca_status collect_global(ca_problem* h, double* dst, int mask) {
  if (!h->comm) return launch_collect(h, dst, mask);
  CUDA_TRY(cudaMemsetAsync(h->tmpB, 0, sizeof(double) * NST * h->B, h->stream));
  ca_status st = launch_collect(h, h->tmpB, mask);
  if (st) return st;
  if ((st = allreduce_stats(h, h->tmpB, h->B, h->comm))) return st;
  for (int f = 0; f < NST; ++f)
    if ((mask >> f) & 1)
      CUDA_TRY(cudaMemcpy2DAsync(dst + f, NST * sizeof(double), h->tmpB + f, NST * sizeof(double), sizeof(double),
                                 h->B, cudaMemcpyDeviceToDevice, h->stream));
  return CA_OK;
}

// scene-sharded runs (a5 of the scene grid): the completed per-scene statistics of one
// iteration (slot, [B][NST]) into the global table glob_k ([B_total][NST]) and one
// ncclAllReduce over every rank -- the global Eq. 18 residuals of every scene on every
// rank (the stop decision of ca_admm_solve, the global history of ca_admm_iterate).
ca_status scene_exchange(ca_problem* h, const double* slot, double* glob_k) {
  if (!h->comm_all) return CA_OK;
  const int n = h->B * NST;
  ca::k_scatter_slot<<<(unsigned)((n + 127) / 128), 128, 0, h->stream>>>(glob_k, slot, h->B, h->b0, h->ro == 0);
  CUDA_TRY(cudaGetLastError());
  h->launches[4]++;
  cudaEvent_t c0 = nullptr;
  t_begin(h, &c0);
  NCCL_TRY(ncclAllReduce(glob_k, glob_k, (size_t)h->B_total * NST, ncclDouble, ncclSum, h->comm_all, h->stream));
  t_end(h, 5, c0);
  return CA_OK;
}

// The rank-local view of the full problem: scenes [b0, b1), obstacles [j0, j1) of each
// (pure data movement; the caller's arrays are only read).
struct LocalObs {
  std::vector<int> off;
  std::vector<double> C, d, step, s0, sref, sinit, dA, dB, dc;
};
void slice_problem(const ca_problem_desc* D, int b0, int b1, int j0, int j1, LocalObs& L, ca_problem_desc& out) {
  const int M = D->n_obs, dim = D->dim, Ml = j1 - j0, ns = D->n_state, nu = D->n_ctrl, N = D->horizon;
  L = LocalObs{};
  L.off.assign(1, 0);
  for (int b = b0; b < b1; ++b)
    for (int j = j0; j < j1; ++j) {
      if (D->obs_step)
        for (int a = 0; a < dim; ++a) L.step.push_back(D->obs_step[((long long)b * M + j) * dim + a]);
      const int lo = D->obs_off[(long long)b * M + j], hi = D->obs_off[(long long)b * M + j + 1];
      for (int r = lo; r < hi; ++r) {
        for (int a = 0; a < dim; ++a) L.C.push_back(D->obs_C[(long long)r * dim + a]);
        L.d.push_back(D->obs_d[r]);
      }
      L.off.push_back(L.off.back() + (hi - lo));
    }
  out = *D;
  out.n_obs = Ml;
  out.obs_off = L.off.data();
  out.obs_C = L.C.empty() ? nullptr : L.C.data();
  out.obs_d = L.d.empty() ? nullptr : L.d.data();
  out.obs_step = (D->obs_step && !L.step.empty()) ? L.step.data() : nullptr;
  if (b0 == 0 && b1 == D->n_scenes) return;
  // scene slice of the per-scene arrays
  out.n_scenes = b1 - b0;
  L.s0.assign(D->s0 + (long long)b0 * ns, D->s0 + (long long)b1 * ns);
  L.sref.assign(D->s_ref + (long long)b0 * (N + 1) * ns, D->s_ref + (long long)b1 * (N + 1) * ns);
  out.s0 = L.s0.data();
  out.s_ref = L.sref.data();
  if (D->s_init) {
    L.sinit.assign(D->s_init + (long long)b0 * (N + 1) * ns, D->s_init + (long long)b1 * (N + 1) * ns);
    out.s_init = L.sinit.data();
  }
  if (D->dyn_per_scene && D->dyn_model == 0) {
    const long long nt = D->dyn_per_time ? N : 1;
    L.dA.assign(D->dyn_A + b0 * nt * ns * ns, D->dyn_A + b1 * nt * ns * ns);
    L.dB.assign(D->dyn_B + b0 * nt * ns * nu, D->dyn_B + b1 * nt * ns * nu);
    L.dc.assign(D->dyn_c + b0 * nt * ns, D->dyn_c + b1 * nt * ns);
    out.dyn_A = L.dA.data();
    out.dyn_B = L.dB.data();
    out.dyn_c = L.dc.data();
  }
}

// The grid position of dist->rank (include/ca.h ca_dist_desc) and its local problem.
struct GridPos {
  int world = 1, rank = 0, Ws = 1, Wo = 1, rs = 0, ro = 0, b0 = 0, b1 = 0, j0 = 0, j1 = 0, B_total = 0, M_full = 0;
};
ca_status grid_position(const ca_problem_desc* D, const ca_dist_desc* dist, GridPos& g, LocalObs& L,
                        ca_problem_desc& Dl) {
  if (!dist->nccl_id || dist->world_size < 1 || dist->rank < 0 || dist->rank >= dist->world_size)
    return fail(CA_E_INVALID, "bad ca_dist_desc");
  g.world = dist->world_size;
  g.rank = dist->rank;
  int Ws = dist->scene_shards, Wo = dist->obstacle_shards;
  if (Ws <= 0 && Wo <= 0) {
    Ws = 1;
    Wo = g.world;
  } else if (Ws <= 0) {
    Ws = g.world / std::max(1, Wo);
  } else if (Wo <= 0) {
    Wo = g.world / std::max(1, Ws);
  }
  if (Ws * Wo != g.world) return fail(CA_E_INVALID, "scene_shards * obstacle_shards != world_size");
  if (Ws > D->n_scenes) return fail(CA_E_INVALID, "more scene shards than scenes");
  g.Ws = Ws;
  g.Wo = Wo;
  g.rs = g.rank / Wo;
  g.ro = g.rank % Wo;
  g.B_total = D->n_scenes;
  g.M_full = D->n_obs;
  g.b0 = (int)((long long)D->n_scenes * g.rs / Ws);
  g.b1 = (int)((long long)D->n_scenes * (g.rs + 1) / Ws);
  // the obstacle partition of this scene shard (balanced by its face counts)
  ca_status st;
  if ((st = ca_obstacle_partition(g.b1 - g.b0, D->n_obs, D->n_obs > 0 ? D->obs_off + (long long)g.b0 * D->n_obs : nullptr,
                                  Wo, g.ro, &g.j0, &g.j1)))
    return st;
  slice_problem(D, g.b0, g.b1, g.j0, g.j1, L, Dl);
  return CA_OK;
}

ca_status ensure_slots(ca_problem* h, int n) {
  if (n <= h->slots_cap) return CA_OK;
  ca_status st;
  if ((st = h->alloc(&h->slots, (size_t)n * h->B * NST))) return st;
  if ((st = h->alloc(&h->hist_dev, (size_t)n * NST))) return st;
  if (h->scene_xchg && (st = h->alloc(&h->glob, (size_t)n * h->B_total * NST))) return st;
  h->slots_cap = n;
  return CA_OK;
}

// combined statistics [NST] (ca::S_* order) -> ca_residuals
void fill_res(const double* c, long long n_pairs, ca_residuals* r) {
  *r = ca_residuals{};
  r->r_dual = c[ca::S_RDUAL];
  r->r_pri = c[ca::S_RPRI];
  r->pivots = (int64_t)c[ca::S_PIV];
  r->n_fail = (int64_t)c[ca::S_FAIL];
  r->n_ray = (int64_t)c[ca::S_RAY];
  r->n_iterlimit = (int64_t)c[ca::S_ITER];
  r->n_neg_ye = (int64_t)c[ca::S_NEGYE];
  r->max_pivots = (int32_t)c[ca::S_PMAX];
  r->n_pairs = n_pairs;
}

// per-scene statistics [nb][NST] on the device -> their combination over scenes (sum;
// max for S_PMAX), in scene order
ca_status sums(ca_problem* h, const double* dst_dev, ca_residuals* out, int nb = -1) {
  if (nb < 0) nb = h->B;
  std::vector<double> v((size_t)nb * NST);
  CUDA_TRY(cudaMemcpyAsync(v.data(), dst_dev, sizeof(double) * v.size(), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  double c[NST] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = 0; b < nb; ++b)
    for (int f = 0; f < NST; ++f) c[f] = ca::stat_comb(f, c[f], v[(size_t)b * NST + f]);
  ca_residuals r;
  fill_res(c, h->P, &r);
  if (out) *out = r;
  return CA_OK;
}

// the timed device milliseconds (families of flush_timing) into a ca_residuals
void fill_ms(const double* fam_ms, ca_residuals* r) {
  r->ms_sweep = (float)fam_ms[0];
  r->ms_riccati = (float)fam_ms[1];
  r->ms_mult = (float)fam_ms[2];
  r->ms_comm = (float)fam_ms[5];
}

ca_status check_handle(ca_problem* h) {
  if (!h) return fail(CA_E_INVALID, "NULL handle");
  if (h->sticky) return fail(CA_E_CUDA, "handle unusable after an earlier CUDA error");
  if (cudaSetDevice(h->device) != cudaSuccess) return fail(CA_E_CUDA, "cudaSetDevice failed");
  return CA_OK;
}

ca_status mark(ca_problem* h, ca_status st) {
  if (st == CA_E_CUDA) h->sticky = true;
  return st;
}

}  // namespace

extern "C" {

const char* ca_last_error(void) { return g_err.c_str(); }

// the grid position of a sharded handle (NULL: single GPU)
void set_grid(ca_problem* h, const GridPos* g) {
  if (!g) return;
  h->dist_mode = true;
  h->world = g->world;
  h->rank = g->rank;
  h->Ws = g->Ws;
  h->Wo = g->Wo;
  h->rs = g->rs;
  h->ro = g->ro;
  h->b0 = g->b0;
  h->B_total = g->B_total;
  h->j0 = g->j0;
  h->j1 = g->j1;
  h->n_obs_full = g->M_full;
  h->M_full = g->M_full;
  const char* fg = std::getenv("CA_FORCE_SCENE_GRID");
  h->scene_xchg = g->Ws > 1 || (g->world == 1 && fg && fg[0] == '1');
}

// Host-side setup of a handle: shapes, work decomposition and every device buffer
// (through h->alloc, so a planning pass can size the caller's workspace).
ca_status setup_handle(ca_problem* h, const ca_problem_desc* D) {
  h->d = D->dim;
  h->B = D->n_scenes;
  h->N = D->horizon;
  h->ns = D->n_state;
  h->nu = D->n_ctrl;
  h->np = D->n_parts;
  h->M = D->n_obs;
  h->part_off.assign(D->part_off, D->part_off + h->np + 1);
  int nrmax = 0, nomax = 0;
  for (int i = 0; i < h->np; ++i) nrmax = std::max(nrmax, D->part_off[i + 1] - D->part_off[i]);
  h->obs_counts.resize((size_t)h->B * h->M);
  for (long long o = 0; o < (long long)h->B * h->M; ++o) {
    h->obs_counts[o] = D->obs_off[o + 1] - D->obs_off[o];
    nomax = std::max(nomax, h->obs_counts[o]);
  }
  h->nmax = (h->M > 0) ? nrmax + nomax + 1 : 1;
  h->dev.nrmax = nrmax;
  h->dev.nomax = nomax;
  h->nmax_t = nmax_template(h->nmax);
  h->rows_max = nrmax + nomax;
  h->P = (long long)h->B * h->N * h->np * h->M;
  ca::Dev& v = h->dev;
  v.d = h->d; v.B = h->B; v.N = h->N; v.ns = h->ns; v.nu = h->nu; v.np = h->np; v.M = h->M;
  v.pose_model = D->pose_model;
  v.npc = (D->pose_model == CA_POSE_TRANSLATION) ? h->d : h->d + 1;
  v.nagg = ca::rec_nagg(h->d);
  v.rec = ca::rec_n(h->d);
  v.active = nullptr;
  if (!h->M_full) h->M_full = D->n_obs;
  for (int a = 0; a < 4; ++a) v.pidx[a] = D->pose_idx[a];
  v.dyn_ps = (D->dyn_per_scene || D->dyn_model) ? 1 : 0;  // relinearised: one block per (scene, t)
  v.dyn_pt = (D->dyn_per_time || D->dyn_model) ? 1 : 0;
  v.dyn_model = D->dyn_model;
  v.dt = D->dt;
  v.sigma = D->sigma;
  v.lp.pivot_tol = D->lemke_pivot_tol > 0 ? D->lemke_pivot_tol : 1e-11;
  v.lp.tie_tol = D->lemke_tie_tol > 0 ? D->lemke_tie_tol : 1e-9;
  v.lp.max_pivot_factor = D->lemke_max_pivot_factor > 0 ? D->lemke_max_pivot_factor : 50;
  v.ny = h->nmax;
  v.P = h->P;
  v.G = h->np * h->M;
  v.nchunk = std::max(1, (v.G + ca::CTA - 1) / ca::CTA);
  v.CH = std::max(1, (v.G + v.nchunk - 1) / v.nchunk);
  // sweep sort pools: TG consecutive timesteps (~CA_SWEEP_POOL pairs) per (scene,
  // group) when the sweep spans many waves (lane utilisation); one timestep per
  // pool for small problems, whose sweep is one latency-bound wave
  {
    const long long items1 = (long long)h->B * h->N * v.nchunk;
    const int tg = std::max(1, std::min(h->N, CA_SWEEP_POOL / std::max(1, v.G)));
    v.TG = (items1 >= CA_SWEEP_POOL_MIN_ITEMS) ? std::min(tg, 8) : 1;  // <= 8: k_stage_grouped smem
  }
  v.NG = (h->N + v.TG - 1) / v.TG;
  v.GG = v.TG * std::max(1, v.G);
  v.nchunkG = (v.GG + 31) / 32;
  v.CHG = (v.GG + v.nchunkG - 1) / v.nchunkG;  // balanced: lanes used per chunk
  // latency mode: a problem whose pairs fit one wave of resident warps at one pair per
  // warp is solved pair by pair with the warp-cooperative dense Lemke (a single pair's
  // revised path is a long dependent chain; below one wave only the sweep's latency
  // counts).  Measured (profiles/r01/small_configs_v21.txt), us per ADMM iteration:
  // C2 111 -> 93, C3 224 -> 182, C2t 128 -> 107, C1 even; more than one pair per warp
  // (C4: 6000 pairs) is slower dense and keeps the revised path.  CA_SWEEP_DENSE=0
  // disables.
  {
    const long long P = (long long)h->B * h->N * h->np * h->M;
    const long long resident = 148LL * CA_SWEEP_MINB;  // warps of one wave on B200
    const char* env = std::getenv("CA_SWEEP_DENSE");
    // prox_eps > 0 (reading #2) breaks the low-rank structure the revised path relies
    // on (M + eps (I + kt kt^T)): such problems take the dual Newton solver (NEXT f4,
    // one pair per thread, normal work items) or, with prox_solver 1, the dense path
    v.prox_eps = D->prox_eps;
    v.prox_newton = (D->prox_eps > 0.0 && D->prox_solver == 0) ? 1 : 0;
    v.dense = (P > 0 && !v.prox_newton && (D->prox_eps > 0.0 || (P <= resident && !(env && env[0] == '0')))) ? 1 : 0;
    if (v.dense) {  // one pair per warp, one timestep per pool (one record per pair)
      v.TG = 1;
      v.NG = h->N;
      v.GG = std::max(1, v.G);
      v.nchunkG = v.GG;
      v.CHG = 1;
    }
  }
  h->eps_pri = D->eps_pri;
  h->eps_dual = D->eps_dual;
  h->max_iters = D->max_iters > 0 ? D->max_iters : 100;
  const int d = h->d, B = h->B, N = h->N, ns = h->ns, nu = h->nu;
  const long long nd = (long long)(v.dyn_ps ? B : 1) * (v.dyn_pt ? N : 1);  // device layout
  const long long orow = (h->M > 0) ? D->obs_off[(long long)B * h->M] : 0;
  ca_status st;
#define AL(ptr, T, cnt)                          \
  do {                                           \
    T* tmp_ = nullptr;                           \
    if ((st = h->alloc(&tmp_, (size_t)(cnt)))) { \
      return st;                                 \
    }                                            \
    ptr = tmp_;                                  \
  } while (0)
  AL(v.part_rows, double, 4 * (size_t)D->part_off[h->np]);
  AL(v.part_off, int, h->np + 1);
  AL(v.obs_rows, double, 4 * (size_t)std::max<long long>(orow, 1));
  AL(v.obs_off, int, (size_t)B * h->M + 1);
  AL(v.dynA, double, nd * ns * ns);
  AL(v.dynB, double, nd * ns * nu);
  AL(v.dync, double, nd * ns);
  AL(v.Qs, double, ns * ns);
  AL(v.Qu, double, nu * nu);
  AL(v.s0, double, (size_t)B * ns);
  AL(v.sref, double, (size_t)B * (N + 1) * ns);
  AL(v.s, double, (size_t)B * (N + 1) * ns);
  AL(v.u, double, (size_t)B * N * nu);
  AL(v.y, double, (size_t)h->nmax * std::max<long long>(h->P, 1));
  AL(v.zeta, double, std::max<long long>(h->P, 1));
  AL(v.xi, double, (size_t)d * std::max<long long>(h->P, 1));
  AL(v.pst, uint32_t, std::max<long long>(h->P, 1));
  h->agg_n = (size_t)B * v.NG * v.nchunkG * v.TG * v.rec;
  AL(v.agg, double, h->agg_n);
  AL(h->scene_res, double, (size_t)B * NST);
  AL(h->s_start, double, (size_t)B * (N + 1) * ns);
  AL(v.gperm, int, (size_t)B * std::max(1, v.G));
  AL(v.gperm2, uint32_t, (size_t)B * v.NG * v.GG);
  AL(v.pose, double, (size_t)B * N * 12);
  AL(v.work, int, 1);
  AL(v.obs_vert, double, 2 * (size_t)std::max<long long>(orow, 1));
  AL(v.obs_nv, int, (size_t)B * h->M + 1);
  AL(v.part_vert, double, 2 * (size_t)D->part_off[h->np]);
  AL(v.part_nv, int, (size_t)h->np);
  AL(v.ric, double, (size_t)B * N * nu * (ns + 1));
  AL(v.stg, double, (size_t)B * N * (ns * ns + ns));
  AL(v.stg_stats, double, (size_t)B * N * NST);
  v.nitems = (int)std::min<long long>((long long)B * v.NG * v.nchunkG, 0x7fffffff);
  AL(v.lam, double, (size_t)h->np * std::max(1, v.nrmax - 1) * (d + 2));
  AL(v.part_e, int, (size_t)h->np);
  AL(v.part_be, double, (size_t)h->np);
  v.box = (D->s_min || D->s_max || D->u_min || D->u_max) ? 1 : 0;
  v.box_rho = D->box_rho;
  if (D->part_ctr) AL(v.part_ctr, double, 3 * (size_t)h->np);  // NEXT f3 scaling centres
  if (D->sense_half && h->M > 0) {  // NEXT f3 sensing mask + its box
    uint8_t* m_ = nullptr;
    if ((st = h->alloc(&m_, (size_t)B * h->M))) return st;
    v.sensed = m_;
    AL(h->sense_half, double, 3);
  }
  if (v.box) {  // NEXT f1 box block
    AL(v.box_lim, double, 2 * (size_t)(ns + nu));
    AL(v.box_ws, double, (size_t)B * (N + 1) * ns);
    AL(v.box_ls, double, (size_t)B * (N + 1) * ns);
    AL(v.box_wu, double, (size_t)B * N * nu);
    AL(v.box_lu, double, (size_t)B * N * nu);
    AL(v.box_res, double, (size_t)B);
  }
#undef AL
  // lazily used buffers that also live in the workspace: scale factors, per-iteration
  // statistics for max_iters iterations, moving-obstacle steps
  if ((st = h->alloc(&h->alpha, (size_t)h->P + h->B))) return st;
  if ((st = ensure_slots(h, h->max_iters))) return st;
  if (D->obs_step && (st = h->alloc(&h->obs_step_buf, (size_t)B * h->M * d))) return st;
  // ca_admm_solve (per-scene Eq. 18) and ca_scale_detect(states) staging
  if ((st = h->alloc(&h->active, (size_t)B)) || (st = h->alloc(&h->s_iters, (size_t)B)) ||
      (st = h->alloc(&h->s_fin, (size_t)B * NST)) || (st = h->alloc(&h->d_remaining, 1)) ||
      (st = h->alloc(&h->states_buf, (size_t)B * (N + 1) * ns)))
    return st;
  if (h->dist_mode) {  // sharded: reduced records, statistics staging, S_PMAX column
    if ((st = h->alloc(&h->rb, (size_t)B * N * v.rec)) || (st = h->alloc(&h->tmpB, (size_t)B * NST)) ||
        (st = h->alloc(&h->pmx, (size_t)std::max(B * N, B))))
      return st;
  }
  return CA_OK;
}

// create a handle for the (rank-local) problem D; g = its grid position (NULL: one GPU)
ca_status create_impl(const ca_problem_desc* D, int device, void* stream, const GridPos* g, ca_problem** out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0)
    return fail(CA_E_CUDA, "no CUDA device (this library has no CPU fallback)");
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(CA_E_CUDA, "built for sm_100a (B200); device is sm_" + std::to_string(prop.major * 10 + prop.minor));
  CUDA_TRY(cudaSetDevice(device));
  ca_problem* h = new ca_problem();
  h->device = device;
  h->stream = static_cast<cudaStream_t>(stream);
  if (D->workspace) {
    h->ws = static_cast<char*>(D->workspace);
    h->ws_size = D->workspace_bytes;
  }
  set_grid(h, g);
  ca_status st;
  if ((st = setup_handle(h, D))) {
    delete h;
    return st;
  }
  ca::Dev& v = h->dev;
  v.zmask = nullptr;
  v.dbg_p = -1;
  v.dbg = nullptr;
  if ((st = upload(h, D))) {
    delete h;
    return st;
  }
  *out = h;
  return CA_OK;
}

ca_status ca_problem_create(const ca_problem_desc* D, int device, void* stream, ca_problem** out) {
  if (!out) return fail(CA_E_INVALID, "out is NULL");
  *out = nullptr;
  ca_status st = validate(D);
  if (st) return st;
  return create_impl(D, device, stream, nullptr, out);
}

ca_status ca_workspace_size(const ca_problem_desc* D, const ca_dist_desc* dist, size_t* bytes) {
  if (!bytes) return fail(CA_E_INVALID, "bytes is NULL");
  *bytes = 0;
  ca_status st = validate(D);
  if (st) return st;
  LocalObs lobs;
  ca_problem_desc Dl;
  GridPos g;
  const ca_problem_desc* Du = D;
  if (dist) {
    if ((st = grid_position(D, dist, g, lobs, Dl))) return st;
    Du = &Dl;
  }
  ca_problem h;
  h.count_only = true;
  set_grid(&h, dist ? &g : nullptr);
  if ((st = setup_handle(&h, Du))) return st;
  *bytes = h.ws_used;
  return CA_OK;
}

void ca_problem_destroy(ca_problem* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  delete h;
}

ca_status ca_problem_load(ca_problem* h, const ca_problem_desc* Dfull) {
  ca_status st = check_handle(h);
  if (st) return st;
  h->drop_graph();  // captured kernel parameters may change
  if ((st = validate(Dfull))) return st;
  LocalObs lobs;
  ca_problem_desc Dl;
  const ca_problem_desc* D = Dfull;
  if (h->dist_mode) {  // the FULL problem: keep this rank's scene and obstacle block
    if (Dfull->n_obs != h->n_obs_full || Dfull->n_scenes != h->B_total)
      return fail(CA_E_INVALID, "ca_problem_load: scene / obstacle count differs");
    slice_problem(Dfull, h->b0, h->b0 + h->B, h->j0, h->j1, lobs, Dl);
    D = &Dl;
  }
  if (D->dim != h->d || D->n_scenes != h->B || D->horizon != h->N || D->n_state != h->ns ||
      D->n_ctrl != h->nu || D->n_parts != h->np || D->n_obs != h->M)
    return fail(CA_E_INVALID, "ca_problem_load: shapes differ from the handle");
  for (int i = 0; i <= h->np; ++i)
    if (D->part_off[i] != h->part_off[i]) return fail(CA_E_INVALID, "ca_problem_load: robot part rows differ");
  if (D->dyn_model != h->dev.dyn_model ||
      (!D->dyn_model && ((D->dyn_per_scene ? 1 : 0) != h->dev.dyn_ps || (D->dyn_per_time ? 1 : 0) != h->dev.dyn_pt)))
    return fail(CA_E_INVALID, "ca_problem_load: dynamics model / layout differs from the handle");
  for (long long o = 0; o < (long long)h->B * h->M; ++o)
    if (D->obs_off[o + 1] - D->obs_off[o] != h->obs_counts[o])
      return fail(CA_E_INVALID, "ca_problem_load: obstacle row counts differ");
  if ((D->s_min || D->s_max || D->u_min || D->u_max) != (h->dev.box != 0))
    return fail(CA_E_INVALID, "ca_problem_load: box presence differs from the handle");
  if ((D->part_ctr != nullptr) != (h->dev.part_ctr != nullptr))
    return fail(CA_E_INVALID, "ca_problem_load: scaling-centre presence differs from the handle");
  if ((D->sense_half && h->M > 0) != (h->dev.sensed != nullptr))
    return fail(CA_E_INVALID, "ca_problem_load: sensing presence differs from the handle");
  return mark(h, upload(h, D));
}

ca_status ca_debug_trace(ca_problem* h, int64_t p, double* out) {
  ca_status st = check_handle(h);
  if (st) return st;
  h->drop_graph();  // captured kernel parameters may change
  if (!h->dev.dbg) {
    if ((st = h->alloc(&h->dev.dbg, 64 * 48))) return st;
  }
  if (out) {
    CUDA_TRY(cudaMemcpy(out, h->dev.dbg, sizeof(double) * 64 * 48, cudaMemcpyDeviceToHost));
  }
  CUDA_TRY(cudaMemset(h->dev.dbg, 0xff, sizeof(double) * 64 * 48));
  h->dev.dbg_p = p;
  return CA_OK;
}

ca_status ca_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(CA_E_INVALID, "out is NULL");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return CA_OK;
}

ca_status ca_obstacle_partition(int32_t n_scenes, int32_t n_obs, const int32_t* obs_off, int32_t world, int32_t rank,
                                int32_t* j0, int32_t* j1) {
  if (!j0 || !j1 || world < 1 || rank < 0 || rank >= world || n_obs < 0 || n_scenes < 1 || (n_obs > 0 && !obs_off))
    return fail(CA_E_INVALID, "bad partition arguments");
  std::vector<long long> cnt(n_obs, 0);
  long long total = 0;
  for (int b = 0; b < n_scenes; ++b)
    for (int j = 0; j < n_obs; ++j) {
      const long long c = obs_off[(long long)b * n_obs + j + 1] - obs_off[(long long)b * n_obs + j];
      cnt[j] += c;
      total += c;
    }
  auto bnd = [&](int k) -> int {
    if (k <= 0) return 0;
    if (k >= world) return n_obs;
    long long acc = 0;
    for (int j = 0; j < n_obs; ++j) {
      if (acc * world >= (long long)k * total) return j;
      acc += cnt[j];
    }
    return n_obs;
  };
  *j0 = bnd(rank);
  *j1 = bnd(rank + 1);
  return CA_OK;
}

ca_status ca_problem_create_dist(const ca_problem_desc* D, const ca_dist_desc* dist, int device, void* stream,
                                 ca_problem** out) {
  if (!dist) return ca_problem_create(D, device, stream, out);
  if (!out) return fail(CA_E_INVALID, "out is NULL");
  *out = nullptr;
  ca_status st = validate(D);
  if (st) return st;
  LocalObs lobs;
  ca_problem_desc Dl;
  GridPos g;
  if ((st = grid_position(D, dist, g, lobs, Dl))) return st;
  ca_problem* h = nullptr;
  if ((st = create_impl(&Dl, device, stream, &g, &h))) return st;
  // the world communicator; the obstacle group by ncclCommSplit (color = scene shard)
  ncclUniqueId id;
  std::memcpy(&id, dist->nccl_id, sizeof(id));
  ncclComm_t world = nullptr;
  ncclResult_t r = ncclCommInitRank(&world, g.world, id, g.rank);
  if (r != ncclSuccess) {
    delete h;
    return fail(CA_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  if (!h->scene_xchg) {
    h->comm = world;  // one scene shard: the world is the obstacle group
  } else {
    h->comm_all = world;
    if (g.Wo > 1) {
      r = ncclCommSplit(world, g.rs, g.ro, &h->comm, nullptr);
      if (r != ncclSuccess) {
        h->comm = nullptr;
        delete h;
        return fail(CA_E_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
      }
    }
  }
  *out = h;
  return CA_OK;
}

ca_status ca_reset_iterate(ca_problem* h) {
  ca_status st = check_handle(h);
  if (st) return st;
  return mark(h, reset_iterate(h));
}

ca_status ca_problem_info(const ca_problem* h, int64_t* n_pairs, int32_t* ny, int64_t* device_bytes) {
  if (!h) return fail(CA_E_INVALID, "NULL handle");
  if (n_pairs) *n_pairs = h->P;
  if (ny) *ny = h->nmax;
  if (device_bytes) *device_bytes = h->bytes;
  return CA_OK;
}

ca_status ca_set_timing(ca_problem* h, int32_t enable) {
  if (!h) return fail(CA_E_INVALID, "NULL handle");
  h->timing = enable != 0;
  return CA_OK;
}

ca_status ca_kernel_times(ca_problem* h, double* ms, int64_t* launches, int32_t reset) {
  ca_status st = check_handle(h);
  if (st) return st;
  if ((st = flush_timing(h))) return mark(h, st);
  for (int f = 0; f < NFAM; ++f) {
    if (ms) ms[f] = h->ms[f];
    if (launches) launches[f] = h->launches[f];
    if (reset) {
      h->ms[f] = 0;
      h->launches[f] = 0;
    }
  }
  return CA_OK;
}

ca_status ca_set_record_basis(ca_problem* h, int32_t enable) {
  ca_status st = check_handle(h);
  if (st) return st;
  h->drop_graph();
  if (enable && !h->dev.zmask) {
    uint32_t* z = nullptr;
    if ((st = h->alloc(&z, std::max<long long>(h->P, 1)))) return st;
    CUDA_TRY(cudaMemsetAsync(z, 0, sizeof(uint32_t) * std::max<long long>(h->P, 1), h->stream));
    h->dev.zmask = z;
  } else if (!enable) {
    h->dev.zmask = nullptr;
  }
  return CA_OK;
}

// the device milliseconds per family of the launches recorded since `mark` (timing on)
ca_status step_ms(ca_problem* h, ca_residuals* r) {
  if (!h->timing) return CA_OK;
  double fam[NFAM] = {0, 0, 0, 0, 0, 0};
  const int it = h->cur_iter;
  for (auto& pe : h->pending) pe.iter = 0;
  ca_status st = flush_timing(h, fam, 1);
  h->cur_iter = it;
  if (st) return st;
  fill_ms(fam, r);
  return CA_OK;
}

ca_status ca_dual_sweep(ca_problem* h, ca_residuals* out) {
  ca_status st = check_handle(h);
  if (st) return st;
  if ((st = flush_timing(h))) return mark(h, st);
  if ((st = launch_sweep(h, false))) return mark(h, st);
  CUDA_TRY(cudaMemsetAsync(h->scene_res, 0, sizeof(double) * NST * h->B, h->stream));
  if ((st = collect_global(h, h->scene_res, 0xff & ~(1 << ca::S_RPRI)))) return mark(h, st);
  ca_residuals r{};
  if ((st = sums(h, h->scene_res, &r))) return mark(h, st);
  if ((st = step_ms(h, &r))) return mark(h, st);
  r.r_pri = 0.0;
  if (out) *out = r;
  return r.n_fail ? CA_W_PAIR_FAILURES : CA_OK;
}

ca_status ca_primal_step(ca_problem* h) {
  ca_status st = check_handle(h);
  if (st) return st;
  if ((st = launch_riccati(h, nullptr, nullptr))) return mark(h, st);
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

// the dist-path buffers (reduced records, S_PMAX column) on a single-GPU handle
ca_status ensure_rb(ca_problem* h) {
  ca_status st;
  if (!h->rb && (st = h->alloc(&h->rb, (size_t)h->B * h->N * h->dev.rec))) return st;
  if (!h->pmx && (st = h->alloc(&h->pmx, (size_t)std::max(h->B * h->N, h->B)))) return st;
  return CA_OK;
}

ca_status ca_get_stage_records(ca_problem* h, double* rec) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (!rec) return fail(CA_E_INVALID, "rec is NULL");
  if ((st = ensure_rb(h))) return mark(h, st);
  const long long nq = (long long)h->B * h->N;
  const unsigned gq = (unsigned)((nq + 127) / 128);
  ca::k_reduce_records<<<gq, 128, 0, h->stream>>>(h->dev, h->rb, h->pmx);
  CUDA_TRY(cudaGetLastError());
  ca::k_pmax_back<<<gq, 128, 0, h->stream>>>(h->dev, h->rb, h->pmx);
  CUDA_TRY(cudaGetLastError());
  h->launches[4] += 2;
  CUDA_TRY(cudaMemcpyAsync(rec, h->rb, sizeof(double) * nq * h->dev.rec, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_primal_step_records(ca_problem* h, const double* rec) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (!rec) return fail(CA_E_INVALID, "rec is NULL");
  if ((st = ensure_rb(h))) return mark(h, st);
  const long long nq = (long long)h->B * h->N;
  CUDA_TRY(cudaMemcpyAsync(h->rb, rec, sizeof(double) * nq * h->dev.rec, cudaMemcpyHostToDevice, h->stream));
  if ((st = launch_riccati(h, nullptr, nullptr, h->rb))) return mark(h, st);
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_multiplier_update(ca_problem* h, ca_residuals* out) {
  ca_status st = check_handle(h);
  if (st) return st;
  if ((st = flush_timing(h))) return mark(h, st);
  if ((st = launch_mult(h))) return mark(h, st);
  if ((st = collect_global(h, h->scene_res, 1 << ca::S_RPRI))) return mark(h, st);
  ca_residuals r{};
  if ((st = sums(h, h->scene_res, &r))) return mark(h, st);
  ca_residuals o{};
  if ((st = step_ms(h, &o))) return mark(h, st);
  o.r_pri = r.r_pri;
  o.n_pairs = h->P;
  if (out) *out = o;
  return CA_OK;
}

// The device work of one ca_admm_iterate(iters): K sweeps + primal steps, the final
// multiplier update, residual collection and the per-iteration history.  Scene-sharded
// runs add one allreduce of every scene's statistics per iteration (scene_exchange) and
// take the history from that global table.
ca_status enqueue_iterations(ca_problem* h, int iters) {
  ca_status st;
  const size_t SL = (size_t)h->B * NST, GL = (size_t)h->B_total * NST;
  CUDA_TRY(cudaMemsetAsync(h->slots, 0, sizeof(double) * (size_t)iters * SL, h->stream));
  if (h->comm_all) CUDA_TRY(cudaMemsetAsync(h->glob, 0, sizeof(double) * (size_t)iters * GL, h->stream));
  for (int it = 0; it < iters; ++it) {
    h->cur_iter = it;
    if ((st = launch_sweep(h, it > 0))) return st;
    double* cur = h->slots + (size_t)it * SL;
    double* prev = it > 0 ? h->slots + (size_t)(it - 1) * SL : nullptr;
    if ((st = launch_riccati(h, cur, prev))) return st;
    if (prev && (st = scene_exchange(h, prev, h->glob + (size_t)(it - 1) * GL))) return st;  // slot it-1 complete
  }
  h->cur_iter = iters - 1;
  if ((st = launch_mult(h))) return st;
  double* last = h->slots + (size_t)(iters - 1) * SL;
  if ((st = collect_global(h, last, 1 << ca::S_RPRI))) return st;
  if ((st = scene_exchange(h, last, h->glob + (size_t)(iters - 1) * GL))) return st;
  CUDA_TRY(cudaMemcpyAsync(h->scene_res, last, sizeof(double) * SL, cudaMemcpyDeviceToDevice, h->stream));
  if (h->comm_all) ca::k_hist<<<iters, 256, 0, h->stream>>>(h->glob, h->B_total, iters, h->hist_dev);
  else ca::k_hist<<<iters, 256, 0, h->stream>>>(h->slots, h->B, iters, h->hist_dev);
  CUDA_TRY(cudaGetLastError());
  h->launches[4]++;
  h->cur_iter = -1;
  return CA_OK;
}

// Replay (capturing on first use) the CUDA graph of enqueue_iterations(iters):
// single-GPU handles with timing off (small configurations are
// launch-bound).  The launch counters advance as if the kernels had been enqueued.
ca_status launch_iterations_graph(ca_problem* h, int iters) {
  if (!h->gexec || h->g_iters != iters) {
    h->drop_graph();
    long long before[NFAM];
    for (int f = 0; f < NFAM; ++f) before[f] = h->launches[f];
    if (!h->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    const cudaStream_t user = h->stream;
    h->stream = h->cap_stream;  // the launch helpers enqueue on h->stream
    const cudaError_t be = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal);
    if (be != cudaSuccess) {
      h->stream = user;
      return fail(CA_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(be));
    }
    ca_status st = enqueue_iterations(h, iters);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    h->stream = user;
    if (st) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess) return fail(CA_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&h->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      h->gexec = nullptr;
      return fail(CA_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    }
    h->g_iters = iters;
    for (int f = 0; f < NFAM; ++f) {
      h->g_launches[f] = h->launches[f] - before[f];
      h->launches[f] = before[f];
    }
  }
  CUDA_TRY(cudaGraphLaunch(h->gexec, h->stream));
  for (int f = 0; f < NFAM; ++f) h->launches[f] += h->g_launches[f];
  return CA_OK;
}

// K iterations; hist (HOST [iters], nullable) gets each iteration's statistics (global
// in scene-sharded runs) and, with timing on, its device milliseconds per family.
ca_status iterate_impl(ca_problem* h, int32_t iters, ca_residuals* hist) {
  ca_status st;
  if (iters > h->slots_cap) h->drop_graph();  // slot buffers are reallocated
  if ((st = ensure_slots(h, iters))) return st;
  if ((st = flush_timing(h))) return st;
  // the per-iteration NCCL collectives are captured too (NCCL supports stream capture):
  // the sharded iteration replays as one graph like the single-GPU one
  const bool graph = h->use_graphs && !h->timing && h->dev.dbg_p < 0 && !h->dev.active;
  if ((st = graph ? launch_iterations_graph(h, iters) : enqueue_iterations(h, iters))) return st;
  if (!hist) {
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return CA_OK;
  }
  std::vector<double> hv((size_t)iters * NST), fam;
  CUDA_TRY(cudaMemcpyAsync(hv.data(), h->hist_dev, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (h->timing) {
    fam.assign((size_t)iters * NFAM, 0.0);
    if ((st = flush_timing(h, fam.data(), iters))) return st;
  }
  for (int k = 0; k < iters; ++k) {
    fill_res(&hv[(size_t)k * NST], h->P, &hist[k]);
    if (h->timing) fill_ms(&fam[(size_t)k * NFAM], &hist[k]);
  }
  return CA_OK;
}

ca_status ca_admm_iterate(ca_problem* h, int32_t iters, ca_residuals* hist) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (iters <= 0) return fail(CA_E_INVALID, "iters must be > 0");
  std::vector<ca_residuals> own;
  if (!hist) {  // the failure count decides the warning
    own.resize((size_t)iters);
    hist = own.data();
  }
  if ((st = iterate_impl(h, iters, hist))) return mark(h, st);
  int64_t fails = 0;
  for (int k = 0; k < iters; ++k) fails += hist[k].n_fail;
  return fails ? CA_W_PAIR_FAILURES : CA_OK;
}

// ADMM until Eq. 18 per scene: one iteration at a time; after each, k_stop
// freezes the scenes that meet Eq. 18 (the kernels skip them from the next iteration on,
// so their iterate stays where they stopped) and counts the scenes still running (in a
// scene-sharded run summed over every rank: the same count, hence the same loop, on
// every rank -- no rank can leave a collective the others still enter).
ca_status solve_impl(ca_problem* h, ca_solve_report* out) {
  ca_status st;
  const double pairs_per_scene = (double)h->N * h->np * h->M_full;  // the FULL problem's
  const double ep = h->eps_pri > 0 ? h->eps_pri : 1e-3 * std::max(1.0, pairs_per_scene);
  const double ed = h->eps_dual > 0 ? h->eps_dual : 1e-3 * std::max(1.0, pairs_per_scene);
  CUDA_TRY(cudaMemsetAsync(h->active, 1, (size_t)h->B, h->stream));
  CUDA_TRY(cudaMemsetAsync(h->s_iters, 0, sizeof(int) * h->B, h->stream));
  CUDA_TRY(cudaMemsetAsync(h->s_fin, 0, sizeof(double) * NST * h->B, h->stream));
  h->drop_graph();
  h->dev.active = h->active;
  h->solved = true;
  int done_iters = 0;
  for (int k = 0; k < h->max_iters; ++k) {
    if ((st = iterate_impl(h, 1, nullptr))) return st;
    CUDA_TRY(cudaMemsetAsync(h->d_remaining, 0, sizeof(int), h->stream));
    ca::k_stop<<<(h->B + 127) / 128, 128, 0, h->stream>>>(h->scene_res, h->active, h->s_iters, h->s_fin, h->B, ep, ed,
                                                         k, h->d_remaining);
    CUDA_TRY(cudaGetLastError());
    h->launches[4]++;
    if (h->comm_all) {
      cudaEvent_t c0 = nullptr;
      t_begin(h, &c0);
      NCCL_TRY(ncclAllReduce(h->d_remaining, h->d_remaining, 1, ncclInt32, ncclSum, h->comm_all, h->stream));
      t_end(h, 5, c0);
    }
    int remaining = 0;
    CUDA_TRY(cudaMemcpyAsync(&remaining, h->d_remaining, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    done_iters = k + 1;
    if (remaining == 0) break;
  }
  // every scene's statistics at its own last iteration become the scene residuals
  CUDA_TRY(cudaMemcpyAsync(h->scene_res, h->s_fin, sizeof(double) * NST * h->B, cudaMemcpyDeviceToDevice, h->stream));
  std::vector<int> it((size_t)h->B);
  std::vector<uint8_t> act((size_t)h->B);
  CUDA_TRY(cudaMemcpyAsync(it.data(), h->s_iters, sizeof(int) * h->B, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(act.data(), h->active, (size_t)h->B, cudaMemcpyDeviceToHost, h->stream));
  ca_solve_report rep{};
  if ((st = sums(h, h->s_fin, &rep.last))) return st;
  int conv = 1, mx = 0;
  for (int b = 0; b < h->B; ++b) {
    conv &= act[b] ? 0 : 1;
    mx = std::max(mx, it[b]);
  }
  rep.iterations = h->comm_all ? done_iters : mx;
  rep.converged = conv;
  if (h->comm_all) {  // statistics of every scene of every rank (each scene counted once)
    double c[NST] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (h->ro == 0) {
      c[ca::S_RDUAL] = rep.last.r_dual;
      c[ca::S_RPRI] = rep.last.r_pri;
      c[ca::S_PIV] = (double)rep.last.pivots;
      c[ca::S_FAIL] = (double)rep.last.n_fail;
      c[ca::S_RAY] = (double)rep.last.n_ray;
      c[ca::S_ITER] = (double)rep.last.n_iterlimit;
      c[ca::S_NEGYE] = (double)rep.last.n_neg_ye;
      c[ca::S_PMAX] = (double)rep.last.max_pivots;
    }
    CUDA_TRY(cudaMemcpyAsync(h->tmpB, c, sizeof(c), cudaMemcpyHostToDevice, h->stream));
    if ((st = allreduce_stats(h, h->tmpB, 1, h->comm_all))) return st;
    CUDA_TRY(cudaMemcpyAsync(c, h->tmpB, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    fill_res(c, h->P, &rep.last);
  }
  if (h->comm_all) {  // global: every scene of every rank
    int c = conv;
    int* dc = h->d_remaining;
    CUDA_TRY(cudaMemcpyAsync(dc, &c, sizeof(int), cudaMemcpyHostToDevice, h->stream));
    NCCL_TRY(ncclAllReduce(dc, dc, 1, ncclInt32, ncclMin, h->comm_all, h->stream));
    CUDA_TRY(cudaMemcpyAsync(&c, dc, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    rep.converged = c;
  }
  if (out) *out = rep;
  return rep.converged ? CA_OK : CA_W_NOT_CONVERGED;
}

ca_status ca_admm_solve(ca_problem* h, ca_solve_report* out) {
  ca_status st = check_handle(h);
  if (st) return st;
  st = solve_impl(h, out);
  h->dev.active = nullptr;  // later ca_admm_iterate calls run every scene again
  h->drop_graph();
  return (st < 0) ? mark(h, st) : st;
}

ca_status ca_get_solve_scenes(ca_problem* h, int32_t* iterations, int32_t* converged) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (!h->solved) return fail(CA_E_INVALID, "no ca_admm_solve has run on this handle");
  std::vector<int> it((size_t)h->B);
  std::vector<uint8_t> act((size_t)h->B);
  CUDA_TRY(cudaMemcpyAsync(it.data(), h->s_iters, sizeof(int) * h->B, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(act.data(), h->active, (size_t)h->B, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int b = 0; b < h->B; ++b) {
    if (iterations) iterations[b] = it[b];
    if (converged) converged[b] = act[b] ? 0 : 1;
  }
  return CA_OK;
}

ca_status ca_get_scene_residuals(ca_problem* h, double* r_pri, double* r_dual) {
  ca_status st = check_handle(h);
  if (st) return st;
  std::vector<double> v((size_t)h->B * NST);
  CUDA_TRY(cudaMemcpyAsync(v.data(), h->scene_res, sizeof(double) * v.size(), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  for (int b = 0; b < h->B; ++b) {
    if (r_pri) r_pri[b] = v[(size_t)b * NST + ca::S_RPRI];
    if (r_dual) r_dual[b] = v[(size_t)b * NST + ca::S_RDUAL];
  }
  return CA_OK;
}

ca_status ca_get_trajectory(ca_problem* h, double* s, double* u) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (s) CUDA_TRY(cudaMemcpyAsync(s, h->dev.s, sizeof(double) * (size_t)h->B * (h->N + 1) * h->ns, cudaMemcpyDeviceToHost, h->stream));
  if (u) CUDA_TRY(cudaMemcpyAsync(u, h->dev.u, sizeof(double) * (size_t)h->B * h->N * h->nu, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_get_pair_state(ca_problem* h, int64_t p0, int64_t count, double* y, double* zeta, double* xi,
                            int32_t* pivots, int32_t* status, uint32_t* zmask) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (p0 < 0 || count < 0 || p0 + count > h->P) return fail(CA_E_INVALID, "pair range out of bounds");
  if (count == 0) return CA_OK;
  const int ny = h->nmax, d = h->d;
  std::vector<double> tmp((size_t)count);
  if (y) {
    for (int k = 0; k < ny; ++k) {
      CUDA_TRY(cudaMemcpyAsync(tmp.data(), h->dev.y + (size_t)k * h->P + p0, sizeof(double) * count, cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
      for (int64_t q = 0; q < count; ++q) y[q * ny + k] = tmp[q];
    }
  }
  if (zeta) CUDA_TRY(cudaMemcpyAsync(zeta, h->dev.zeta + p0, sizeof(double) * count, cudaMemcpyDeviceToHost, h->stream));
  if (xi) {
    for (int a = 0; a < d; ++a) {
      CUDA_TRY(cudaMemcpyAsync(tmp.data(), h->dev.xi + (size_t)a * h->P + p0, sizeof(double) * count, cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
      for (int64_t q = 0; q < count; ++q) xi[q * d + a] = tmp[q];
    }
  }
  if (pivots || status) {
    std::vector<uint32_t> ps((size_t)count);
    CUDA_TRY(cudaMemcpyAsync(ps.data(), h->dev.pst + p0, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (int64_t q = 0; q < count; ++q) {
      if (pivots) pivots[q] = (int32_t)(ps[q] & 0xffffu);
      if (status) status[q] = (int32_t)((ps[q] >> 16) & 0xf) | (int32_t)(ps[q] & (1u << 20) ? 0x100 : 0);
    }
  }
  if (zmask) {
    if (!h->dev.zmask) return fail(CA_E_INVALID, "basis recording is off (ca_set_record_basis)");
    CUDA_TRY(cudaMemcpyAsync(zmask, h->dev.zmask + p0, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost, h->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_set_iterate(ca_problem* h, const double* s, const double* u, const double* y, const double* zeta,
                         const double* xi) {
  ca_status st = check_handle(h);
  if (st) return st;
  const int ny = h->nmax, d = h->d;
  if (s) CUDA_TRY(cudaMemcpyAsync(h->dev.s, s, sizeof(double) * (size_t)h->B * (h->N + 1) * h->ns, cudaMemcpyHostToDevice, h->stream));
  if (u) CUDA_TRY(cudaMemcpyAsync(h->dev.u, u, sizeof(double) * (size_t)h->B * h->N * h->nu, cudaMemcpyHostToDevice, h->stream));
  if (zeta && h->P) CUDA_TRY(cudaMemcpyAsync(h->dev.zeta, zeta, sizeof(double) * h->P, cudaMemcpyHostToDevice, h->stream));
  std::vector<double> tmp;
  if (y && h->P) {
    tmp.resize((size_t)h->P);
    for (int k = 0; k < ny; ++k) {
      for (long long q = 0; q < h->P; ++q) tmp[q] = y[q * ny + k];
      CUDA_TRY(cudaMemcpyAsync(h->dev.y + (size_t)k * h->P, tmp.data(), sizeof(double) * h->P, cudaMemcpyHostToDevice, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
  }
  if (xi && h->P) {
    tmp.resize((size_t)h->P);
    for (int a = 0; a < d; ++a) {
      for (long long q = 0; q < h->P; ++q) tmp[q] = xi[q * d + a];
      CUDA_TRY(cudaMemcpyAsync(h->dev.xi + (size_t)a * h->P, tmp.data(), sizeof(double) * h->P, cudaMemcpyHostToDevice, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
  }
  if ((st = box_reset(h, 0))) return mark(h, st);
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_get_box_state(ca_problem* h, double* w_s, double* l_s, double* w_u, double* l_u, double* res) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (!h->dev.box) return fail(CA_E_INVALID, "the problem has no state/control box");
  const size_t ns_n = (size_t)h->B * (h->N + 1) * h->ns, nu_n = (size_t)h->B * h->N * h->nu;
  if (w_s) CUDA_TRY(cudaMemcpyAsync(w_s, h->dev.box_ws, sizeof(double) * ns_n, cudaMemcpyDeviceToHost, h->stream));
  if (l_s) CUDA_TRY(cudaMemcpyAsync(l_s, h->dev.box_ls, sizeof(double) * ns_n, cudaMemcpyDeviceToHost, h->stream));
  if (w_u) CUDA_TRY(cudaMemcpyAsync(w_u, h->dev.box_wu, sizeof(double) * nu_n, cudaMemcpyDeviceToHost, h->stream));
  if (l_u) CUDA_TRY(cudaMemcpyAsync(l_u, h->dev.box_lu, sizeof(double) * nu_n, cudaMemcpyDeviceToHost, h->stream));
  if (res) CUDA_TRY(cudaMemcpyAsync(res, h->dev.box_res, sizeof(double) * h->B, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_scale_detect(ca_problem* h, const double* states, double* alpha, double* min_alpha) {
  ca_status st = check_handle(h);
  if (st) return st;
  if (h->P == 0) {  // no local pairs: +inf minima -- but still join the group's min-allreduce
    std::vector<double> inf((size_t)h->B, INFINITY);
    CUDA_TRY(cudaMemcpyAsync(h->alpha, inf.data(), sizeof(double) * h->B, cudaMemcpyHostToDevice, h->stream));
    if (h->comm) NCCL_TRY(ncclAllReduce(h->alpha, h->alpha, h->B, ncclDouble, ncclMin, h->comm, h->stream));
    if (min_alpha) CUDA_TRY(cudaMemcpyAsync(min_alpha, h->alpha, sizeof(double) * h->B, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return CA_OK;
  }
  const double* sd = h->dev.s;
  if (states) {  // the handle's own staging buffer (allocated at create)
    CUDA_TRY(cudaMemcpyAsync(h->states_buf, states, sizeof(double) * (size_t)h->B * (h->N + 1) * h->ns,
                             cudaMemcpyHostToDevice, h->stream));
    sd = h->states_buf;
  }
  cudaEvent_t e0 = nullptr;
  t_begin(h, &e0);
  const size_t sm = sizeof(double) * (size_t)ca::CTA * h->rows_max * (h->d + 2);
  const long long grid = (long long)h->B * h->N * h->dev.nchunk;
  if (h->d == 2) {
    ca::k_scale2<<<(unsigned)((h->P + 127) / 128), 128, 0, h->stream>>>(h->dev, sd, h->alpha);
  } else {
    CUDA_TRY(cudaFuncSetAttribute(ca::k_scale<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    ca::k_scale<3><<<(unsigned)grid, ca::CTA, sm, h->stream>>>(h->dev, sd, h->alpha);
  }
  CUDA_TRY(cudaGetLastError());
  ca::k_scene_min<<<h->B, 256, 0, h->stream>>>(h->alpha, h->P / h->B, h->alpha + h->P);
  CUDA_TRY(cudaGetLastError());
  h->launches[3]++;  // k_scene_min (k_scale is counted by t_end)
  if (h->comm)  // obstacle group: the per-scene minimum over every rank's obstacles
    NCCL_TRY(ncclAllReduce(h->alpha + h->P, h->alpha + h->P, h->B, ncclDouble, ncclMin, h->comm, h->stream));
  t_end(h, 3, e0);
  if (alpha) CUDA_TRY(cudaMemcpyAsync(alpha, h->alpha, sizeof(double) * h->P, cudaMemcpyDeviceToHost, h->stream));
  if (min_alpha) CUDA_TRY(cudaMemcpyAsync(min_alpha, h->alpha + h->P, sizeof(double) * h->B, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return CA_OK;
}

ca_status ca_fp64_peak(int device, double ms_target, double* tflops) {
  if (!tflops) return fail(CA_E_INVALID, "tflops is NULL");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  double* out = nullptr;
  CUDA_TRY(cudaMalloc(&out, sizeof(double)));
  const int blocks = prop.multiProcessorCount * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  long long iters = 1000;
  float ms = 0.f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    ca::k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    CUDA_TRY(cudaEventSynchronize(b));
    CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
    if (ms >= 0.5 * ms_target) break;
    iters = (long long)(iters * std::min(50.0, std::max(2.0, ms_target / std::max(ms, 1e-3f))));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double fmas = (double)blocks * threads * iters * 32.0;
  *tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
  return CA_OK;
}

}  // extern "C"
