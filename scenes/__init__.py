"""Seeded synthetic scene generators for the five BASELINE.json configs.

This module is shared by the CPU oracle tests and the CUDA path.  It holds the
*problem definition only* (geometry in H-representation, the linear-time-varying
dynamics a user would supply, weights, reference trajectory, initial state) and
none of the method's arithmetic (no scale LP, pair QP, LCP, Lemke, Riccati,
multiplier or residual code).  Every scene is a pure function of its seed.

Recipe:
  * dt = 0.1 s, sigma = 300 (Sec. V-A).
  * Face rows of every polytope have unit norm (reading c.3 #17).
  * Robot parts contain their body origin (b_i > 0, reading c.3 #22).
  * Car scenes (C1, C2, C4, C5): kinematic unicycle s=(x,y,theta,v), u=(a,omega),
    linearised by the generator about the reference (the user-supplied LTV
    dynamics of BASELINE.json north_star; PAPER.md:272 linearisation).
    Q_s = diag(1,1,0.1,0.1), Q_u = diag(0.1,0.1).
  * Quadrotor (C3): s=(p in R^3, v in R^3, psi), u=(a in R^3, omega_z); exactly
    linear.  Q_s = diag(1,1,1,0.1,0.1,0.1,0.1), Q_u = 0.1 I.
  * Seeds: C1..C4 use seed 1..4; C5 scene b uses seed 5_000_000 + b, so any
    subset of C5 scenes can be regenerated alone (oracle sampling).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

POSE_TRANSLATION = 0
POSE_SE2 = 1
POSE_TRANS_YAW = 2

DT = 0.1
SIGMA = 300.0

CONFIG_NAMES = {
    1: "C1: 2D rectangle vehicle vs 1 square obstacle, N=10, K=50",
    2: "C2: 2D car through 4 polygonal obstacles, N=50, K=200",
    3: "C3: 3D quadrotor (3 boxes) through a gap in 8 polyhedra, N=40, K=100",
    4: "C4: dense traffic, ego car vs 100 vehicles, N=60, K=300",
    5: "C5: 4096 scenes x 200 obstacles x N=50, K=100",
    6: "C4m: C4 with moving traffic (vehicles at 12-18 m/s, NEXT f3), N=60, K=300",
    7: "C2n: C2 with the unicycle relinearised at every ADMM iterate (SQP, NEXT f2), N=50, K=200",
    8: "C2b: C2 with state/control boxes (|a| <= 0.5, |om| <= 1.5, 2.5 <= v <= 3.5; NEXT f1), N=50, K=200",
    9: "C4s: C4m sensing only the vehicles within 60 m x 8 m of the ego (P:541; NEXT f3), N=60, K=300",
    10: "C2t: C2 with a rigid trailer behind the body origin, scaled about its own centre (NEXT f3), N=50, K=200",
    11: "C2p: C2's obstacles, point-mass (double-integrator) car of fixed heading, TRANSLATION pose, N=50, K=200",
    12: "C3p: C3's wall and quadrotor with the TRANSLATION pose (yaw not part of the pose), N=40, K=100",
}


@dataclasses.dataclass
class Scene:
    """A batch of B independent MPC problems sharing robot geometry and horizon.

    Layouts (all row-major, float64 unless noted):
      part_off  int32[n_parts+1]   CSR row offsets of robot parts
      part_A    [rows, d]          body-frame face normals a_k  (A_i x <= b_i)
      part_b    [rows]             b_i > 0
      obs_off   int32[B*M+1]       CSR row offsets, obstacle (b, j) = b*M + j
      obs_C     [rows, d]          world-frame face normals c_l (C_j y <= d_j)
      obs_d     [rows]
      dyn_A     [nd, ns, ns]       nd = (B if dyn_per_scene else 1) * (N if dyn_per_time else 1)
      dyn_B     [nd, ns, nu]       s_{t+1} = A_t s_t + B_t u_t + c_t
      dyn_c     [nd, ns]
      s0        [B, ns]
      s_ref     [B, N+1, ns]
    """

    name: str
    dim: int
    n_scenes: int
    horizon: int
    n_state: int
    n_ctrl: int
    pose_model: int
    pose_idx: np.ndarray
    part_off: np.ndarray
    part_A: np.ndarray
    part_b: np.ndarray
    n_obs: int
    obs_off: np.ndarray
    obs_C: np.ndarray
    obs_d: np.ndarray
    dyn_per_scene: int
    dyn_per_time: int
    dyn_A: np.ndarray
    dyn_B: np.ndarray
    dyn_c: np.ndarray
    Qs: np.ndarray
    Qu: np.ndarray
    s0: np.ndarray
    s_ref: np.ndarray
    sigma: float = SIGMA
    iters: int = 50
    dt: float = DT
    seed: int = 0
    config: int = 0
    # NEXT f3 (moving obstacles): None = static (reading #15), else [B*M, d] displacement
    # of each obstacle per timestep (obstacle j at timestep t is O_j + t*obs_step[j])
    obs_step: Optional[np.ndarray] = None
    # 0: dyn_A/B/c as given; 1: the car's unicycle relinearised at every ADMM iterate
    # (SQP step; NEXT f2) -- dyn_A/B/c then only seed nothing
    dyn_model: int = 0
    # NEXT f1: state / control boxes of Eq. 13c-d; None = unbounded, else
    # [n_state] / [n_ctrl] (+-inf entries allowed); box_rho = penalty of the box block
    s_min: Optional[np.ndarray] = None
    s_max: Optional[np.ndarray] = None
    u_min: Optional[np.ndarray] = None
    u_max: Optional[np.ndarray] = None
    box_rho: float = 0.0
    # NEXT f3 sensing: None = every obstacle, else [dim] half-extents of the
    # world-aligned box around the robot's current position; only obstacles meeting it
    # enter the (i, j, t) table
    sense_half: Optional[np.ndarray] = None
    # NEXT f3: per-part scaling centres [n_parts, d] (body frame, strictly inside each
    # part); None = every part scales about the body origin (reading #22)
    part_ctr: Optional[np.ndarray] = None

    @property
    def n_parts(self) -> int:
        return len(self.part_off) - 1

    @property
    def n_pairs(self) -> int:
        return self.n_scenes * self.horizon * self.n_parts * self.n_obs

    @property
    def n_max(self) -> int:
        """Largest LCP size n = n_r + n_o + 1 over all pairs."""
        nr = np.diff(self.part_off).max()
        no = np.diff(self.obs_off).max() if self.n_obs > 0 else 0
        return int(nr + no + 1)

    def lcp_sizes(self) -> np.ndarray:
        """n per pair in pair order p = ((b*N + t-1)*n_p + i)*M + j."""
        nr = np.diff(self.part_off)
        no = np.diff(self.obs_off).reshape(self.n_scenes, self.n_obs)
        per_b = nr[None, :, None] + no[:, None, :] + 1  # [B, n_p, M]
        return np.broadcast_to(per_b[:, None], (self.n_scenes, self.horizon) + per_b.shape[1:]).reshape(-1)

    def subset(self, scene_ids: Sequence[int]) -> "Scene":
        """The same problems restricted to a subset of scenes (independent problems)."""
        ids = list(scene_ids)
        M = self.n_obs
        offs, Cs, ds = [0], [], []
        for b in ids:
            for j in range(M):
                lo, hi = self.obs_off[b * M + j], self.obs_off[b * M + j + 1]
                Cs.append(self.obs_C[lo:hi])
                ds.append(self.obs_d[lo:hi])
                offs.append(offs[-1] + hi - lo)
        d = self.dim
        obs_C = np.concatenate(Cs) if Cs else np.zeros((0, d))
        obs_d = np.concatenate(ds) if ds else np.zeros((0,))
        nt = self.horizon if self.dyn_per_time else 1
        if self.dyn_per_scene:
            sel = np.concatenate([np.arange(b * nt, (b + 1) * nt) for b in ids])
            dA, dB, dc = self.dyn_A[sel], self.dyn_B[sel], self.dyn_c[sel]
        else:
            dA, dB, dc = self.dyn_A, self.dyn_B, self.dyn_c
        return dataclasses.replace(
            self,
            n_scenes=len(ids),
            obs_off=np.asarray(offs, np.int32),
            obs_C=np.ascontiguousarray(obs_C),
            obs_d=np.ascontiguousarray(obs_d),
            dyn_A=np.ascontiguousarray(dA),
            dyn_B=np.ascontiguousarray(dB),
            dyn_c=np.ascontiguousarray(dc),
            s0=np.ascontiguousarray(self.s0[ids]),
            s_ref=np.ascontiguousarray(self.s_ref[ids]),
            obs_step=None if self.obs_step is None else np.ascontiguousarray(
                np.concatenate([self.obs_step[b * M:(b + 1) * M] for b in ids])),
        )


# ----------------------------------------------------------------------------
# geometry builders (H-representation; unit-norm rows)
# ----------------------------------------------------------------------------

def box_hrep(center, half, yaw: float = 0.0):
    """Axis-aligned (then yawed about z) box. Rows: +e0,-e0,+e1,-e1[,+e2,-e2]."""
    center = np.asarray(center, float)
    half = np.asarray(half, float)
    d = len(center)
    A = np.zeros((2 * d, d))
    for k in range(d):
        A[2 * k, k] = 1.0
        A[2 * k + 1, k] = -1.0
    b = np.repeat(half, 2)
    if yaw != 0.0:
        c, s = math.cos(yaw), math.sin(yaw)
        Rz = np.eye(d)
        Rz[0, 0], Rz[0, 1], Rz[1, 0], Rz[1, 1] = c, -s, s, c
        A = A @ Rz.T  # face normals rotate with the body
    return A, b + A @ center


def polygon_hrep(center, radius, angles):
    """Convex polygon with vertices center + r(cos a, sin a), a sorted CCW."""
    center = np.asarray(center, float)
    V = center[None, :] + radius * np.stack([np.cos(angles), np.sin(angles)], 1)
    E = np.roll(V, -1, axis=0) - V
    N = np.stack([E[:, 1], -E[:, 0]], 1)
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    d = np.einsum("ij,ij->i", N, V)
    return N, d


def random_polygon_angles(rng: np.random.Generator, nv: int):
    """Jittered uniform angles: sorted, max gap < pi (origin strictly inside)."""
    base = 2 * math.pi * np.arange(nv) / nv
    jit = rng.uniform(-0.25, 0.25, nv) * 2 * math.pi / nv
    return base + jit + rng.uniform(0, 2 * math.pi)


def _pack(polys):
    off = [0]
    for A, _ in polys:
        off.append(off[-1] + A.shape[0])
    A = np.concatenate([p[0] for p in polys]) if polys else np.zeros((0, 2))
    b = np.concatenate([p[1] for p in polys]) if polys else np.zeros((0,))
    return np.asarray(off, np.int32), np.ascontiguousarray(A), np.ascontiguousarray(b)


# ----------------------------------------------------------------------------
# dynamics (problem definition: the LTV model a user supplies)
# ----------------------------------------------------------------------------

def unicycle_ltv(s_bar: np.ndarray, dt: float = DT):
    """Jacobians of s' = s + f(s,u), f = dt*(v cos th, v sin th, omega, a), at (s_bar, u=0).

    Returns A [T,4,4], B [T,4,2], c [T,4] with c = s_bar + f(s_bar,0) - A s_bar.
    """
    T = s_bar.shape[0]
    A = np.tile(np.eye(4), (T, 1, 1))
    th, v = s_bar[:, 2], s_bar[:, 3]
    A[:, 0, 2] += -dt * v * np.sin(th)
    A[:, 0, 3] += dt * np.cos(th)
    A[:, 1, 2] += dt * v * np.cos(th)
    A[:, 1, 3] += dt * np.sin(th)
    B = np.zeros((T, 4, 2))
    B[:, 2, 1] = dt
    B[:, 3, 0] = dt
    f = np.stack([dt * v * np.cos(th), dt * v * np.sin(th), np.zeros(T), np.zeros(T)], 1)
    c = s_bar + f - np.einsum("tij,tj->ti", A, s_bar)
    return A, B, c


def quadrotor_lti(dt: float = DT):
    A = np.eye(7)
    for k in range(3):
        A[k, 3 + k] = dt
    B = np.zeros((7, 4))
    for k in range(3):
        B[3 + k, k] = dt
    B[6, 3] = dt
    return A[None], B[None], np.zeros((1, 7))


def _car_common(name, cfg, seed, N, iters, speed, polys_per_scene, s0=None, lane_y=0.0):
    B = len(polys_per_scene)
    part_off, part_A, part_b = _pack([box_hrep([0.0, 0.0], [2.25, 1.0])])
    flat = [p for polys in polys_per_scene for p in polys]
    M = len(polys_per_scene[0])
    obs_off, obs_C, obs_d = _pack(flat)
    t = np.arange(N + 1) * DT
    ref = np.stack([speed * t, np.full(N + 1, lane_y), np.zeros(N + 1), np.full(N + 1, speed)], 1)
    A, Bm, c = unicycle_ltv(ref[:N])
    if s0 is None:
        s0 = ref[0]
    return Scene(
        name=name, dim=2, n_scenes=B, horizon=N, n_state=4, n_ctrl=2,
        pose_model=POSE_SE2, pose_idx=np.array([0, 1, 2, 0], np.int32),
        part_off=part_off, part_A=part_A, part_b=part_b,
        n_obs=M, obs_off=obs_off, obs_C=obs_C, obs_d=obs_d,
        dyn_per_scene=0, dyn_per_time=1, dyn_A=A, dyn_B=Bm, dyn_c=c,
        Qs=np.diag([1.0, 1.0, 0.1, 0.1]), Qu=np.diag([0.1, 0.1]),
        s0=np.tile(np.asarray(s0, float), (B, 1)),
        s_ref=np.tile(ref, (B, 1, 1)),
        iters=iters, seed=seed, config=cfg,
    )


def make_c1(seed: int = 1) -> Scene:
    rng = np.random.default_rng(seed)
    y = rng.choice([-1.0, 1.0]) * rng.uniform(0.2, 1.0)
    poly = box_hrep([6.0, y], [1.0, 1.0])
    return _car_common("C1", 1, seed, N=10, iters=50, speed=8.0, polys_per_scene=[[poly]])


def make_c2(seed: int = 2) -> Scene:
    rng = np.random.default_rng(seed)
    polys = []
    for k in range(4):
        nv = int(rng.integers(4, 9))
        r = rng.uniform(1.0, 2.5)
        side = 1.0 if k % 2 == 0 else -1.0
        cx = 5.0 + 15.0 * (k + 0.5) / 4 + rng.uniform(-0.5, 0.5)
        cy = side * (3.0 - r * rng.uniform(0.3, 0.9))
        polys.append(polygon_hrep([cx, cy], r, random_polygon_angles(rng, nv)))
    return _car_common("C2", 2, seed, N=50, iters=200, speed=3.0, polys_per_scene=[polys])


def _chamfered_block(lo, hi, rng):
    """Box [lo,hi] in 3D with two yz-corners chamfered: a hexagonal prism (8 faces)."""
    A, b = box_hrep((lo + hi) / 2, (hi - lo) / 2)
    rows_A, rows_b = [A], [b]
    for sy, sz in ((1.0, 1.0), (-1.0, -1.0)):
        n = np.array([0.0, sy, sz]) / math.sqrt(2.0)
        corner = np.array([0.0, hi[1] if sy > 0 else lo[1], hi[2] if sz > 0 else lo[2]])
        cut = rng.uniform(0.1, 0.3) * min(hi[1] - lo[1], hi[2] - lo[2])
        rows_A.append(n[None])
        rows_b.append(np.array([n @ corner - cut / math.sqrt(2.0)]))
    return np.concatenate(rows_A), np.concatenate(rows_b)


def make_c3(seed: int = 3) -> Scene:
    rng = np.random.default_rng(seed)
    parts = [
        box_hrep([0.0, 0.0, 0.0], [0.15, 0.15, 0.05]),
        box_hrep([0.0, 0.0, 0.0], [0.35, 0.03, 0.03]),
        box_hrep([0.0, 0.0, 0.0], [0.03, 0.35, 0.03]),
    ]
    part_off, part_A, part_b = _pack(parts)
    N, speed, z0 = 40, 1.5, 1.0
    gy = rng.choice([-1.0, 1.0]) * rng.uniform(0.1, 0.3)
    gz = z0 + rng.choice([-1.0, 1.0]) * rng.uniform(0.1, 0.3)
    g = 0.45
    ys = [-3.0, gy - g, gy + g, 3.0]
    zs = [-0.5, gz - g, gz + g, 2.5]
    x0, x1 = 3.85, 4.15
    polys = []
    for a in range(3):
        for c in range(3):
            if a == 1 and c == 1:
                continue  # the gap
            lo = np.array([x0, ys[a], zs[c]])
            hi = np.array([x1, ys[a + 1], zs[c + 1]])
            if a != 1 and c != 1:
                polys.append(_chamfered_block(lo, hi, rng))
            else:
                polys.append(box_hrep((lo + hi) / 2, (hi - lo) / 2))
    obs_off, obs_C, obs_d = _pack(polys)
    t = np.arange(N + 1) * DT
    ref = np.zeros((N + 1, 7))
    ref[:, 0] = speed * t
    ref[:, 2] = z0
    ref[:, 3] = speed
    A, Bm, c = quadrotor_lti()
    return Scene(
        name="C3", dim=3, n_scenes=1, horizon=N, n_state=7, n_ctrl=4,
        pose_model=POSE_TRANS_YAW, pose_idx=np.array([0, 1, 2, 6], np.int32),
        part_off=part_off, part_A=part_A, part_b=part_b,
        n_obs=len(polys), obs_off=obs_off, obs_C=obs_C, obs_d=obs_d,
        dyn_per_scene=0, dyn_per_time=0, dyn_A=A, dyn_B=Bm, dyn_c=c,
        Qs=np.diag([1.0, 1.0, 1.0, 0.1, 0.1, 0.1, 0.1]), Qu=0.1 * np.eye(4),
        s0=ref[0][None].copy(), s_ref=ref[None].copy(),
        iters=100, seed=seed, config=3,
    )


def make_c4(seed: int = 4, moving: bool = False) -> Scene:
    """C4 dense traffic; moving=True (NEXT f3, config 6): the vehicles drive along +x at
    U(12, 18) m/s (the ego at 20 m/s overtakes them), the polygonal barriers stay."""
    rng = np.random.default_rng(seed)
    lanes = [-3.5, 0.0, 3.5]
    placed = {0: [], 1: [], 2: []}
    polys = []
    moves = []
    while len(polys) < 100:
        lane = int(rng.integers(0, 3))
        x = rng.uniform(0.0, 600.0)
        if lane == 1 and x < 12.0:
            continue  # keep the ego start pose free
        if any(abs(x - x2) < 6.5 for x2 in placed[lane]):
            continue
        placed[lane].append(x)
        y = lanes[lane] + rng.uniform(-0.3, 0.3)
        if rng.uniform() < 0.1:
            nv = int(rng.integers(5, 7))
            polys.append(polygon_hrep([x, y], rng.uniform(0.8, 1.2), random_polygon_angles(rng, nv)))
            moves.append(False)
        else:
            L, W = rng.uniform(4.0, 5.0), rng.uniform(1.7, 2.0)
            yaw = math.radians(rng.uniform(-3.0, 3.0))
            polys.append(box_hrep([x, y], [L / 2, W / 2], yaw))
            moves.append(True)
    if not moving:
        return _car_common("C4", 4, seed, N=60, iters=300, speed=20.0, polys_per_scene=[polys])
    # speeds drawn after the static recipe so the geometry equals C4's
    v = rng.uniform(12.0, 18.0, len(polys)) * np.asarray(moves, float)
    sc = _car_common("C4m", 6, seed, N=60, iters=300, speed=20.0, polys_per_scene=[polys])
    return dataclasses.replace(sc, obs_step=np.stack([v * DT, np.zeros_like(v)], 1))


C5_SEED_BASE = 5_000_000
C5_SCENES = 4096
C5_OBS = 200


def _c5_scene_arrays(b: int):
    """Scene b of C5: 200 convex polygons (4-8 vertices, radius U(0.5,2)) uniform in
    [0,150] x [-15,15], rejecting overlap with the start pose.  Vectorised; the draw
    order is part of the recipe.  Returns (n_rows[200], C[rows,2], d[rows])."""
    rng = np.random.default_rng(C5_SEED_BASE + b)
    K = C5_OBS
    nv = rng.integers(4, 9, K)
    r = rng.uniform(0.5, 2.0, K)
    cx = rng.uniform(0.0, 150.0, K)
    cy = rng.uniform(-15.0, 15.0, K)
    bad = np.hypot(cx, cy) < r + 3.0
    while bad.any():  # reject overlap with the start pose
        k = int(bad.sum())
        cx[bad] = rng.uniform(0.0, 150.0, k)
        cy[bad] = rng.uniform(-15.0, 15.0, k)
        bad = np.hypot(cx, cy) < r + 3.0
    jit = rng.uniform(-0.25, 0.25, (K, 8))
    rot = rng.uniform(0.0, 2 * math.pi, K)
    k = np.arange(8)[None, :]
    step = 2 * math.pi / nv[:, None]
    ang = k * step + jit * step + rot[:, None]
    V = np.stack([cx[:, None] + r[:, None] * np.cos(ang), cy[:, None] + r[:, None] * np.sin(ang)], -1)
    nxt = (k + 1) % nv[:, None]
    Vn = np.take_along_axis(V, nxt[..., None].repeat(2, -1), axis=1)
    E = Vn - V
    Nrm = np.stack([E[..., 1], -E[..., 0]], -1)
    Nrm /= np.linalg.norm(Nrm, axis=-1, keepdims=True)
    dd = np.einsum("pkj,pkj->pk", Nrm, V)
    mask = k < nv[:, None]
    return nv.astype(np.int32), Nrm[mask], dd[mask]


def make_c5(n_scenes: int | None = None, scene_ids: Sequence[int] | None = None) -> Scene:
    if scene_ids is None:
        scene_ids = range(C5_SCENES if n_scenes is None else n_scenes)
    scene_ids = list(scene_ids)
    dummy = [[(np.zeros((3, 2)), np.zeros(3))] * C5_OBS]  # placeholder geometry, replaced below
    sc = _car_common("C5", 5, C5_SEED_BASE, N=50, iters=100, speed=10.0, polys_per_scene=dummy * len(scene_ids))
    parts = [_c5_scene_arrays(b) for b in scene_ids]
    counts = np.concatenate([p[0] for p in parts])
    sc.obs_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    sc.obs_C = np.ascontiguousarray(np.concatenate([p[1] for p in parts]))
    sc.obs_d = np.ascontiguousarray(np.concatenate([p[2] for p in parts]))
    return sc


def double_integrator_lti(dt: float = DT):
    """s = (x, y, vx, vy), u = (ax, ay): x' = x + dt v, v' = v + dt a (exact, time-invariant)."""
    A = np.eye(4)
    A[0, 2] = A[1, 3] = dt
    B = np.zeros((4, 2))
    B[2, 0] = B[3, 1] = dt
    return A[None], B[None], np.zeros((1, 4))


def make_c2p(seed: int = 2) -> Scene:
    """Config 11: C2's corridor with a translating rectangle (TRANSLATION pose: R = I,
    rho = (x, y); P:197-200 with a robot that does not rotate) driven as a double
    integrator along the same 3 m/s reference."""
    sc = make_c2(seed)
    N = sc.horizon
    t = np.arange(N + 1) * DT
    ref = np.stack([3.0 * t, np.zeros(N + 1), np.full(N + 1, 3.0), np.zeros(N + 1)], 1)
    A, Bm, c = double_integrator_lti()
    return dataclasses.replace(sc, name="C2p", config=11, pose_model=POSE_TRANSLATION,
                               pose_idx=np.array([0, 1, 0, 0], np.int32), dyn_per_time=0,
                               dyn_A=A, dyn_B=Bm, dyn_c=c, Qs=np.diag([1.0, 1.0, 0.1, 0.1]),
                               s0=ref[0][None].copy(), s_ref=ref[None].copy())


def make_config(cfg: int, **kw) -> Scene:
    if cfg == 11:
        return make_c2p(**kw)
    if cfg == 12:  # C3 with the TRANSLATION pose: rho = (x, y, z), R = I (yaw left out of the pose)
        return dataclasses.replace(make_c3(**kw), name="C3p", config=12, pose_model=POSE_TRANSLATION,
                                   pose_idx=np.array([0, 1, 2, 0], np.int32))
    if cfg == 6:
        return make_c4(moving=True, **kw)
    if cfg == 7:
        return dataclasses.replace(make_c2(**kw), name="C2n", config=7, dyn_model=1)
    if cfg == 10:
        sc = make_c2(**kw)
        part_off, part_A, part_b = _pack([box_hrep([0.0, 0.0], [2.25, 1.0]), box_hrep([-5.0, 0.0], [2.5, 1.1])])
        return dataclasses.replace(sc, name="C2t", config=10, part_off=part_off, part_A=part_A, part_b=part_b,
                                   part_ctr=np.array([[0.0, 0.0], [-5.0, 0.0]]))
    if cfg == 9:
        return dataclasses.replace(make_c4(moving=True, **kw), name="C4s", config=9, sense_half=np.array([60.0, 8.0]))
    if cfg == 8:
        inf = np.inf
        return dataclasses.replace(make_c2(**kw), name="C2b", config=8, s_min=np.array([-inf, -inf, -1.2, 2.5]),
                                   s_max=np.array([inf, inf, 1.2, 3.5]), u_min=np.array([-0.5, -1.5]),
                                   u_max=np.array([0.5, 1.5]), box_rho=3.0)
    return {1: make_c1, 2: make_c2, 3: make_c3, 4: make_c4, 5: make_c5}[cfg](**kw)
