"""Seeded synthetic inputs for the Power Foam rasterizer (shared by oracle tests,
GPU parity tests and bench.py).

This module holds NONE of the method's arithmetic: it only draws sites, radii,
densities, colours, neighbour lists (the input graph), cameras and upstream
gradients. Both the oracle (``oracle/``) and the CUDA path consume its arrays;
neither is imported here.

Recipes follow SURVEY.md §8(d) "Synthetic inputs" (restated in DESIGN.md §3):

* radii   r_i = 0.5 * u_i * d_i^(K)   (d^(K) = distance to the K-th nearest
  site, u ~ U[0.8, 1]); weights w_i = r_i^2 ("squared radius
  (also known ... as a weight)").
* neighbour lists = symmetrised K-NN, filtered to the Čech complex
  (strict overlap |p_i - p_j| < r_i + r_j) for K=16 presets.
  By SURVEY.md Lemma L3 symmetrised K-NN contains the Čech complex when
  r_i <= d_i^(K)/2, so these lists are the exact Čech complex.
* densities: sigma_i * r_i drawn per class (bimodal, PAPER.md l.239
  "bimodal density distribution"); colours U[0,1]^3.
* cameras: OpenCV axes (x right, y down, z forward), c2w row-major 3x4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Camera", "Scene", "make_scene", "make_cameras", "make_grad_out",
    "look_at", "knn_cech_lists", "PRESETS",
]


@dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    c2w: np.ndarray          # f32[12] row-major [R | Q], world-from-camera
    near: float
    model: int = 0           # 0 pinhole, 1 equidistant fisheye (NEXT-4)

    def as_tuple(self):
        return (self.width, self.height, self.fx, self.fy, self.cx, self.cy,
                [float(v) for v in np.asarray(self.c2w, np.float32).reshape(12)],
                self.near)


@dataclass
class Scene:
    sites: np.ndarray        # f32[N,3]
    weights: np.ndarray      # f32[N]
    radii: np.ndarray        # f32[N]
    density: np.ndarray      # f32[N]
    rgb: np.ndarray          # f32[N,3]
    nbr_offsets: np.ndarray  # i64[N+1]
    nbr_indices: np.ndarray  # i32[E]
    background: tuple = (0.0, 0.0, 0.0)
    name: str = ""
    meta: dict = field(default_factory=dict)
    normals: np.ndarray | None = None   # f32[N,3] dipole normals (NEXT-1), or None
    detail: "Detail | None" = None      # detail sites of the dipole faces (NEXT-2), or None

    @property
    def num_cells(self) -> int:
        return int(self.sites.shape[0])

    @property
    def num_edges(self) -> int:
        return int(self.nbr_indices.shape[0])

    def copy(self) -> "Scene":
        return Scene(self.sites.copy(), self.weights.copy(), self.radii.copy(),
                     self.density.copy(), self.rgb.copy(),
                     self.nbr_offsets.copy(), self.nbr_indices.copy(),
                     tuple(self.background), self.name, dict(self.meta),
                     None if self.normals is None else self.normals.copy(),
                     None if self.detail is None else self.detail.copy())


@dataclass
class Detail:
    """Detail sites of the dipole faces (NEXT-2)."""
    uv: np.ndarray       # f32[N,K,2] site positions in the face chart (world units)
    disp: np.ndarray     # f32[N,K] displacements along the unit normal
    sv: np.ndarray       # f32[N,K,8,3] Spherical-Voronoi radiance per axis
    axes: np.ndarray     # f32[8,3] shared unit SV axes
    gamma: float = 4.0   # SV sharpness (SPEC S:245 default)
    tau: float = 1.0     # soft-Voronoi temperature (1 / world units)

    @property
    def K(self) -> int:
        return int(self.uv.shape[1])

    def copy(self) -> "Detail":
        return Detail(self.uv.copy(), self.disp.copy(), self.sv.copy(), self.axes.copy(),
                      float(self.gamma), float(self.tau))


# --------------------------------------------------------------------------
# cameras
# --------------------------------------------------------------------------

def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """c2w (row-major 3x4, f32) for an OpenCV camera at `eye` looking at `target`."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    right = np.cross(f, np.asarray(up, np.float64))
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(f, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f], axis=1)  # columns = camera axes in world
    M = np.concatenate([R, eye[:, None]], axis=1)
    return M.astype(np.float32).reshape(12)


def _orbit(n, radius, height, az0=0.0, az_step=None, height_jitter=0.0, rng=None):
    out = []
    az_step = (2 * math.pi / n) if az_step is None else az_step
    for k in range(n):
        az = az0 + k * az_step
        h = height
        if height_jitter and rng is not None:
            h = height + rng.uniform(-height_jitter, height_jitter)
        eye = (radius * math.cos(az), radius * math.sin(az), h)
        out.append(eye)
    return out


# --------------------------------------------------------------------------
# neighbour lists (input graph)
# --------------------------------------------------------------------------

def knn_cech_lists(sites: np.ndarray, K: int, rng: np.random.Generator,
                   cech_filter: bool, u_lo: float = 0.8, u_hi: float = 1.0):
    """Radii r = 0.5*u*d^(K) and CSR neighbour lists (sym-KNN, optionally
    Čech-filtered). kd-tree in double on the fp32-rounded coordinates."""
    from scipy.spatial import cKDTree
    N = sites.shape[0]
    P = sites.astype(np.float64)
    Kq = min(K, N - 1)
    tree = cKDTree(P)
    dist, idx = tree.query(P, k=Kq + 1, workers=-1)
    dK = dist[:, Kq]
    u = rng.uniform(u_lo, u_hi, size=N)
    radii = (0.5 * u * dK).astype(np.float32)
    nb = idx[:, 1:].astype(np.int64)
    src = np.repeat(np.arange(N, dtype=np.int64), Kq)
    dst = nb.reshape(-1)
    keep = dst != src
    src, dst = src[keep], dst[keep]
    a = np.concatenate([src, dst])
    b = np.concatenate([dst, src])
    key = np.unique(a * N + b)
    a = key // N
    b = key % N
    if cech_filter:
        r64 = radii.astype(np.float64)
        d = np.linalg.norm(P[a] - P[b], axis=1)
        m = d < (r64[a] + r64[b])
        a, b = a[m], b[m]
    counts = np.bincount(a, minlength=N)
    offsets = np.zeros(N + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    return radii, offsets, b.astype(np.int32)


def directed_knn_lists(sites: np.ndarray, K: int):
    from scipy.spatial import cKDTree
    N = sites.shape[0]
    tree = cKDTree(sites.astype(np.float64))
    _, idx = tree.query(sites.astype(np.float64), k=K + 1)
    nb = idx[:, 1:].astype(np.int32)
    offsets = np.arange(0, N * K + 1, K, dtype=np.int64)
    return offsets, nb.reshape(-1)


def all_pairs_lists(N: int):
    idx = []
    for i in range(N):
        idx.extend(j for j in range(N) if j != i)
    offsets = np.arange(0, N * (N - 1) + 1, N - 1, dtype=np.int64)
    return offsets, np.asarray(idx, np.int32)


# --------------------------------------------------------------------------
# site distributions
# --------------------------------------------------------------------------

def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _object_surface(n, rng):
    """Synthetic object: sphere (r 0.6) ∪ torus (R 1.0, r 0.22) ∪ box."""
    kind = rng.choice(3, size=n, p=[0.3, 0.45, 0.25])
    pts = np.zeros((n, 3))
    m = kind == 0
    pts[m] = 0.6 * _unit(rng.normal(size=(m.sum(), 3))) + np.array([0.0, 0.0, 0.15])
    m = kind == 1
    k = m.sum()
    th = rng.uniform(0, 2 * math.pi, k)
    ph = rng.uniform(0, 2 * math.pi, k)
    R, r = 1.0, 0.22
    pts[m] = np.stack([(R + r * np.cos(ph)) * np.cos(th),
                       (R + r * np.cos(ph)) * np.sin(th),
                       r * np.sin(ph)], axis=1)
    m = kind == 2
    k = m.sum()
    half = np.array([0.45, 0.3, 0.2])
    ctr = np.array([0.0, 0.0, -0.45])
    face = rng.integers(0, 6, k)
    q = rng.uniform(-1, 1, size=(k, 3))
    ax = face // 2
    q[np.arange(k), ax] = np.where(face % 2 == 0, -1.0, 1.0)
    pts[m] = ctr + q * half
    return pts


def _densities(radii, rng, cls_p=(0.10, 0.27, 0.63), dense=(0.5, 4.0), thin=(0.01, 0.3)):
    """sigma*r bimodal: class 0 -> sigma=0, 1 -> dense, 2 -> thin."""
    N = radii.shape[0]
    cls = rng.choice(3, size=N, p=list(cls_p))
    sr = np.where(cls == 1, rng.uniform(*dense, N), rng.uniform(*thin, N))
    sr = np.where(cls == 0, 0.0, sr)
    return (sr / radii.astype(np.float64)).astype(np.float32)


def _finish(sites, radii, offsets, nbrs, rng, bg, name, density=None, meta=None):
    sites = sites.astype(np.float32)
    radii = radii.astype(np.float32)
    weights = (radii.astype(np.float32) * radii.astype(np.float32)).astype(np.float32)
    if density is None:
        density = _densities(radii, rng)
    rgb = rng.uniform(0.0, 1.0, size=(sites.shape[0], 3)).astype(np.float32)
    return Scene(sites, weights, radii, density.astype(np.float32), rgb,
                 offsets.astype(np.int64), nbrs.astype(np.int32), tuple(bg), name,
                 dict(meta or {}))


def _scene_tiny(seed, variant="sym8"):
    rng = np.random.default_rng(seed)
    N = 64
    sites = rng.uniform(-1.0, 1.0, size=(N, 3)).astype(np.float32)
    radii, offs, nbrs = knn_cech_lists(sites, 8, rng, cech_filter=False)
    sr = rng.uniform(0.5, 5.0, N)
    density = (sr / radii.astype(np.float64)).astype(np.float32)
    sc = _finish(sites, radii, offs, nbrs, rng, (0.0, 0.0, 0.0), "tiny", density)
    if variant == "knn8":
        sc.nbr_offsets, sc.nbr_indices = directed_knn_lists(sites, 8)
    elif variant == "allpairs_w0":
        sc.nbr_offsets, sc.nbr_indices = all_pairs_lists(N)
        sc.weights = np.zeros(N, np.float32)
    elif variant != "sym8":
        raise ValueError(variant)
    sc.meta["variant"] = variant
    return sc


def _scene_object(N, seed, bg, K=16, frac_obj=0.85, name="nerfsynth", cech_filter=True):
    rng = np.random.default_rng(seed)
    n_obj = int(round(frac_obj * N))
    pts = _object_surface(n_obj, rng) + rng.normal(0.0, 0.004, size=(n_obj, 3))
    box = rng.uniform(-1.5, 1.5, size=(N - n_obj, 3))
    sites = np.concatenate([pts, box]).astype(np.float32)
    sites = sites[rng.permutation(N)]
    radii, offs, nbrs = knn_cech_lists(sites, K, rng, cech_filter=cech_filter)
    return _finish(sites, radii, offs, nbrs, rng, bg, name)


def _scene_mip360(N, seed, K=16, name="mip360", cech_filter=True):
    rng = np.random.default_rng(seed)
    n_obj = int(round(0.45 * N))
    n_gnd = int(round(0.20 * N))
    n_bg = N - n_obj - n_gnd
    obj = _object_surface(n_obj, rng) + rng.normal(0.0, 0.004, size=(n_obj, 3))
    rr = 6.0 * np.sqrt(rng.uniform(0, 1, n_gnd))
    th = rng.uniform(0, 2 * math.pi, n_gnd)
    gnd = np.stack([rr * np.cos(th), rr * np.sin(th), np.full(n_gnd, -0.5)], axis=1)
    gnd += rng.normal(0.0, 0.004, size=gnd.shape)
    rad = np.exp(rng.uniform(math.log(8.0), math.log(80.0), n_bg))
    z = rng.uniform(-0.2, 1.0, n_bg)          # upper-hemisphere biased
    ph = rng.uniform(0, 2 * math.pi, n_bg)
    s = np.sqrt(np.maximum(0.0, 1 - z * z))
    shell = rad[:, None] * np.stack([s * np.cos(ph), s * np.sin(ph), z], axis=1)
    sites = np.concatenate([obj, gnd, shell]).astype(np.float32)
    cls = np.concatenate([np.zeros(n_obj, np.int8), np.ones(n_gnd, np.int8),
                          np.full(n_bg, 2, np.int8)])
    perm = rng.permutation(N)
    sites, cls = sites[perm], cls[perm]
    radii, offs, nbrs = knn_cech_lists(sites, K, rng, cech_filter=cech_filter)
    dens = _densities(radii, rng)
    m = cls == 2
    sr_bg = rng.uniform(0.01, 0.5, m.sum())
    dens[m] = (sr_bg / radii[m].astype(np.float64)).astype(np.float32)
    return _finish(sites, radii, offs, nbrs, rng, (0.0, 0.0, 0.0), name, dens)


# preset -> (scene builder, camera builder)
def _cams_tiny(variant="outside"):
    if variant == "outside":
        eye = (0.0, 0.0, -3.5)
        c2w = np.array([1, 0, 0, eye[0], 0, 1, 0, eye[1], 0, 0, 1, eye[2]], np.float32)
    elif variant == "inside":   # camera inside the foam: negative keys, straddling spheres
        c2w = look_at((0.1, -0.2, 0.05), (1.0, 0.4, 0.3))
    else:
        raise ValueError(variant)
    return [Camera(64, 64, 80.0, 80.0, 32.0, 32.0, np.asarray(c2w, np.float32), 0.05)]


def _cams_nerfsynth(n=8, W=800, H=800):
    out = []
    R, el = 4.0311, math.radians(30.0)
    for k in range(n):
        az = k * 2 * math.pi / n
        eye = (R * math.cos(el) * math.cos(az), R * math.cos(el) * math.sin(az), R * math.sin(el))
        out.append(Camera(W, H, 1111.11 * W / 800.0, 1111.11 * H / 800.0, W / 2.0, H / 2.0,
                          look_at(eye, (0, 0, 0)), 0.1))
    return out


def _cams_mip360(n=1, W=1920, H=1080, height=0.8, jitter=0.0, seed=0, az_step=None):
    rng = np.random.default_rng(1000 + seed)
    f = 1371.0 * W / 1920.0
    out = []
    for eye in _orbit(n, 4.0, height, az_step=az_step, height_jitter=jitter, rng=rng):
        out.append(Camera(W, H, f, f, W / 2.0, H / 2.0, look_at(eye, (0, 0, 0)), 0.05))
    return out


PRESETS = {
    # name: (N, description)
    "tiny": 64,
    "small": 3000,
    "nerfsynth200k": 200_000,
    "mip360_1m": 1_000_000,
    "train8_1m": 1_000_000,
    "sweep64_3m": 3_000_000,
}


def add_dipoles(sc: Scene, seed: int = 77, toward=(0.0, 0.0, 0.0)) -> Scene:
    """Oriented-point dipoles (NEXT-1): a unit normal per cell.
    Normals are random unit vectors biased away from `toward` (so most occupied
    halves face inward, as a trained surface would), seeded."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(sc.num_cells, 3))
    out = sc.sites.astype(np.float64) - np.asarray(toward, np.float64)[None, :]
    out /= np.maximum(np.linalg.norm(out, axis=1, keepdims=True), 1e-9)
    n = v / np.linalg.norm(v, axis=1, keepdims=True) + 1.5 * out
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    sc.normals = n.astype(np.float32)
    sc.meta["dipoles"] = seed
    return sc


def fibonacci_axes(n: int = 8) -> np.ndarray:
    """n unit directions on the Fibonacci sphere (the SV axes)."""
    k = np.arange(n, dtype=np.float64) + 0.5
    z = 1.0 - 2.0 * k / n
    phi = np.pi * (3.0 - np.sqrt(5.0)) * k
    rr = np.sqrt(1.0 - z * z)
    return np.stack([rr * np.cos(phi), rr * np.sin(phi), z], 1).astype(np.float32)


def add_detail(sc: Scene, K: int = 8, seed: int = 91, gamma: float = 4.0,
               tau_scale: float = 8.0, clamp_frac: float = 0.02) -> Scene:
    """Detail sites (NEXT-2) on a dipole scene.  Recipe: uv on a
    centred ring of radius r/2 at equal angles plus N(0, (0.15 r)^2)
    jitter; displacements U(-0.3 r, 0.3 r), except a `clamp_frac` share of cells
    at +-1.5 r (exercising the |delta| <= r clamp); SV values: the cell's rgb
    times U(0.6, 1.4) per (site, axis, channel), clipped to [0, 1];
    tau = tau_scale / median radius, gamma = 4."""
    if sc.normals is None:
        add_dipoles(sc)
    rng = np.random.default_rng(seed)
    N = sc.num_cells
    r = sc.radii.astype(np.float64)
    ang = 2.0 * np.pi * np.arange(K) / K
    ring = np.stack([np.cos(ang), np.sin(ang)], 1)[None] * (0.5 * r)[:, None, None]
    uv = ring + rng.normal(scale=0.15, size=(N, K, 2)) * r[:, None, None]
    disp = rng.uniform(-0.3, 0.3, size=(N, K)) * r[:, None]
    big = rng.random(N) < clamp_frac
    disp[big] = np.where(rng.random((int(big.sum()), K)) < 0.5, -1.5, 1.5) * r[big, None]
    sv = sc.rgb.astype(np.float64)[:, None, None, :] * rng.uniform(0.6, 1.4, size=(N, K, 8, 3))
    sc.detail = Detail(uv.astype(np.float32), disp.astype(np.float32),
                       np.clip(sv, 0.0, 1.0).astype(np.float32), fibonacci_axes(8),
                       float(gamma), float(np.float32(tau_scale / np.median(r))))
    sc.meta["detail"] = (K, seed)
    return sc


def make_scene(preset: str, seed: int | None = None, variant: str | None = None,
               num_cells: int | None = None, dipoles: bool = False,
               detail: int = 0) -> Scene:
    """Deterministic scene for a preset; dipoles=True adds
    seeded dipole normals (NEXT-1); detail=K adds K detail sites per face (NEXT-2)."""
    sc = _make_scene(preset, seed, variant, num_cells)
    if dipoles or detail:
        add_dipoles(sc)
    if detail:
        add_detail(sc, K=int(detail))
    return sc


def _make_scene(preset, seed, variant, num_cells):
    if preset == "tiny":
        return _scene_tiny(0 if seed is None else seed, variant or "sym8")
    # variant "knn": the unfiltered sym-16NN lists (a superset of the Čech lists by
    # Lemma L3; same sites, radii and appearance) -- the paper's extraneous-edge
    # comparison
    if variant not in (None, "cech", "knn"):
        raise ValueError(variant)
    cf = variant != "knn"
    sc = _make_scene_lists(preset, seed, num_cells, cf)
    if not cf:
        sc.meta["variant"] = "knn"
    return sc


def _make_scene_lists(preset, seed, num_cells, cf):
    if preset == "small":   # test-size nerfsynth-shaped foam
        return _scene_object(num_cells or 3000, 5 if seed is None else seed, (1.0, 1.0, 1.0),
                             name="small", cech_filter=cf)
    if preset == "small360":  # test-size mip360-shaped foam
        return _scene_mip360(num_cells or 20000, 6 if seed is None else seed, name="small360",
                             cech_filter=cf)
    if preset == "nerfsynth200k":
        return _scene_object(num_cells or 200_000, 1 if seed is None else seed, (1.0, 1.0, 1.0),
                             name=preset, cech_filter=cf)
    if preset in ("mip360_1m", "train8_1m"):
        return _scene_mip360(num_cells or 1_000_000, 2 if seed is None else seed, name=preset,
                             cech_filter=cf)
    if preset == "sweep64_3m":
        return _scene_mip360(num_cells or 3_000_000, 3 if seed is None else seed, name=preset,
                             cech_filter=cf)
    raise ValueError(f"unknown preset {preset}")


def make_cameras(preset: str, variant: str | None = None, width: int | None = None,
                 height: int | None = None, n: int | None = None) -> list:
    if preset == "tiny":
        return _cams_tiny(variant or "outside")
    if preset == "small":
        return _cams_nerfsynth(n or 2, width or 200, height or 136)
    if preset == "small360":
        return _cams_mip360(n or 2, width or 240, height or 136, az_step=math.pi / 4)
    if preset == "nerfsynth200k":
        return _cams_nerfsynth(n or 8, width or 800, height or 800)
    if preset == "mip360_1m":
        return _cams_mip360(n or 1, width or 1920, height or 1080)
    if preset == "train8_1m":
        return _cams_mip360(n or 8, width or 1920, height or 1080)
    if preset == "sweep64_3m":
        return _cams_mip360(n or 64, width or 1920, height or 1080, jitter=0.3, seed=3,
                            az_step=math.radians(5.625))
    raise ValueError(f"unknown preset {preset}")


def fisheye(cam: Camera, fov_deg: float = 200.0) -> Camera:
    """Equidistant fisheye (NEXT-4) with the same pose and image size: the
    image circle of diameter min(W, H) spans fov_deg."""
    import copy
    c = copy.deepcopy(cam)
    f = 0.5 * min(cam.width, cam.height) / math.radians(0.5 * fov_deg)
    c.fx = c.fy = float(f)
    c.cx, c.cy = cam.width / 2.0, cam.height / 2.0
    c.model = 1
    return c


def make_grad_out(num_views: int, H: int, W: int, seed: int = 11) -> np.ndarray:
    """Upstream gradient dL/d(out) ~ N(0,1)/(H*W), f32[V,H,W,4] (channel 3 = dL/dT)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal(size=(num_views, H, W, 4)) / float(H * W)
    return g.astype(np.float32)
