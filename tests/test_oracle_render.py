"""Pins for the oracle's compositing, full-image rendering, ordering and invariances."""
import math

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import camera, ray_np, scene_from


# ---------------------------------------------------------------- compositing

def test_composite_spec_examples():
    # S:298 empty list -> (background, 1)
    out, K = oracle.composite([], [], np.zeros((0, 3)), bg=(0.2, 0.3, 0.4))
    assert np.allclose(out, [0.2, 0.3, 0.4, 1.0]) and K == 0
    # S:299 one segment sigma*l = 50 -> (c, ~0) within 1e-9
    out, K = oracle.composite([50.0], [1.0], [[0.7, 0.1, 0.3]])
    assert np.allclose(out[:3], [0.7, 0.1, 0.3], atol=1e-9) and out[3] < 1e-9
    # S:300 two segments sigma=1, l=ln 2 -> 0.5 c1 + 0.25 c2, T = 0.25
    c1, c2 = np.array([0.9, 0.2, 0.4]), np.array([0.1, 0.8, 0.6])
    out, K = oracle.composite([1.0, 1.0], [math.log(2)] * 2, [c1, c2])
    assert np.allclose(out[:3], 0.5 * c1 + 0.25 * c2, atol=1e-15)
    assert out[3] == pytest.approx(0.25, abs=1e-15) and K == 2


def test_composite_early_stop_after_threshold_segment():
    # stop after the segment that makes T < 1e-4; later segments ignored
    sig = [1.0, 1.0, 1.0]
    dt = [math.log(50.0), math.log(1000.0), 1.0]  # T: 1/50, 2e-5 -> stop
    rgb = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    out, K = oracle.composite(sig, dt, rgb, bg=(1.0, 1.0, 1.0))
    assert K == 2
    T2 = (1 / 50) * (1 / 1000)
    assert out[3] == pytest.approx(T2, rel=1e-12)
    assert out[0] == pytest.approx(1 - 1 / 50 + T2, rel=1e-12)
    assert out[1] == pytest.approx((1 / 50) * (1 - 1 / 1000) + T2, rel=1e-12)
    assert out[2] == pytest.approx(T2, rel=1e-12)


def test_composite_associativity():
    # S:313 integrating A then B over the remaining transmittance == integrating A||B
    rng = np.random.default_rng(0)
    sig = rng.uniform(0, 2, 8); dt = rng.uniform(0, 0.5, 8); rgb = rng.uniform(0, 1, (8, 3))
    full, _ = oracle.composite(sig, dt, rgb)
    a, _ = oracle.composite(sig[:3], dt[:3], rgb[:3])
    b, _ = oracle.composite(sig[3:], dt[3:], rgb[3:])
    assert np.allclose(full[:3], a[:3] + a[3] * b[:3], atol=1e-14)
    assert full[3] == pytest.approx(a[3] * b[3], rel=1e-14)


# ---------------------------------------------------------------- images

def test_single_cell_closed_form_image():
    """Single sphere: alpha(px) = 1 - exp(-2 sigma sqrt(r^2 - rho^2)); S:349 gives
    the central-ray special case ((1-e^-2) c, T=e^-2) for sigma=2, chord 1."""
    sig, r = 2.0, 0.25
    rgb = [0.3, 0.6, 0.9]
    sc = scene_from([[0.05, -0.03, 0.0]], radii=[r], density=[sig], rgb=[rgb], bg=(0.1, 0.1, 0.1))
    cam = camera(W=48, H=40, f=200.0)
    out = oracle.render(sc, cam, mode=oracle.O1)["out"]
    p = sc.sites[0].astype(np.float64)
    ref = np.zeros((cam.height, cam.width, 4))
    well = np.zeros((cam.height, cam.width), bool)   # away from the silhouette
    for y in range(cam.height):
        for x in range(cam.width):
            Q, d, tn = ray_np(cam, x, y)
            c = p - Q
            e = c - (c @ d) * d
            h = float(np.float32(r)) ** 2 - e @ e
            well[y, x] = abs(h) > 1e-6
            T = math.exp(-2 * float(np.float32(sig)) * math.sqrt(h)) if h > 0 else 1.0
            a = 1 - T
            ref[y, x, :3] = a * np.asarray(rgb, np.float32).astype(np.float64) + T * float(np.float32(0.1))
            ref[y, x, 3] = T
    assert np.abs(out - ref).max() < 1e-7          # sqrt(h) is singular at the rim
    assert np.abs(out - ref)[well].max() < 1e-12
    assert (out[..., 3] < 0.9).sum() > 50
    # S:349 / SURVEY 8(c): sigma=2, chord length 1 through the centre
    sc1 = scene_from([[0.0, 0.0, 0.0]], radii=[0.5], density=[2.0], rgb=[rgb])
    cam1 = camera(W=2, H=2, f=50.0)
    o = oracle.render(sc1, cam1, mode=oracle.O1, pixels=np.array([[0, 0]]))["out"][0]
    Q, d, _ = ray_np(cam1, 0, 0)
    rho2 = Q @ Q - (Q @ d) ** 2
    chord = 2 * math.sqrt(0.25 - rho2)
    assert o[3] == pytest.approx(math.exp(-2 * chord), rel=1e-12)


def test_modes_agree_on_tiny_and_theorem2_order():
    """O1 (all pairs) == O2 (list planes) == O3 (tile lists) on the tiny config, and
    the key (list) order equals the geometric entry order (Theorem 2)."""
    sc = pf_synth.make_scene("tiny")
    for variant in ("outside", "inside"):
        cam = pf_synth.make_cameras("tiny", variant=variant)[0]
        r1 = oracle.render(sc, cam, mode=oracle.O1, signature=True)
        r2 = oracle.render(sc, cam, mode=oracle.O2, signature=True)
        r3 = oracle.render(sc, cam, mode=oracle.O3, signature=True)
        assert np.abs(r1["out"] - r2["out"]).max() < 1e-13
        assert np.abs(r1["out"] - r3["out"]).max() < 1e-13
        assert np.array_equal(r1["sig"], r2["sig"])
        assert r3["viol"] == 0
        assert (r1["nseg"] > 0).mean() > 0.3


def test_theorem2_random_origins():
    """first-entry order of intersected cells == ascending pow(Q,p)."""
    rng = np.random.default_rng(21)
    N = 80
    P = rng.uniform(-1, 1, size=(N, 3))
    from scipy.spatial import cKDTree
    dk = cKDTree(P).query(P, k=9)[0][:, 8]
    r = 0.5 * dk * rng.uniform(0.8, 1.0, N)
    sc = scene_from(P, r, lists="cech")
    P64 = sc.sites.astype(np.float64); w64 = sc.weights.astype(np.float64)
    viol = 0; pairs = 0
    for _ in range(1500):
        Q = rng.uniform(-1.5, 1.5, 3)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        segs = []
        for i in range(N):
            hit, tin, tout, _ = oracle.cell_interval(sc, i, Q, d, mode=oracle.O2)
            if hit and tout > tin and tout > 0:
                segs.append((tin, i))
        segs.sort()
        keys = [((P64[i] - Q) ** 2).sum() - w64[i] for _, i in segs]
        for k0, k1 in zip(keys, keys[1:]):
            pairs += 1
            viol += not (k0 < k1)
    assert pairs > 500 and viol == 0


def test_weight_shift_and_scale_invariance():
    """w -> w + c leaves every power cell unchanged (P:575 argmin is shift-invariant);
    scaling p, Q, r, near by s, w by s^2 and sigma by 1/s leaves the image unchanged."""
    sc = pf_synth.make_scene("tiny")
    cam = pf_synth.make_cameras("tiny")[0]
    # weights on a 2^-20 grid so that w + 0.375 is exact in fp32
    sc.weights = (np.round(sc.weights.astype(np.float64) * 2**20) / 2**20).astype(np.float32)
    base = oracle.render(sc, cam, mode=oracle.O1)["out"]
    sh = sc.copy()
    sh.weights = (sh.weights.astype(np.float64) + 0.375).astype(np.float32)
    assert np.array_equal(sh.weights.astype(np.float64) - 0.375, sc.weights.astype(np.float64))
    # radii untouched: only the faces' offsets move, by a shift that cancels
    out = oracle.render(sh, cam, mode=oracle.O1)["out"]
    assert np.abs(out - base).max() < 1e-12
    s = 2.0  # power of two: exact in fp32
    sc2 = sc.copy()
    sc2.sites = sc.sites * s; sc2.radii = sc.radii * s; sc2.weights = sc.weights * s * s
    sc2.density = sc.density / s
    cam2 = pf_synth.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy,
                           cam.c2w.copy(), cam.near * s)
    cam2.c2w[[3, 7, 11]] *= s
    out2 = oracle.render(sc2, cam2, mode=oracle.O1)["out"]
    assert np.abs(out2 - base).max() < 1e-12


def test_small_scene_o1_equals_o3_on_pixel_subset():
    sc = pf_synth.make_scene("small", num_cells=1500)
    cam = pf_synth.make_cameras("small", width=96, height=72)[0]
    rng = np.random.default_rng(4)
    pix = np.stack([rng.integers(0, cam.width, 300), rng.integers(0, cam.height, 300)], 1)
    r1 = oracle.render(sc, cam, mode=oracle.O1, pixels=pix, signature=True)
    r3 = oracle.render(sc, cam, mode=oracle.O3, pixels=pix, signature=True)
    assert np.abs(r1["out"] - r3["out"]).max() < 1e-12
    assert np.array_equal(r1["sig"], r3["sig"])
    full = oracle.render(sc, cam, mode=oracle.O3)
    assert full["viol"] == 0
