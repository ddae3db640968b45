"""Pins for the oracle's equidistant-fisheye rasterization (NEXT-4; PAPER.md
l.699-709 "lossless non-pinhole rasterization")."""
import math

import numpy as np
import pytest

import oracle
import pf_synth


def _fish(cam, fov=200.0):
    return pf_synth.fisheye(cam, fov)


def _expected_dir(cam, x, y):
    """Independent numpy restatement of S:285 (equidistant: angle = |(a,b)|)."""
    f32 = lambda v: float(np.float32(v))
    a = (x + 0.5 - f32(cam.cx)) / f32(cam.fx); b = (y + 0.5 - f32(cam.cy)) / f32(cam.fy)
    th = math.hypot(a, b)
    dc = np.array([math.sin(th) * a / th, math.sin(th) * b / th, math.cos(th)]) if th > 0 \
        else np.array([0.0, 0.0, 1.0])
    M = np.asarray(cam.c2w, np.float32).astype(np.float64).reshape(3, 4)
    d = M[:, :3] @ dc
    return d / np.linalg.norm(d), th


def test_spec_fisheye_rays():
    cam = pf_synth.Camera(64, 64, 20.0, 20.0, 0.5, 31.5,
                          pf_synth.look_at((0, 0, -3), (0.2, 0.1, 0)), 0.05, 1)
    axis = np.asarray(cam.c2w, np.float64).reshape(3, 4)[:, 2]
    # the pixel whose centre is the principal point -> the optical axis
    Q, d, tn = oracle.pixel_ray(cam, 0, 31)
    assert np.abs(d - axis / np.linalg.norm(axis)).max() < 1e-7
    assert tn == pytest.approx(cam.near)            # fisheye near = distance (reading R5)
    # rho = f pi/2 -> perpendicular to the optical axis (pixel centre at u = 0.5 + f pi/2
    # is not on the grid; check the model on grid pixels and the angle law instead)
    for x in (0, 10, 31, 40, 60):   # theta <= pi (inside the image circle)
        Q, d, _ = oracle.pixel_ray(cam, x, 31)
        e, th = _expected_dir(cam, x, 31)
        assert np.abs(d - e).max() < 1e-14
        assert math.acos(max(-1.0, min(1.0, d @ (axis / np.linalg.norm(axis))))) == \
            pytest.approx(th, abs=1e-6)
        assert np.linalg.norm(d) == pytest.approx(1.0, abs=1e-14)
    # x = 31: u - cx = 31 = f * 1.55 rad ~ pi/2 -> nearly perpendicular
    Q, d, _ = oracle.pixel_ray(cam, 31, 31)
    assert abs(d @ (axis / np.linalg.norm(axis)) - math.cos(31.0 / 20.0)) < 1e-6


def test_pinhole_and_fisheye_agree_on_the_axis():
    """the optical-axis ray is the same for both models."""
    sc = pf_synth.make_scene("tiny")
    pin = pf_synth.Camera(65, 65, 80.0, 80.0, 32.5, 32.5,
                          pf_synth.make_cameras("tiny")[0].c2w.copy(), 0.05, 0)
    fish = pf_synth.Camera(65, 65, 30.0, 30.0, 32.5, 32.5, pin.c2w.copy(), 0.05, 1)
    a = oracle.render(sc, pin, mode=oracle.O1, pixels=np.array([[32, 32]]))["out"][0]
    b = oracle.render(sc, fish, mode=oracle.O1, pixels=np.array([[32, 32]]))["out"][0]
    # same ray; near differs only by |d_cam| = 1 on the axis
    assert np.abs(a - b).max() < 1e-14


def test_fisheye_binning_conservative_brute_force():
    rng = np.random.default_rng(2)
    sc = pf_synth.make_scene("tiny")
    cam = _fish(pf_synth.Camera(96, 80, 1, 1, 0, 0, pf_synth.look_at((0.3, -0.2, 0.1), (1, 0.5, 0.2)),
                                0.05), 220.0)
    b = oracle.binning(sc, cam)
    tiles = (b["keys"] >> np.uint64(32)).astype(np.int64)
    per_cell = {}
    for t, v in zip(tiles, b["vals"]):
        per_cell.setdefault(int(v), set()).add(int(t))
    P = sc.sites.astype(np.float64); r = sc.radii.astype(np.float64)
    checked = 0
    for y in range(cam.height):
        for x in range(cam.width):
            Q, d, tn = oracle.pixel_ray(cam, x, y)
            a_ = (x + 0.5 - cam.cx) / cam.fx; b_ = (y + 0.5 - cam.cy) / cam.fy
            if math.hypot(a_, b_) > math.pi:
                continue
            t = (y // 16) * b["tiles_x"] + x // 16
            for i in range(sc.num_cells):
                c = P[i] - Q; tc = c @ d; e = c - tc * d; h = r[i] ** 2 - e @ e
                if h > 0 and tc + math.sqrt(h) > tn:
                    assert t in per_cell.get(i, set()), (i, x, y)
                    checked += 1
    assert checked > 3000


@pytest.mark.parametrize("variant", ["outside", "inside"])
def test_fisheye_modes_agree_and_theorem2(variant):
    """the power order is valid for any ray through Q, so tile
    rasterization is lossless for the fisheye: O1 (definition) == O3 (tiles)."""
    sc = pf_synth.make_scene("tiny")
    cam = _fish(pf_synth.make_cameras("tiny", variant=variant)[0], 200.0)
    r1 = oracle.render(sc, cam, mode=oracle.O1, signature=True)
    r3 = oracle.render(sc, cam, mode=oracle.O3, signature=True)
    assert np.abs(r1["out"] - r3["out"]).max() < 1e-13
    assert np.array_equal(r1["sig"], r3["sig"]) and r3["viol"] == 0
    assert (r1["out"][..., 3] < 0.99).mean() > 0.03


def test_fisheye_backward_fd():
    sc = pf_synth.make_scene("tiny")
    cam = _fish(pf_synth.make_cameras("tiny", variant="inside")[0], 180.0)
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=8)[0] * (cam.height * cam.width)
    an = oracle.backward(sc, cam, g, mode=oracle.O2)

    def L(s):
        rr = oracle.render(s, cam, mode=oracle.O2, signature=True)
        return float((rr["out"].reshape(-1, 4) * g.reshape(-1, 4).astype(np.float64)).sum()), rr["sig"]

    L0, sig0 = L(sc)
    rng = np.random.default_rng(3)
    ok = bad = 0
    for which in ("sites", "radii", "density"):
        arr = getattr(sc, which); flat = an[which].reshape(-1)
        nz = np.flatnonzero(np.abs(flat) > 0)
        for q in rng.choice(nz, size=min(8, nz.size), replace=False):
            i = q // (arr.shape[1] if arr.ndim == 2 else 1)
            h = 1e-5 * (float(sc.radii[i]) if which != "density" else max(float(sc.density[i]), 1.0))
            vals = []
            for sgn in (1, -1):
                s2 = sc.copy(); a2 = getattr(s2, which).reshape(-1)
                a2[q] = np.float32(arr.reshape(-1)[q] + sgn * h)
                Lv, sg = L(s2)
                vals.append((float(a2[q]), Lv, np.array_equal(sg, sig0)))
            if not (vals[0][2] and vals[1][2]):
                continue
            fd = (vals[0][1] - vals[1][1]) / (vals[0][0] - vals[1][0])
            if abs(fd - flat[q]) <= 2e-4 * abs(flat[q]) + 1e-7 * np.abs(flat).max():
                ok += 1
            else:
                bad += 1
    assert ok >= 15 and bad == 0, (ok, bad)
