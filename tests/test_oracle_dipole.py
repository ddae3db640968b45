"""Pins for the oracle's oriented-point dipole clip (NEXT-1; PAPER.md l.238-249,
SPEC.md l.225-233 and the S:242 convention: occupied = (x - p_i).n_i <= 0)."""
import math

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import camera, ray_np, scene_from

END_SPHERE, END_NEAR, END_PLANE, END_DIPOLE = 0, 1, 2, 3


def _one(normal, r=1.0, p=(0, 0, 0)):
    sc = scene_from([p], radii=[r])
    sc.normals = np.asarray([normal], np.float32)
    return sc


def test_spec_dipole_examples():
    # plane through the centre, ray along -n through the centre, r=1 -> length 1
    sc = _one((0, 0, 1))
    Q = np.array([0.0, 0.0, 5.0]); d = np.array([0.0, 0.0, -1.0])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert hit and tout - tin == pytest.approx(1.0, abs=1e-12)
    assert k[0] == END_DIPOLE and k[1] == END_SPHERE
    # ray parallel to the plane on the inside -> the whole chord
    Q = np.array([-5.0, 0.0, -0.5]); d = np.array([1.0, 0.0, 0.0])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert tout - tin == pytest.approx(2 * math.sqrt(1 - 0.25), abs=1e-12)
    # parallel on the outside -> empty
    Q = np.array([-5.0, 0.0, 0.5])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert hit and tout <= tin


def test_complementary_halves_sum_to_full_interval():
    """L(n) + L(-n) = L(no dipole): the two half-spaces partition the cell."""
    rng = np.random.default_rng(3)
    P = rng.uniform(-1, 1, size=(30, 3))
    from scipy.spatial import cKDTree
    dk = cKDTree(P).query(P, k=9)[0][:, 8]
    r = 0.5 * dk * rng.uniform(0.8, 1.0, 30)
    base = scene_from(P, r, lists="cech")
    nrm = rng.normal(size=(30, 3))
    nrm = (nrm / np.linalg.norm(nrm, axis=1, keepdims=True)).astype(np.float32)
    a, b = base.copy(), base.copy()
    a.normals, b.normals = nrm, -nrm
    n_checked = 0
    for _ in range(150):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = rng.normal(size=3) * 0.3 - Q / 3.0; d /= np.linalg.norm(d)
        for i in range(30):
            h0, i0, o0, _ = oracle.cell_interval(base, i, Q, d, mode=oracle.O2)
            if not h0:
                continue
            _, i1, o1, _ = oracle.cell_interval(a, i, Q, d, mode=oracle.O2)
            _, i2, o2, _ = oracle.cell_interval(b, i, Q, d, mode=oracle.O2)
            L0, L1, L2 = max(0, o0 - i0), max(0, o1 - i1), max(0, o2 - i2)
            assert L1 + L2 == pytest.approx(L0, abs=1e-12)
            assert 0 <= L1 <= L0 + 1e-15
            n_checked += 1
    assert n_checked > 100


def test_single_dipole_cell_closed_form_image():
    """alpha(px) = 1 - exp(-sigma * |chord ∩ {(x-p).n <= 0}|), chord clipped by hand."""
    sig, r = 3.0, 0.3
    rgb = [0.2, 0.7, 0.4]
    nrm = np.array([0.3, -0.5, 0.8]); nrm /= np.linalg.norm(nrm)
    sc = scene_from([[0.02, 0.05, 0.1]], radii=[r], density=[sig], rgb=[rgb])
    sc.normals = nrm[None].astype(np.float32)
    cam = camera(W=40, H=36, f=120.0)
    out = oracle.render(sc, cam, mode=oracle.O1)["out"]
    p = sc.sites[0].astype(np.float64); n = sc.normals[0].astype(np.float64)
    r32 = float(np.float32(r))
    worst = 0.0
    for y in range(cam.height):
        for x in range(cam.width):
            Q, d, _ = ray_np(cam, x, y)
            c = p - Q; tc = c @ d; e = c - tc * d; h = r32 ** 2 - e @ e
            L = 0.0
            if h > 1e-8:
                t0, t1 = tc - math.sqrt(h), tc + math.sqrt(h)
                # occupied: (Q + t d - p).n <= 0
                A, B = d @ n, c @ n
                if A > 0:
                    t1 = min(t1, B / A)
                elif A < 0:
                    t0 = max(t0, B / A)
                L = max(0.0, t1 - t0)
            T = math.exp(-float(np.float32(sig)) * L)
            if h > 1e-8:
                worst = max(worst, abs(out[y, x, 3] - T))
    assert worst < 1e-12
    assert (out[..., 3] < 0.95).sum() > 30


def test_dipole_backward_matches_fd():
    """Central finite differences of the double oracle, all arrays incl. normals."""
    sc = pf_synth.make_scene("tiny", dipoles=True)
    cam = pf_synth.make_cameras("tiny")[0]
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=5)[0] * (cam.height * cam.width)
    an = oracle.backward(sc, cam, g, mode=oracle.O2)
    assert "normals" in an

    def L(s):
        rr = oracle.render(s, cam, mode=oracle.O2, signature=True)
        return float((rr["out"].reshape(-1, 4) * g.reshape(-1, 4).astype(np.float64)).sum()), rr["sig"]

    L0, sig0 = L(sc)
    rng = np.random.default_rng(9)
    for which, hrel in (("normals", 1e-5), ("sites", 1e-5), ("radii", 1e-5)):
        arr = getattr(sc, which)
        flat = an[which].reshape(-1)
        nz = np.flatnonzero(np.abs(flat) > 1e-12 * np.abs(flat).max())
        pick = rng.choice(nz, size=min(16, nz.size), replace=False)
        scale = np.abs(flat).max()
        ok = bad = 0
        for q in pick:
            i = q // (arr.shape[1] if arr.ndim == 2 else 1)
            h = hrel * (1.0 if which == "normals" else float(sc.radii[i]))
            vals = []
            for sgn in (1, -1):
                s2 = sc.copy()
                a2 = getattr(s2, which).reshape(-1)
                a2[q] = np.float32(arr.reshape(-1)[q] + sgn * h)
                Lv, sg = L(s2)
                vals.append((float(a2[q]), Lv, np.array_equal(sg, sig0)))
            if not (vals[0][2] and vals[1][2]):
                continue
            fd = (vals[0][1] - vals[1][1]) / (vals[0][0] - vals[1][0])
            if abs(fd - flat[q]) <= 2e-4 * abs(flat[q]) + 1e-7 * scale:
                ok += 1
            else:
                bad += 1
        assert ok >= 8 and bad <= 0.05 * (ok + bad) + 0.5, (which, ok, bad)


def test_dipole_modes_agree_and_theorem2():
    sc = pf_synth.make_scene("small", num_cells=1500, dipoles=True)
    cam = pf_synth.make_cameras("small", width=96, height=72)[0]
    rng = np.random.default_rng(4)
    pix = np.stack([rng.integers(0, cam.width, 200), rng.integers(0, cam.height, 200)], 1)
    r1 = oracle.render(sc, cam, mode=oracle.O1, pixels=pix)
    r3 = oracle.render(sc, cam, mode=oracle.O3, pixels=pix)
    assert np.abs(r1["out"] - r3["out"]).max() < 1e-12
    assert oracle.render(sc, cam, mode=oracle.O3)["viol"] == 0


def test_cell_stats_telescoping_and_closed_form():
    """sum_i contrib_i = sum_pixels (1 - T_final) (the weights T_k alpha_k telescope);
    single cell on the optical axis: contrib = 1 - e^{-sigma L}, normal term =
    contrib * max(n.d, 0)^2."""
    sc = pf_synth.make_scene("tiny", dipoles=True)
    cam = pf_synth.make_cameras("tiny")[0]
    st = oracle.cell_stats(sc, cam, mode=oracle.O2)
    img = oracle.render(sc, cam, mode=oracle.O2)["out"]
    assert st["contrib"].sum() == pytest.approx((1.0 - img[..., 3]).sum(), rel=1e-12)
    assert np.all(st["normal"] <= st["contrib"] + 1e-15) and st["normal"].sum() > 0
    nrm = np.array([0.0, 0.6, 0.8], np.float32)   # n.d = 0.8 > 0 on the axis
    one = _one(nrm, r=0.5)
    one.density = np.array([2.0], np.float32)
    cam1 = camera(W=3, H=3, f=50.0)            # pixel (1,1): the optical axis (+z)
    s1 = oracle.cell_stats(one, cam1, mode=oracle.O1, pixels=np.array([[1, 1]]))
    Q, d, _ = ray_np(cam1, 1, 1)
    hit, tin, tout, _ = oracle.cell_interval(one, 0, Q, d, mode=oracle.O1)
    a = 1 - math.exp(-2.0 * (tout - tin))
    assert s1["contrib"][0] == pytest.approx(a, rel=1e-12)
    nd = max(float(nrm.astype(np.float64) @ d), 0.0)
    assert nd > 0.5 and s1["normal"][0] == pytest.approx(a * nd * nd, rel=1e-12)
