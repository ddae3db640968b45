"""Pins for the oracle's detail sites (NEXT-2; PAPER.md l.278-297 Eqs. svdisp and
svrad, l.326-327; SPEC.md l.185-258 tangent_frame / soft_voronoi_weights /
displacement_at / radiance_at / dipole_clip and the readings R6 of DESIGN.md)."""
import itertools
import math

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import scene_from

END_SPHERE, END_NEAR, END_PLANE, END_DIPOLE = 0, 1, 2, 3
AXES = pf_synth.fibonacci_axes(8)


def _detail_cell(normal=(0, 0, 1), r=1.0, uv=((0.0, 0.0),), disp=(0.0,), sv=None, tau=8.0,
                 gamma=4.0, axes=AXES, p=(0, 0, 0)):
    sc = scene_from([p], radii=[r])
    sc.normals = np.asarray([normal], np.float32)
    K = len(uv)
    if sv is None:
        sv = np.full((K, 8, 3), 0.5)
    sc.detail = pf_synth.Detail(np.asarray([uv], np.float32), np.asarray([disp], np.float32),
                                np.asarray([sv], np.float32), np.asarray(axes, np.float32),
                                gamma, tau)
    return sc


# ---- tangent_frame -------------------------------------------

def test_spec_tangent_frame():
    u, v, m, _ = oracle.tangent_frame([0, 0, 1])
    assert np.allclose(u, [1, 0, 0], atol=0) and np.allclose(v, [0, 1, 0], atol=0)
    u, v, m, _ = oracle.tangent_frame([0, 0, -1])
    assert abs(u @ v) < 1e-15 and np.allclose(np.cross(u, v), [0, 0, -1], atol=1e-15)
    rng = np.random.default_rng(0)
    for n in rng.normal(size=(500, 3)).astype(np.float32):
        u, v, m, k = oracle.tangent_frame(n)
        assert k == int(np.argmin(np.abs(n))) or np.abs(n)[k] == np.abs(n).min()
        for a in (u, v, m):
            assert abs(np.linalg.norm(a) - 1) < 1e-12
        assert max(abs(u @ v), abs(u @ m), abs(v @ m)) < 1e-12
        assert np.allclose(np.cross(u, v), m, atol=1e-12)          # right-handed
        assert np.allclose(m, n / np.linalg.norm(n.astype(np.float64)), atol=1e-12)
    # scale invariance: the frame depends on the direction only
    a = oracle.tangent_frame(np.float32([0.3, -2.0, 0.7]))
    b = oracle.tangent_frame(np.float32([0.6, -4.0, 1.4]))
    assert all(np.allclose(x, y, atol=1e-15) for x, y in zip(a[:3], b[:3]))


# ---- soft_voronoi_weights -------------------------------------

def test_spec_soft_voronoi():
    assert oracle.soft_voronoi([0.3, 0.1], [[1.0, 2.0]], 5.0) == pytest.approx([1.0])
    w = oracle.soft_voronoi([0.0, 0.0], [[1.0, 0.0], [0.0, -1.0]], 3.0)
    assert w == pytest.approx([0.5, 0.5], abs=1e-15)
    # hard-Voronoi limit vs a nearest-neighbour scan
    rng = np.random.default_rng(1)
    hits = 0
    for _ in range(200):
        uv = rng.uniform(-1, 1, size=(8, 2))
        q = rng.uniform(-1, 1, size=2)
        dist = np.linalg.norm(uv - q, axis=1)
        srt = np.sort(dist)
        if srt[1] - srt[0] < 0.1:
            continue
        w = oracle.soft_voronoi(q, uv, 1e6)
        onehot = np.zeros(8); onehot[np.argmin(dist)] = 1
        assert np.abs(w - onehot).max() < 1e-10
        hits += 1
    assert hits > 50


def test_soft_voronoi_invariants():
    rng = np.random.default_rng(2)
    for tau in (1e-3, 0.5, 8.0, 1e3, 1e6):
        uv = rng.uniform(-1, 1, size=(8, 2)).astype(np.float32)
        q = rng.uniform(-1, 1, size=2)
        w = oracle.soft_voronoi(q, uv, tau)
        assert abs(w.sum() - 1) < 1e-12 and (w >= 0).all() and (w <= 1).all()
        perm = rng.permutation(8)
        assert np.allclose(oracle.soft_voronoi(q, uv[perm], tau), w[perm], atol=1e-15)
        # plain definition (exp without max-subtraction) where it does not overflow
        if tau <= 8.0:
            e = np.exp(-tau * np.linalg.norm(uv.astype(np.float64) - q, axis=1))
            assert np.allclose(w, e / e.sum(), rtol=1e-13, atol=0)


# ---- displacement_at / dipole_clip ------------------------------

def _down_ray(q=(0.0, 0.0), h=5.0):
    """ray along -n (n = +z) through the chart point q of the face through p = 0"""
    return np.array([q[0], q[1], h]), np.array([0.0, 0.0, -1.0])


def test_spec_displacement_examples():
    # all d_i = 0 -> 0; all d_i = 0.3 -> 0.3 anywhere
    uv = [(0.3, 0.1), (-0.2, 0.4), (0.1, -0.5)]
    for dv, q in itertools.product((0.0, 0.3), ((0.0, 0.0), (0.4, -0.2), (5.0, 3.0))):
        sc = _detail_cell(uv=uv, disp=[dv] * 3, r=10.0)
        Q, d = _down_ray(q)
        pr = oracle.detail_probe(sc, 0, Q, d)
        assert pr["delta"] == pytest.approx(float(np.float32(dv)), abs=1e-15)
        assert np.allclose(pr["qb"], q, atol=1e-15)
    # k=2, d=(0.2,-0.2), q equidistant -> 0
    sc = _detail_cell(uv=[(0.5, 0.0), (-0.5, 0.0)], disp=[0.2, -0.2])
    pr = oracle.detail_probe(sc, 0, *_down_ray((0.0, 0.7)))
    assert abs(pr["delta"]) < 1e-15


def test_spec_dipole_clip_examples():
    # zero displacement: plane through the centre, ray along -n, r = 1 -> length 1 and
    # the surface point at the centre
    sc = _detail_cell(disp=[0.0])
    Q, d = _down_ray()
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert hit and tout - tin == pytest.approx(1.0, abs=1e-12) and k[0] == END_DIPOLE
    pr = oracle.detail_probe(sc, 0, Q, d)
    assert np.allclose(Q + pr["ts"] * d, 0.0, atol=1e-15)
    # d(x_bar) = 0.25 -> length 1.25
    sc = _detail_cell(disp=[0.25])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert tout - tin == pytest.approx(1.25, abs=1e-12)
    assert tin == pytest.approx(5.0 - 0.25, abs=1e-12)
    # parallel ray on the inside -> the whole chord, no surface point
    Q = np.array([-5.0, 0.0, -0.5]); d = np.array([1.0, 0.0, 0.0])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert tout - tin == pytest.approx(2 * math.sqrt(0.75), abs=1e-12)
    assert oracle.detail_probe(sc, 0, Q, d, t_entry=tin)["parallel"]
    Q = np.array([-5.0, 0.0, 0.5])     # parallel on the outside -> empty
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert hit and tout <= tin


def test_displacement_clamp_and_monotonicity():
    """|delta| <= r; the length is non-decreasing in d(x_bar) when n.d < 0
     and follows the hand geometry 1 + clamp(delta, -1, 1)."""
    Q, d = _down_ray()
    last = -1.0
    for dv in np.linspace(-2.0, 2.0, 41):
        sc = _detail_cell(disp=[dv])
        hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
        L = max(0.0, tout - tin)
        assert L == pytest.approx(1.0 + min(max(float(np.float32(dv)), -1.0), 1.0), abs=1e-12)
        assert L >= last - 1e-15
        last = L


def test_oblique_ray_displaced_face_hand_geometry():
    """Oblique ray: x_bar on the base face, then x on the face offset by delta along
    n, both from plane-line intersections written out here."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        uv = rng.uniform(-0.5, 0.5, size=(8, 2))
        disp = rng.uniform(-0.4, 0.4, size=8)
        sc = _detail_cell(normal=n, uv=uv, disp=disp, tau=6.0)
        n32 = sc.normals[0].astype(np.float64); m = n32 / np.linalg.norm(n32)
        u, v, _, _ = oracle.tangent_frame(sc.normals[0])
        Q = rng.normal(size=3) * 3
        d = -Q + rng.normal(size=3) * 0.2; d /= np.linalg.norm(d)
        t_bar = (-Q @ m) / (d @ m)
        xb = Q + t_bar * d
        q = np.array([xb @ u, xb @ v])
        w = oracle.soft_voronoi(q, sc.detail.uv[0], 6.0)
        delta = float(np.clip(w @ sc.detail.disp[0].astype(np.float64), -1.0, 1.0))
        t_s = (delta - Q @ m) / (d @ m)
        pr = oracle.detail_probe(sc, 0, Q, d)
        assert abs(xb @ m) < 1e-12
        assert pr["delta"] == pytest.approx(delta, abs=1e-12)
        assert pr["ts"] == pytest.approx(t_s, rel=1e-12)
        assert np.allclose(pr["qs"], [(Q + t_s * d) @ u, (Q + t_s * d) @ v], atol=1e-11)


# ---- radiance_at ----------------------------------------------

def test_spec_radiance_examples():
    # constant values (0.5, 0.2, 0.1) -> that colour for any view
    rng = np.random.default_rng(5)
    uv = rng.uniform(-0.5, 0.5, size=(8, 2))
    sv = np.broadcast_to(np.float32([0.5, 0.2, 0.1]), (8, 8, 3))
    sc = _detail_cell(uv=uv, disp=[0.0] * 8, sv=sv)
    for _ in range(20):
        Q = rng.normal(size=3) * 3; d = -Q / np.linalg.norm(Q)
        col = oracle.detail_probe(sc, 0, Q, d)["col"]
        assert np.allclose(col, np.float32([0.5, 0.2, 0.1]), atol=1e-15)
    # gamma = tau = 1e6, view along axis 3, surface point at site 1 -> v_{1,3}
    axes = AXES.astype(np.float64)
    d = axes[3] / np.linalg.norm(axes[3])
    sv = rng.uniform(0, 1, size=(8, 8, 3)).astype(np.float32)
    uv = rng.uniform(-0.5, 0.5, size=(8, 2)).astype(np.float32)
    sc = _detail_cell(uv=uv, disp=[0.0] * 8, sv=sv, tau=1e6, gamma=1e6, normal=-d)
    u, v, _, _ = oracle.tangent_frame(sc.normals[0])
    x = float(uv[1, 0]) * u + float(uv[1, 1]) * v      # the face point with chart coords s_1
    Q = x - 4.0 * d
    col = oracle.detail_probe(sc, 0, Q, d)["col"]
    assert np.allclose(col, sv[1, 3], atol=1e-9)


def test_radiance_permutation_invariance_and_hard_axis_limit():
    rng = np.random.default_rng(6)
    uv = rng.uniform(-0.5, 0.5, size=(8, 2)).astype(np.float32)
    sv = rng.uniform(0, 1, size=(8, 8, 3)).astype(np.float32)
    disp = rng.uniform(-0.3, 0.3, size=8).astype(np.float32)
    base = _detail_cell(normal=(0.2, 0.3, 0.9), uv=uv, disp=disp, sv=sv, tau=4.0)
    Q = np.array([0.3, -0.2, 4.0]); d = -Q / np.linalg.norm(Q)
    ref = oracle.detail_probe(base, 0, Q, d)
    ps, pa = rng.permutation(8), rng.permutation(8)
    sc = _detail_cell(normal=(0.2, 0.3, 0.9), uv=uv[ps], disp=disp[ps], sv=sv[ps][:, pa],
                      axes=AXES[pa], tau=4.0)
    got = oracle.detail_probe(sc, 0, Q, d)
    assert np.allclose(got["col"], ref["col"], atol=1e-14)
    assert got["delta"] == pytest.approx(ref["delta"], abs=1e-15)
    # gamma -> inf: the site colours collapse to the nearest axis' values
    sc = _detail_cell(normal=(0.2, 0.3, 0.9), uv=uv, disp=disp, sv=sv, tau=1e6, gamma=1e6)
    pr = oracle.detail_probe(sc, 0, Q, d)
    a = int(np.argmax(AXES.astype(np.float64) @ d))
    k = int(np.argmin(np.linalg.norm(uv.astype(np.float64) - pr["qs"], axis=1)))
    assert np.allclose(pr["col"], sv[k, a], atol=1e-9)


# ---- whole renders -----------------------------------------------------------

def _detail_scene(seed=0, K=8):
    sc = pf_synth.make_scene("tiny", dipoles=True)
    return pf_synth.add_detail(sc, K=K, seed=91 + seed)


def test_reduces_to_plain_dipole_scene():
    """zero displacements and view/site-independent values v_{k,a} = rgb_i give the
    plain dipole image; gradients reduce too (sum_{k,a} dL/dv = dL/drgb)."""
    sc = pf_synth.make_scene("tiny", dipoles=True)
    dt = _detail_scene()
    dt.detail.disp[:] = 0.0
    dt.detail.sv[:] = dt.rgb[:, None, None, :]
    cam = pf_synth.make_cameras("tiny")[0]
    a = oracle.render(sc, cam, mode=oracle.O2)["out"]
    b = oracle.render(dt, cam, mode=oracle.O2)["out"]
    assert np.abs(a - b).max() < 1e-12 and (a[..., 3] < 0.99).mean() > 0.05
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=3)[0]
    ga = oracle.backward(sc, cam, g, mode=oracle.O2)
    gb = oracle.backward(dt, cam, g, mode=oracle.O2)
    for k in ("sites", "weights", "radii", "density", "normals"):
        scale = np.abs(ga[k]).max()
        assert np.abs(ga[k] - gb[k]).max() <= 1e-9 * scale, k
    assert np.abs(gb["detail_sv"].sum(axis=(1, 2)) - ga["rgb"]).max() < 1e-12
    assert np.abs(gb["rgb"]).max() == 0.0


@pytest.mark.parametrize("variant", ["outside", "inside"])
def test_modes_agree_and_theorem2(variant):
    """The displaced face only shrinks a cell's (convex-cell) interval, so the
    power order of Theorem 2 still orders the segments: O1 == O2 == O3."""
    sc = _detail_scene()
    cam = pf_synth.make_cameras("tiny", variant=variant)[0]
    r1 = oracle.render(sc, cam, mode=oracle.O1, signature=True)
    r3 = oracle.render(sc, cam, mode=oracle.O3, signature=True)
    assert np.abs(r1["out"] - r3["out"]).max() < 1e-13
    assert np.array_equal(r1["sig"], r3["sig"]) and r3["viol"] == 0
    assert (r1["out"][..., 3] < 0.99).mean() > 0.05


@pytest.mark.parametrize("variant", ["inside", "outside"])
def test_backward_fd(variant):
    """Central differences of L = <g, out> w.r.t. every parameter family, where the
    active set (signature) is unchanged by the step."""
    sc = _detail_scene()
    cam = pf_synth.make_cameras("tiny", variant=variant)[0]
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=8)[0] * (cam.height * cam.width)
    an = oracle.backward(sc, cam, g, mode=oracle.O2)

    def L(s):
        rr = oracle.render(s, cam, mode=oracle.O2, signature=True)
        return float((rr["out"].reshape(-1, 4) * g.reshape(-1, 4).astype(np.float64)).sum()), rr["sig"]

    L0, sig0 = L(sc)
    rng = np.random.default_rng(3)
    fams = {"sites": (None, "sites"), "radii": (None, "radii"), "density": (None, "density"),
            "normals": (None, "normals"), "detail_uv": ("detail", "uv"),
            "detail_disp": ("detail", "disp"), "detail_sv": ("detail", "sv")}
    stats = {}
    for name, (owner, attr) in fams.items():
        get = (lambda s, a=attr: getattr(s, a)) if owner is None else \
            (lambda s, a=attr: getattr(s.detail, a))
        arr = get(sc); flat = an[name].reshape(-1)
        nz = np.flatnonzero(np.abs(flat) > 1e-6 * np.abs(flat).max())
        ok = bad = 0
        for q in rng.choice(nz, size=min(10, nz.size), replace=False):
            x0 = float(arr.reshape(-1)[q])
            i = q // (arr.size // sc.num_cells)
            scale = 1.0 if name in ("density", "detail_sv") else float(sc.radii[i])
            h = 1e-5 * max(scale, abs(x0) if name == "density" else 0.0)
            vals = []
            for sgn in (1, -1):
                s2 = sc.copy(); a2 = get(s2).reshape(-1)
                a2[q] = np.float32(x0 + sgn * h)
                Lv, sg = L(s2)
                vals.append((float(a2[q]), Lv, np.array_equal(sg, sig0)))
            if not (vals[0][2] and vals[1][2]):
                continue
            fd = (vals[0][1] - vals[1][1]) / (vals[0][0] - vals[1][0])
            if abs(fd - flat[q]) <= 2e-4 * abs(flat[q]) + 1e-7 * np.abs(flat).max():
                ok += 1
            else:
                bad += 1
                print(name, q, fd, flat[q])
        stats[name] = (ok, bad)
    assert all(b == 0 for _, b in stats.values()), stats
    assert all(o >= 5 for o, _ in stats.values()), stats


def test_saturated_displacement():
    """|delta| <= r: a face displaced to +r is tangent to the sphere (the
    whole bounded cell is occupied), one at -r leaves nothing."""
    base = _detail_scene()
    full = base.copy(); full.detail.disp[:] = 1.5 * full.radii[:, None]
    none = base.copy(); none.detail.disp[:] = -1.5 * none.radii[:, None]
    plain = base.copy(); plain.normals = None; plain.detail = None
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(40):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = -Q / 3.0 + rng.normal(size=3) * 0.2; d /= np.linalg.norm(d)
        for i in range(base.num_cells):
            h0, i0, o0, _ = oracle.cell_interval(plain, i, Q, d, mode=oracle.O2)
            if not h0 or o0 <= i0:
                continue
            _, i1, o1, _ = oracle.cell_interval(full, i, Q, d, mode=oracle.O2)
            _, i2, o2, _ = oracle.cell_interval(none, i, Q, d, mode=oracle.O2)
            assert (i1, o1) == pytest.approx((i0, o0), abs=1e-12)
            assert o2 - i2 <= 1e-12
            checked += 1
    assert checked > 100
    cam = pf_synth.make_cameras("tiny")[0]
    out = oracle.render(none, cam, mode=oracle.O2)["out"]
    assert np.abs(out[..., 3] - 1.0).max() < 1e-9
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=9)[0]
    an = oracle.backward(full, cam, g, mode=oracle.O2)
    assert np.abs(an["detail_disp"]).max() == 0.0   # saturated: no displacement gradient
    assert np.abs(an["detail_sv"]).max() > 0.0
