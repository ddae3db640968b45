"""Pins for the oracle's interval geometry (oracle/pf_oracle.c: cell_interval).

Each test names the passage whose value / property it checks.
"""
import math

import numpy as np
import pytest

import oracle
from helpers import argmin_power_sampler, scene_from

END_SPHERE, END_NEAR, END_PLANE = 0, 1, 2


@pytest.mark.parametrize("wa,wb,x_plane", [
    (1.0, 1.0, 2.0),     # S:66 equal radii -> midplane x=2
    (4.0, 0.0, 2.5),     # S:67 r_a=2, r_b=0 -> x=2.5 (paper's printed sign gives 1.5)
    (0.0, 36.0, -2.5),   # S:68 r_a=0, r_b=6 -> x=-2.5, outside both spheres
])
def test_radical_plane_spec_examples(wa, wb, x_plane):
    # weights from the SPEC example; extent radii large so the plane is exposed
    sc = scene_from([[0, 0, 0], [4, 0, 0]], radii=[10.0, 10.0], weights=[wa, wb])
    Q = np.array([-20.0, 0.0, 0.0]); d = np.array([1.0, 0.0, 0.0])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
    assert hit and k[1] == END_PLANE and k[3] == 1
    assert tout - 20.0 == pytest.approx(x_plane, abs=1e-12)
    hit, tin, tout, k = oracle.cell_interval(sc, 1, Q, d, mode=oracle.O1)
    assert hit and k[0] == END_PLANE and k[2] == 0
    assert tin - 20.0 == pytest.approx(x_plane, abs=1e-12)


def test_radical_plane_two_balls_closed_form():
    # two balls on an axis: face at x* = (D^2 + w1 - w2) / (2D)   (P:577-585 corrected)
    rng = np.random.default_rng(3)
    for _ in range(50):
        D = rng.uniform(0.5, 3.0)
        w1, w2 = rng.uniform(0, 4, 2)
        sc = scene_from([[0, 0, 0], [D, 0, 0]], radii=[50.0, 50.0], weights=[w1, w2])
        D32 = float(np.float32(D)); w1f, w2f = (float(np.float32(v)) for v in (w1, w2))
        xs = (D32 ** 2 + w1f - w2f) / (2 * D32)
        Q = np.array([-60.0, 0.0, 0.0]); d = np.array([1.0, 0.0, 0.0])
        _, _, tout, k = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
        assert k[1] == END_PLANE
        assert tout - 60.0 == pytest.approx(xs, abs=1e-10)


def test_chord_through_centre_and_off_centre():
    # S:116 single cell, ray through centre, r=1 -> length 2; off-centre 2 sqrt(r^2-rho^2)
    sc = scene_from([[0.3, -0.2, 5.0]], radii=[1.0])
    Q = np.zeros(3)
    for rho in [0.0, 0.1, 0.5, 0.9, 0.999]:
        target = np.array([0.3 + rho, -0.2, 5.0])
        d = target / np.linalg.norm(target)
        # distance of the centre from the ray
        c = np.array([0.3, -0.2, 5.0], np.float32).astype(np.float64)
        e = c - (c @ d) * d
        rr = np.linalg.norm(e)
        hit, tin, tout, _ = oracle.cell_interval(sc, 0, Q, d, mode=oracle.O1)
        assert hit
        assert tout - tin == pytest.approx(2 * math.sqrt(1 - rr * rr), rel=1e-12)
    # S:117 miss
    hit, *_ = oracle.cell_interval(sc, 0, Q, np.array([0.0, 1.0, 0.0]), mode=oracle.O1)
    assert not hit


def test_near_plane_clips_entry():
    sc = scene_from([[0, 0, 0]], radii=[1.0])
    Q = np.array([0.0, 0.0, -0.5]); d = np.array([0.0, 0.0, 1.0])
    hit, tin, tout, k = oracle.cell_interval(sc, 0, Q, d, t_near=0.2, mode=oracle.O1)
    assert hit and k[0] == END_NEAR and tin == pytest.approx(0.2) and tout == pytest.approx(1.5)
    # sphere entirely before t_near -> no hit
    hit, *_ = oracle.cell_interval(sc, 0, Q, d, t_near=1.6, mode=oracle.O1)
    assert not hit


def _random_foam(rng, N, w_mode="r2"):
    P = rng.uniform(-1, 1, size=(N, 3))
    from scipy.spatial import cKDTree
    dk = cKDTree(P).query(P, k=9)[0][:, 8]
    r = 0.5 * rng.uniform(0.8, 1.0, N) * dk * (2.0 if w_mode == "zero" else 1.0)
    w = r * r if w_mode == "r2" else np.zeros(N)
    return P, r, w


@pytest.mark.parametrize("w_mode", ["r2", "zero"])
def test_intervals_vs_fine_step_argmin_sampler(w_mode):
    """interval endpoints vs fine-step argmin-power sampling (brute force).
    w_mode='zero' is the Voronoi reduction (P:575 'When all weights are equal ...')."""
    rng = np.random.default_rng(7 if w_mode == "r2" else 8)
    N = 30
    P, r, w = _random_foam(rng, N, w_mode)
    sc = scene_from(P, r, weights=w, lists="all")
    dt = 1e-3
    ts = np.arange(0.0, 8.0, dt)
    n_checked = 0
    for _ in range(60):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = rng.normal(size=3) * 0.3 - Q / 3.0; d /= np.linalg.norm(d)
        lab, _ = argmin_power_sampler(sc, Q, d, ts)
        ref = np.full(ts.shape, -1)
        ends = []
        for i in range(N):
            hit, tin, tout, _ = oracle.cell_interval(sc, i, Q, d, mode=oracle.O1)
            if hit and tout > tin:
                ref[(ts > tin) & (ts < tout)] = i
                ends += [tin, tout]
        ends = np.asarray(ends)
        far = np.ones(ts.shape, bool)
        for t in ends:
            far &= np.abs(ts - t) > 2 * dt
        n_checked += far.sum()
        assert np.array_equal(lab[far], ref[far])
    assert n_checked > 10000


def test_partition_sum_dt_equals_union_length():
    """SURVEY Lemma L2 (w = r^2): bounded cells tile the union of balls, so along a
    ray the interval lengths sum to |ray ∩ ∪B| and the intervals are disjoint."""
    rng = np.random.default_rng(11)
    P, r, w = _random_foam(rng, 40)
    sc = scene_from(P, r, lists="cech")
    for _ in range(200):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = rng.normal(size=3) * 0.3 - Q / 3.0; d /= np.linalg.norm(d)
        ivs = []
        for i in range(sc.num_cells):
            hit, tin, tout, _ = oracle.cell_interval(sc, i, Q, d, mode=oracle.O2)
            if hit and tout > tin:
                ivs.append((tin, tout))
        # union of sphere chords, computed directly
        chords = []
        P64 = sc.sites.astype(np.float64); r64 = sc.radii.astype(np.float64)
        for i in range(sc.num_cells):
            c = P64[i] - Q; tc = c @ d; h = r64[i] ** 2 - (c @ c - tc * tc)
            if h > 0:
                chords.append((tc - math.sqrt(h), tc + math.sqrt(h)))
        chords.sort()
        union = 0.0; cur = None
        for a, b in chords:
            a = max(a, 0.0)
            if b <= a:
                continue
            if cur is None or a > cur[1]:
                if cur: union += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur: union += cur[1] - cur[0]
        total = sum(b - a for a, b in ivs)
        assert total == pytest.approx(union, abs=1e-9)
        ivs.sort()
        for (a0, b0), (a1, b1) in zip(ivs, ivs[1:]):
            assert a1 >= b0 - 1e-9


def test_cech_lists_equal_all_pairs():
    """P:235 / Fig. 5: Čech-superset lists give the exact intervals (Lemma L1)."""
    rng = np.random.default_rng(12)
    P, r, w = _random_foam(rng, 40)
    sc = scene_from(P, r, lists="cech")
    for _ in range(100):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = rng.normal(size=3) * 0.3 - Q / 3.0; d /= np.linalg.norm(d)
        for i in range(sc.num_cells):
            a = oracle.cell_interval(sc, i, Q, d, mode=oracle.O1)
            b = oracle.cell_interval(sc, i, Q, d, mode=oracle.O2)
            assert a[0] == b[0]
            if a[0]:
                la, lb = max(0, a[2] - a[1]), max(0, b[2] - b[1])
                assert la == pytest.approx(lb, abs=1e-12)


def test_voronoi_nonlocal_faces_need_all_pairs():
    """P:191/P:198 (Fig. 4): with w = 0 (bounded Voronoi) Čech lists are NOT
    sufficient -- some cells differ from the all-pairs result."""
    rng = np.random.default_rng(13)
    N = 60
    P = rng.uniform(-1, 1, size=(N, 3))
    from scipy.spatial import cKDTree
    dk = cKDTree(P).query(P, k=9)[0][:, 8]
    r = dk * rng.uniform(0.1, 1.0, N)
    sc_c = scene_from(P, r, weights=np.zeros(N), lists="cech")
    diff = 0
    for _ in range(300):
        Q = rng.normal(size=3); Q = 3.0 * Q / np.linalg.norm(Q)
        d = rng.normal(size=3) * 0.3 - Q / 3.0; d /= np.linalg.norm(d)
        for i in range(N):
            a = oracle.cell_interval(sc_c, i, Q, d, mode=oracle.O1)
            b = oracle.cell_interval(sc_c, i, Q, d, mode=oracle.O2)
            if a[0] and abs(max(0, a[2] - a[1]) - max(0, b[2] - b[1])) > 1e-9:
                diff += 1
    assert diff > 0
