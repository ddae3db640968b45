"""Pins for the oracle's per-pixel work counters X_s, X_h, X_p, X_c.

The counters define the algorithmic flops of the roofline (F_fwd = 8 X_s + 14 X_h
+ 16 X_p + 15 X_c), so they are pinned against values derived WITHOUT the oracle:

* a hand-built single-tile scene (axis-aligned, pairwise disjoint spheres, two
  "ghost" cells whose power cells are empty, one small off-axis sphere that only
  part of the tile's rays meet) whose counters follow in closed form from the
  ray-point distance, the chord length 2 sqrt(r^2 - rho^2) and the
  termination rule (stop after the segment that makes T < 1e-4);
* an independent numpy brute-force walk of the tiny scene's tile lists that
  computes the intervals with the cell-local formula of SURVEY App. A
  (a t' <= b), not the oracle's absolute-t form, and composites in numpy.

Definitions (oracle/pf_oracle.c `pixel_counters`): walking the
pixel's tile list in key order up to and including the entry of the terminating
segment (the whole list if the pixel never terminates), X_s = entries examined,
X_h = entries whose bounding sphere the ray meets beyond the near plane, X_p =
the list planes of those hits (each evaluated once), X_c = composited segments.
"""
import math

import numpy as np
import pytest

import oracle
from helpers import camera, ray_np, scene_from

LN_STOP = math.log(1e4)   # T < 1e-4  <=>  sum tau > ln(1e4)


def _hand_scene(sigma_axis):
    """8 axis spheres (r = 0.4, centres 1.2 apart: disjoint, so every radical
    plane separates them and no chord is clipped), ghosts of cells 1 and 4 (same
    site and radius, weight r^2 - 0.05: pow_ghost = pow_host + 0.05 everywhere, so
    the ghost's power cell is empty while its sphere is hit), and a small sphere
    (r = 0.15) in the gap between cells 1 and 2, off the axis."""
    z = [-2.0 + 1.2 * k for k in range(8)]
    sites = [[0.0, 0.0, zk] for zk in z]
    radii = [0.4] * 8
    weights = [0.16] * 8
    sig = [sigma_axis] * 8
    for host in (1, 4):
        sites.append(list(sites[host]))
        radii.append(0.4)
        weights.append(0.16 - 0.05)
        sig.append(sigma_axis)
    sites.append([0.1, 0.0, -0.2])
    radii.append(0.15)
    weights.append(0.15 ** 2)
    sig.append(2.5)
    N = len(sites)
    rgb = np.linspace(0.1, 0.9, 3 * N).reshape(N, 3)
    return scene_from(sites, radii, weights=weights, density=sig, rgb=rgb, lists="all")


def _hand_expected(sc, cam):
    """Closed-form counters of every pixel of the 16x16 single-tile image."""
    P = sc.sites.astype(np.float64)
    r = sc.radii.astype(np.float64)
    w = sc.weights.astype(np.float64)
    N = sc.num_cells
    ghosts = {8, 9}
    exp = np.zeros((16, 16, 4), np.int64)
    margin = np.inf
    for y in range(16):
        for x in range(16):
            Q, d, tn = ray_np(cam, x, y)
            key = ((P - Q) ** 2).sum(1) - w            # Theorem 2 order
            order = sorted(range(N), key=lambda i: (key[i], i))
            tau_sum, xs, xh, xp, xc = 0.0, 0, 0, 0, 0
            for i in order:
                xs += 1
                c = P[i] - Q
                rho2 = c @ c - (c @ d) ** 2            # squared ray-site distance
                h = r[i] ** 2 - rho2
                margin = min(margin, abs(h) / r[i] ** 2)
                if h <= 0 or (c @ d) + math.sqrt(h) <= tn:
                    continue
                xh += 1
                xp += N - 1                            # all-pairs lists
                if i in ghosts:
                    continue                           # empty power cell: no segment
                xc += 1
                tau_sum += sc.density[i] * 2.0 * math.sqrt(h)   # full chord
                margin = min(margin, abs(tau_sum - LN_STOP))
                if tau_sum > LN_STOP:
                    break
            exp[y, x] = (xs, xh, xp, xc)
    return exp, margin


@pytest.mark.parametrize("sigma_axis,terminates", [(2.9, True), (0.1, False)])
def test_counters_hand_built_single_tile(sigma_axis, terminates):
    sc = _hand_scene(sigma_axis)
    cam = camera(W=16, H=16, f=400.0)
    exp, margin = _hand_expected(sc, cam)
    assert margin > 1e-6            # no pixel sits on a hit or termination boundary
    # the tile list is every cell in key order (all spheres project into the tile)
    b = oracle.binning(sc, cam)
    key = ((sc.sites.astype(np.float64) - ray_np(cam, 0, 0)[0]) ** 2).sum(1) - sc.weights
    assert list(b["vals"]) == sorted(range(sc.num_cells), key=lambda i: (key[i], i))
    got = oracle.render(sc, cam, mode=oracle.O3, counters=True)["counters"].reshape(16, 16, 4)
    np.testing.assert_array_equal(got, exp)
    # the scene exercises every counter distinction
    assert (exp[..., 0] > exp[..., 1]).any() and (exp[..., 0] == exp[..., 1]).any()  # misses
    assert (exp[..., 1] > exp[..., 3]).all()                                         # ghosts
    assert (exp[..., 2] == 10 * exp[..., 1]).all()
    if terminates:
        assert (exp[..., 0] < sc.num_cells).all() and len(np.unique(exp[..., 3])) >= 1
    else:
        assert (exp[..., 0] == sc.num_cells).all()


def test_counters_hand_built_termination_index():
    """On the axis every chord is 2r = 0.8, so with sigma = 2.9 the k-th axis segment
    brings sum tau to 2.32 k: the 4th crosses ln(1e4) = 9.21 -> the central pixels
    composite exactly 4 segments (+ the off-axis sphere when the ray meets it),
    examining the ghost of cell 1 on the way (X_s = X_h = 5 or 6)."""
    sc = _hand_scene(2.9)
    cam = camera(W=16, H=16, f=400.0)
    got = oracle.render(sc, cam, mode=oracle.O3, counters=True)["counters"].reshape(16, 16, 4)
    c = got[8, 8]
    assert c[3] in (4, 5)
    assert c[0] == c[3] + 1 and c[1] == c[0] and c[2] == 10 * c[1]


def _numpy_counters(sc, cam, b):
    """Independent walk of the oracle's (separately pinned) tile lists: intervals by
    the cell-local formula of SURVEY App. A, compositing in numpy."""
    P = sc.sites.astype(np.float64)
    r = sc.radii.astype(np.float64)
    w = sc.weights.astype(np.float64)
    off, idx = sc.nbr_offsets, sc.nbr_indices
    H, W = cam.height, cam.width
    out = np.zeros((H, W, 4), np.int64)
    amb = np.zeros((H, W), bool)
    for y in range(H):
        for x in range(W):
            Q, d, tn = ray_np(cam, x, y)
            t = (y // 16) * b["tiles_x"] + (x // 16)
            lst = b["vals"][b["ranges"][t, 0]:b["ranges"][t, 1]]
            segs = []        # (t_in, cell, list position, dt)
            hits = []        # list positions of sphere hits
            nplanes = []
            for pos, i in enumerate(lst):
                c = P[i] - Q
                tc = c @ d
                e = c - tc * d
                h = r[i] ** 2 - e @ e
                if abs(h) < 1e-9 * r[i] ** 2:
                    amb[y, x] = True
                if h <= 0:
                    continue
                s = math.sqrt(h)
                if tc + s <= tn:
                    continue
                hits.append(pos)
                js = [j for j in idx[off[i]:off[i + 1]] if j != i]
                nplanes.append(len(js))
                lo, hi, empty = max(-s, tn - tc), s, False
                for j in js:
                    n = P[j] - P[i]
                    a = d @ n
                    bb = 0.5 * (n @ n - (w[j] - w[i])) + n @ e
                    if a > 0:
                        hi = min(hi, bb / a)
                    elif a < 0:
                        lo = max(lo, bb / a)
                    elif bb < 0:
                        empty = True
                if not empty and hi > lo:
                    if hi - lo < 1e-12:
                        amb[y, x] = True
                    segs.append((tc + lo, int(i), pos, hi - lo))
            segs.sort()
            Tsum, xc, last = 0.0, 0, len(lst) - 1
            for (_, i, pos, dt) in segs:
                xc += 1
                Tsum += float(sc.density[i]) * dt
                if abs(Tsum - LN_STOP) < 1e-9:
                    amb[y, x] = True
                if Tsum > LN_STOP:
                    last = pos
                    break
            xh = sum(1 for p in hits if p <= last)
            xp = sum(n for p, n in zip(hits, nplanes) if p <= last)
            out[y, x] = (last + 1, xh, xp, xc)
    return out, amb


@pytest.mark.slow
def test_counters_tiny_numpy_brute_force():
    import pf_synth
    sc = pf_synth.make_scene("tiny")
    cam = pf_synth.make_cameras("tiny")[0]
    b = oracle.binning(sc, cam)
    exp, amb = _numpy_counters(sc, cam, b)
    got = oracle.render(sc, cam, mode=oracle.O3, counters=True)["counters"].reshape(exp.shape)
    assert amb.sum() <= 4
    ok = ~amb
    np.testing.assert_array_equal(got[ok], exp[ok])
    assert exp[..., 3].max() > 1 and exp[..., 2].sum() > exp[..., 1].sum() > 0
