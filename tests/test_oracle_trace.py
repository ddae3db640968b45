"""Pins for the oracle's adjacency-walk ray tracer (NEXT-4; P:157-159, P:210,
reading R7 of DESIGN.md): the walk must reproduce the image of the plain
definition (O1, every cell and every plane), visit exactly the argmin-power cells
a fine-step sampler sees along the ray, and count its steps as the
construction fixes them on hand-built scenes."""
import math

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import argmin_power_sampler, camera, ray_np, scene_from


@pytest.mark.parametrize("variant", ["outside", "inside"])
def test_trace_equals_definition_tiny(variant):
    sc = pf_synth.make_scene("tiny")
    cam = pf_synth.make_cameras("tiny", variant=variant)[0]
    t = oracle.trace(sc, cam)
    o1 = oracle.render(sc, cam, mode=oracle.O1)["out"]
    assert np.abs(t["out"] - o1).max() <= 1e-12
    st = t["stats"].reshape(-1, 3)
    assert (st[:, 0] >= st[:, 2]).all() and (st[:, 1] >= 1).all()


def test_trace_equals_definition_fisheye_dipoles_detail():
    sc = pf_synth.make_scene("tiny")
    cam = pf_synth.fisheye(pf_synth.make_cameras("tiny")[0], 200.0)
    assert np.abs(oracle.trace(sc, cam)["out"] -
                  oracle.render(sc, cam, mode=oracle.O1)["out"]).max() <= 1e-12
    sd = pf_synth.make_scene("tiny", detail=3)
    cam = pf_synth.make_cameras("tiny")[0]
    assert np.abs(oracle.trace(sd, cam)["out"] -
                  oracle.render(sd, cam, mode=oracle.O1)["out"]).max() <= 1e-12
    sp = pf_synth.add_dipoles(pf_synth.make_scene("tiny"))
    assert np.abs(oracle.trace(sp, cam)["out"] -
                  oracle.render(sp, cam, mode=oracle.O1)["out"]).max() <= 1e-12


def test_trace_equals_tile_rasterizer_small360():
    """The paper's equivalence (Fig. 1, §3.2): trace == raster (O3, the tile lists)."""
    sc = pf_synth.make_scene("small360")
    cam = pf_synth.make_cameras("small360")[0]
    rng = np.random.default_rng(4)
    pix = np.stack([rng.integers(0, cam.width, 600), rng.integers(0, cam.height, 600)], 1)
    t = oracle.trace(sc, cam, pixels=pix)["out"]
    r = oracle.render(sc, cam, mode=oracle.O3, pixels=pix)["out"]
    assert np.abs(t - r).max() <= 1e-12


def test_walk_visits_the_argmin_power_cells():
    """the visited sequence equals the sequence of argmin-power cells of a
    fine-step sampler (steps within 1e-6 of a boundary excluded)."""
    sc = pf_synth.make_scene("tiny")
    rng = np.random.default_rng(9)
    checked = 0
    for _ in range(200):
        Q = rng.uniform(-2.5, 2.5, 3)                  # origins inside and around the foam,
        d = rng.uniform(-1.0, 1.0, 3) - Q              # rays aimed through it
        d /= np.linalg.norm(d)
        cells = oracle.trace_cells(sc, Q, d, 0.0)
        assert len(cells) == len(set(cells))          # convex cells: no revisits
        ts = np.arange(0.0, 8.0, 1e-3)
        lab, _ = argmin_power_sampler(sc, Q, d, ts)
        seq = [int(v) for k, v in enumerate(lab) if v >= 0 and (k == 0 or lab[k - 1] != v)]
        # the sampler sees every cell whose segment is longer than its step; the walk's
        # other cells are sub-step slivers
        assert [c for c in cells if c in set(seq)] == seq, (Q, d)
        checked += len(seq) > 0
    assert checked > 150


def test_single_cell_closed_form_and_miss():
    """one cell, sigma = 2, chord 1 -> ((1 - e^-2) c, e^-2); a ray that misses
    every ball returns the background with T = 1 and visits nothing."""
    c = [0.3, 0.6, 0.9]
    sc = scene_from([[0.0, 0.0, 0.0]], radii=[0.5], density=[2.0], rgb=[c], bg=(0.1, 0.2, 0.3))
    cam = camera(W=1, H=1, f=80.0)
    t = oracle.trace(sc, cam)
    out = t["out"][0, 0]
    assert np.allclose(out[:3], (1 - math.exp(-2)) * np.array(c) +
                       math.exp(-2) * np.array([0.1, 0.2, 0.3]), atol=1e-12)
    assert out[3] == pytest.approx(math.exp(-2), rel=1e-12)
    assert list(t["stats"][0, 0]) == [1, 2, 1]        # visit, locate twice (enter, leave)
    miss = camera(W=1, H=1, f=80.0, target=(5.0, 5.0, 0.0))
    t = oracle.trace(sc, miss)
    assert np.allclose(t["out"][0, 0], [0.1, 0.2, 0.3, 1.0])
    assert list(t["stats"][0, 0]) == [0, 1, 0]


def test_walk_steps_disjoint_chain_and_overlapping_chain():
    """Disjoint balls on the axis: every transition is a gap jump (locate per ball, plus
    the first); overlapping (Čech-adjacent) balls: the walk crosses radical planes, one
    locate to enter and one after the last sphere exit."""
    z = [-1.0, 0.0, 1.0, 2.0]
    cam = camera(W=1, H=1, f=80.0)
    dis = scene_from([[0, 0, zk] for zk in z], radii=[0.3] * 4, density=[0.1] * 4, lists="cech")
    t = oracle.trace(dis, cam)
    assert list(t["stats"][0, 0]) == [4, 5, 4]
    ovl = scene_from([[0, 0, zk] for zk in z], radii=[0.7] * 4, density=[0.1] * 4, lists="cech")
    assert ovl.num_edges == 6                          # a chain: 3 undirected edges
    t = oracle.trace(ovl, cam)
    assert list(t["stats"][0, 0]) == [4, 2, 4]
    Q, d, tn = ray_np(cam, 0, 0)
    assert oracle.trace_cells(ovl, Q, d, tn) == [0, 1, 2, 3]
    # equal to the definition
    for sc in (dis, ovl):
        assert np.abs(oracle.trace(sc, cam)["out"] -
                      oracle.render(sc, cam, mode=oracle.O1)["out"]).max() <= 1e-14


def test_early_stop_counts():
    """The walk stops after the segment that makes T < 1e-4: with six
    overlapping opaque cells (tau = 7.2, 6, ...) it composites exactly two."""
    z = [-1.0, 0.0, 1.0, 2.0, 3.0, 4.0]
    sc = scene_from([[0, 0, zk] for zk in z], radii=[0.7] * 6, density=[6.0] * 6, lists="cech")
    cam = camera(W=1, H=1, f=80.0)
    t = oracle.trace(sc, cam)
    assert list(t["stats"][0, 0]) == [2, 1, 2]
    assert t["out"][0, 0, 3] < 1e-4
