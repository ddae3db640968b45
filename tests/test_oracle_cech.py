"""Pins for the oracle's Čech graph and L_connect (NEXT-3; PAPER.md l.234,
l.733-741)."""
import numpy as np
import pytest

import oracle
import pf_synth


def test_spec_cech_examples():
    # radii 2 and 2 at distance 3 -> edge; 5 -> none; exactly 4 -> none (strict)
    for dist, edge in ((3.0, True), (5.0, False), (4.0, False)):
        off, idx = oracle.cech_rows([[0, 0, 0], [dist, 0, 0]], [2.0, 2.0])
        assert (off[-1] == 2) == edge
        if edge:
            assert list(idx) == [1, 0]


def test_equal_radii_reduce_to_kdtree_ball_pairs():
    """Equal radii r: Čech pairs = pairs closer than 2r (scipy query_pairs, an
    independent library routine; ties have measure zero for random data)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(0)
    P = rng.uniform(-1, 1, size=(3000, 3)).astype(np.float32)
    r = np.full(3000, 0.04, np.float32)
    off, idx = oracle.cech_rows(P, r)
    pairs = cKDTree(P.astype(np.float64)).query_pairs(2 * 0.04, output_type="ndarray")
    got = {(i, int(j)) for i in range(3000) for j in idx[off[i]:off[i + 1]]}
    ref = {(int(a), int(b)) for a, b in pairs} | {(int(b), int(a)) for a, b in pairs}
    assert got == ref and len(ref) > 1000


def test_matches_generator_lists():
    """pf_synth's lists are the Čech complex by SURVEY Lemma L3 (sym-KNN filter)."""
    sc = pf_synth.make_scene("small", num_cells=2500)
    off, idx = oracle.cech_rows(sc.sites, sc.radii)
    assert np.array_equal(off, sc.nbr_offsets)
    assert np.array_equal(idx, sc.nbr_indices)
    rows = np.array([0, 17, 2499])
    o2, i2 = oracle.cech_rows(sc.sites, sc.radii, rows=rows)
    for k, i in enumerate(rows):
        assert np.array_equal(i2[o2[k]:o2[k + 1]], idx[off[i]:off[i + 1]])


def test_connect_loss_spec_values_and_fd():
    # r1=2, r2=2, d=3 -> 1.0 per unordered edge (each cell's term)
    off, idx = oracle.cech_rows([[0, 0, 0], [3, 0, 0]], [2.0, 2.0])
    out = oracle.connect_loss([[0, 0, 0], [3, 0, 0]], [2.0, 2.0], off, idx)
    assert np.allclose(out["loss"], [1.0, 1.0])
    # concentric d=0, r=1 -> 4.0
    off, idx = oracle.cech_rows([[0, 0, 0], [0, 0, 0]], [1.0, 1.0])
    out = oracle.connect_loss([[0, 0, 0], [0, 0, 0]], [1.0, 1.0], off, idx)
    assert np.allclose(out["loss"], [4.0, 4.0])
    # central FD of the total on a small foam
    sc = pf_synth.make_scene("tiny")
    off, idx = oracle.cech_rows(sc.sites, sc.radii)
    base = oracle.connect_loss(sc.sites, sc.radii, off, idx)
    rng = np.random.default_rng(1)
    for which in ("sites", "radii"):
        arr = getattr(sc, which)
        for q in rng.choice(arr.size, 12, replace=False):
            h = 1e-4
            vals = []
            for s_ in (1, -1):
                a = arr.copy().reshape(-1)
                a[q] = np.float32(arr.reshape(-1)[q] + s_ * h)
                st = a.reshape(arr.shape)
                kw = dict(sites=st, radii=sc.radii) if which == "sites" else dict(
                    sites=sc.sites, radii=st)
                vals.append((float(a[q]), oracle.connect_loss(kw["sites"], kw["radii"], off,
                                                              idx)["loss"].sum()))
            fd = (vals[0][1] - vals[1][1]) / (vals[0][0] - vals[1][0])
            assert fd == pytest.approx(base[which].reshape(-1)[q], rel=1e-4, abs=1e-8)
