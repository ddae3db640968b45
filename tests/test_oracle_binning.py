"""Pins for the fp32 binning specification (oracle/pf_oracle.c)."""
import math
import struct

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import camera, ray_np, scene_from


def _f2bits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def _key_to_float(u):
    u = int(u)
    b = (u ^ 0x80000000) if (u >> 31) else (~u & 0xFFFFFFFF)
    return struct.unpack("<f", struct.pack("<I", b))[0]


def test_sort_key_spec_examples():
    # S:413 Q at the site position, r=1 -> -1 ; S:414 equal distance 5, radii 1 and 2
    sc = scene_from([[0, 0, 0], [0, 0, 5], [3, 0, 4]], radii=[1.0, 1.0, 2.0])
    cam = camera(W=32, H=32, f=40.0, c2w=np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0],
                                                   np.float32))
    _, _, kb = oracle.bin_cells(sc, cam)
    assert _key_to_float(kb[0]) == -1.0
    assert _key_to_float(kb[1]) == 24.0 and _key_to_float(kb[2]) == 21.0
    assert kb[2] < kb[1]   # larger sphere drawn first


def test_key_bits_order_preserving():
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.normal(size=500) * 10 ** rng.uniform(-8, 8, 500),
                           [0.0, -0.0, 1e-45, -1e-45, 3.4e38, -3.4e38]]).astype(np.float32)
    N = len(vals)
    # K = |p-Q|^2 - w with p = Q  ->  K = -w exactly
    sc = scene_from(np.zeros((N, 3)), radii=np.ones(N), weights=-vals, lists=(
        np.zeros(N + 1, np.int64), np.zeros(0, np.int32)))
    cam = camera(W=16, H=16, f=10.0, c2w=np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0],
                                                   np.float32))
    _, _, kb = oracle.bin_cells(sc, cam)
    for v, k in zip(vals, kb):
        assert _key_to_float(k) == v or (v == 0 and _key_to_float(k) == 0)
    order_bits = np.argsort(kb, kind="stable")
    s = vals[order_bits]
    assert np.all(s[1:] >= s[:-1])


def test_on_axis_box_spec_example():
    # sphere on the optical axis at depth 10, r=1, f=100 -> half-width 100/sqrt(99)=10.05 px
    sc = scene_from([[0, 0, 10]], radii=[1.0])
    cam = camera(W=400, H=400, f=100.0, c2w=np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0],
                                                      np.float32))
    rect, count, _ = oracle.bin_cells(sc, cam)
    hw = 100 / math.sqrt(99)
    lo, hi = 200 - hw - 1, 200 + hw + 1
    t0, t1 = math.floor(lo / 16), math.floor(hi / 16) + 1
    assert tuple(rect[0]) == (t0, t0, t1, t1) and count[0] == (t1 - t0) ** 2


def test_camera_inside_and_behind():
    cam = camera(W=100, H=70, f=60.0, c2w=np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0.5],
                                                    np.float32))
    # S:424 camera inside the sphere -> every tile
    sc = scene_from([[0, 0, 0]], radii=[2.0])
    rect, count, _ = oracle.bin_cells(sc, cam)
    tx, ty = (100 + 15) // 16, (70 + 15) // 16
    assert tuple(rect[0]) == (0, 0, tx, ty) and count[0] == tx * ty
    # S:425 sphere fully behind the camera -> no tile
    sc = scene_from([[0, 0, -3]], radii=[1.0])
    rect, count, _ = oracle.bin_cells(sc, cam)
    assert count[0] == 0


def test_binning_conservative_brute_force():
    """Every pixel whose (double) ray meets a sphere after t_near lies in the
    sphere's tile rectangle; and the rectangle is tight (within one tile of the
    hit pixels) for spheres fully in front of the near plane."""
    rng = np.random.default_rng(5)
    W, H = 96, 80
    N = 120
    P = np.stack([rng.uniform(-3, 3, N), rng.uniform(-3, 3, N), rng.uniform(-1, 6, N)], 1)
    r = rng.uniform(0.05, 1.5, N)
    sc = scene_from(P, r, lists=(np.zeros(N + 1, np.int64), np.zeros(0, np.int32)))
    cam = camera(W=W, H=H, f=50.0, c2w=np.array([1, 0, 0, 0.1, 0, 1, 0, -0.2, 0, 0, 1, -2.0],
                                                 np.float32), near=0.3)
    rect, count, _ = oracle.bin_cells(sc, cam)
    rays = [[ray_np(cam, x, y) for x in range(W)] for y in range(H)]
    P64 = sc.sites.astype(np.float64); r64 = sc.radii.astype(np.float64)
    checked = 0
    for i in range(N):
        hits = []
        for y in range(H):
            for x in range(W):
                Q, d, tn = rays[y][x]
                c = P64[i] - Q; tc = c @ d; e = c - tc * d; h = r64[i] ** 2 - e @ e
                if h > 0 and tc + math.sqrt(h) > tn:
                    hits.append((x, y))
        for x, y in hits:
            assert rect[i, 0] <= x // 16 < rect[i, 2] and rect[i, 1] <= y // 16 < rect[i, 3]
        checked += len(hits)
        cz = P64[i, 2] + 2.0
        if hits and cz - r64[i] > 0.3:
            xs = [h[0] for h in hits]; ys = [h[1] for h in hits]
            assert rect[i, 0] >= min(xs) // 16 - 1 and rect[i, 2] <= max(xs) // 16 + 2
            assert rect[i, 1] >= min(ys) // 16 - 1 and rect[i, 3] <= max(ys) // 16 + 2
    assert checked > 2000


def test_sorted_pairs_and_ranges_small():
    sc = pf_synth.make_scene("small", num_cells=1500)
    cam = pf_synth.make_cameras("small", width=96, height=72)[0]
    b = oracle.binning(sc, cam)
    keys, vals = b["keys"], b["vals"]
    assert b["P"] == int(b["count"].sum()) > 0
    # ascending, equal keys in cell order (stable over cell-major emission, C12)
    assert np.all(keys[1:] >= keys[:-1])
    eq = keys[1:] == keys[:-1]
    assert np.all(vals[1:][eq] > vals[:-1][eq])
    # every pair is (tile in the cell's rect, the cell's key bits)
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    tx, ty = tiles % b["tiles_x"], tiles // b["tiles_x"]
    rc = b["rect"][vals]
    assert np.all((rc[:, 0] <= tx) & (tx < rc[:, 2]) & (rc[:, 1] <= ty) & (ty < rc[:, 3]))
    assert np.array_equal((keys & np.uint64(0xFFFFFFFF)).astype(np.uint32), b["keybits"][vals])
    assert np.array_equal(np.bincount(vals, minlength=sc.num_cells), b["count"])
    # ranges: [start,end) spans exactly the pairs of tile t
    for t in range(b["tiles_x"] * b["tiles_y"]):
        s, e = b["ranges"][t]
        sel = np.flatnonzero(tiles == t)
        if sel.size == 0:
            assert s == e == 0
        else:
            assert s == sel[0] and e == sel[-1] + 1
