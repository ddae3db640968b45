"""Pins for the oracle backward (oracle/pf_oracle.c: oracle_backward):
central finite differences of the double oracle and single-cell closed forms."""
import math

import numpy as np
import pytest

import oracle
import pf_synth
from helpers import camera, scene_from


def _loss(sc, cam, g, mode):
    r = oracle.render(sc, cam, mode=mode, signature=True)
    return float((r["out"].reshape(-1, 4) * g.reshape(-1, 4).astype(np.float64)).sum()), r["sig"]


@pytest.mark.parametrize("which", ["sites", "weights", "radii", "density", "rgb"])
def test_backward_matches_central_fd_tiny(which):
    """SURVEY 8(c) 'Backward' pin / S:536-537: analytic vs central FD,
    excluding coordinates whose active-set signature changes."""
    sc = pf_synth.make_scene("tiny")
    cam = pf_synth.make_cameras("tiny")[0]
    g = pf_synth.make_grad_out(1, cam.height, cam.width, seed=11)[0] * (cam.height * cam.width)
    mode = oracle.O2
    an = oracle.backward(sc, cam, g, mode=mode)[which]
    L0, sig0 = _loss(sc, cam, g, mode)
    rng = np.random.default_rng({"sites": 1, "weights": 2, "radii": 3, "density": 4, "rgb": 5}[which])
    arr = getattr(sc, which)
    flat_an = an.reshape(-1)
    nz = np.flatnonzero(np.abs(flat_an) > 0)
    assert nz.size > 10
    pick = rng.choice(nz, size=min(24, nz.size), replace=False)
    scale = np.abs(flat_an).max()
    ok = bad = skipped = 0
    for q in pick:
        i = q // (arr.shape[1] if arr.ndim == 2 else 1)
        base = arr.reshape(-1)[q]
        h = {"sites": 1e-5 * sc.radii[i], "weights": 1e-5 * sc.weights[i],
             "radii": 1e-5 * sc.radii[i], "density": 1e-5 * max(sc.density[i], 1.0),
             "rgb": 1e-3}[which]
        vals = []
        for s in (+1, -1):
            sc2 = sc.copy()
            a2 = getattr(sc2, which).reshape(-1)
            a2[q] = np.float32(base + s * h)
            L, sig = _loss(sc2, cam, g, mode)
            vals.append((float(a2[q]), L, sig))
        if not (np.array_equal(vals[0][2], sig0) and np.array_equal(vals[1][2], sig0)):
            skipped += 1
            continue
        fd = (vals[0][1] - vals[1][1]) / (vals[0][0] - vals[1][0])
        if abs(fd - flat_an[q]) <= 2e-4 * abs(flat_an[q]) + 1e-7 * scale:
            ok += 1
        else:
            bad += 1
    print(which, ok, bad, skipped)
    assert ok >= 0.95 * (ok + bad) and ok >= 12, (ok, bad, skipped)


def test_single_cell_closed_form_gradients():
    """Central ray through one sphere: C = (1-e^{-2 sigma r}) c + e^{-2 sigma r} bg, so
    dC/dsigma = 2r e^{-2 sigma r}(c-bg), dC/dr = 2 sigma e^{-2 sigma r}(c-bg)."""
    sig, r = 1.7, 0.4
    rgb = np.array([0.8, 0.3, 0.5], np.float32)
    bg = np.array([0.25, 0.5, 0.0], np.float32)
    sc = scene_from([[0.0, 0.0, 0.0]], radii=[r], density=[sig], rgb=[rgb], bg=tuple(bg))
    cam = camera(W=3, H=3, f=50.0)   # pixel (1,1) centre = principal point -> optical axis
    s32, r32 = float(np.float32(sig)), float(np.float32(r))
    E = math.exp(-2 * s32 * r32)
    for ch in range(4):
        go = np.zeros((1, 4), np.float32); go[0, ch] = 1.0
        g = oracle.backward(sc, cam, go, mode=oracle.O1, pixels=np.array([[1, 1]]))
        if ch < 3:
            dc = float(rgb[ch]) - float(bg[ch])
            assert g["density"][0] == pytest.approx(2 * r32 * E * dc, rel=1e-9)
            assert g["radii"][0] == pytest.approx(2 * s32 * E * dc, rel=1e-9)
            assert g["rgb"][0, ch] == pytest.approx(1 - E, rel=1e-12)
        else:  # dT/dsigma = -2r e^{-2 sigma r}
            assert g["density"][0] == pytest.approx(-2 * r32 * E, rel=1e-9)
            assert g["radii"][0] == pytest.approx(-2 * s32 * E, rel=1e-9)
        assert np.abs(g["sites"][0]).max() < 1e-9   # symmetric chord: no site gradient
