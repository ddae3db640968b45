"""Test helpers: hand-built scenes and an independent pixel-ray / sampler in numpy.

Nothing here calls the CUDA path; the brute-force samplers below are the
independent references the oracle is pinned to."""
from __future__ import annotations

import numpy as np

import pf_synth


def scene_from(sites, radii, weights=None, density=None, rgb=None, lists="all", bg=(0, 0, 0)):
    sites = np.asarray(sites, np.float32).reshape(-1, 3)
    N = sites.shape[0]
    radii = np.asarray(radii, np.float32).reshape(N)
    weights = (radii * radii).astype(np.float32) if weights is None else \
        np.asarray(weights, np.float32).reshape(N)
    density = np.ones(N, np.float32) if density is None else np.asarray(density, np.float32)
    rgb = np.full((N, 3), 0.5, np.float32) if rgb is None else \
        np.asarray(rgb, np.float32).reshape(N, 3)
    if isinstance(lists, str) and lists == "all":
        off, idx = pf_synth.all_pairs_lists(N) if N > 1 else (np.zeros(2, np.int64),
                                                              np.zeros(0, np.int32))
    elif isinstance(lists, str) and lists == "cech":
        P = sites.astype(np.float64)
        r = radii.astype(np.float64)
        nb = [[j for j in range(N) if j != i and np.linalg.norm(P[i] - P[j]) < r[i] + r[j]]
              for i in range(N)]
        off = np.zeros(N + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in nb])
        idx = np.asarray([j for x in nb for j in x], np.int32)
    else:
        off, idx = lists
    if N == 1:
        off = np.zeros(2, np.int64)
        idx = np.zeros(0, np.int32)
    return pf_synth.Scene(sites, weights, radii, density, rgb, np.asarray(off, np.int64),
                          np.asarray(idx, np.int32), tuple(bg), "hand")


def camera(W=64, H=64, f=80.0, eye=(0.0, 0.0, -3.5), target=(0.0, 0.0, 0.0), near=0.05,
           c2w=None, cx=None, cy=None):
    if c2w is None:
        c2w = pf_synth.look_at(eye, target, up=(0.0, -1.0, 0.0))
    return pf_synth.Camera(W, H, f, f, W / 2.0 if cx is None else cx,
                           H / 2.0 if cy is None else cy, np.asarray(c2w, np.float32), near)


def ray_np(cam, x, y):
    """Independent numpy pixel ray (pixel centres at +0.5, OpenCV axes)."""
    M = np.asarray(cam.c2w, np.float64).reshape(3, 4)
    dc = np.array([(x + 0.5 - cam.cx) / cam.fx, (y + 0.5 - cam.cy) / cam.fy, 1.0])
    d = M[:, :3] @ dc
    d /= np.linalg.norm(d)
    return M[:, 3].copy(), d, cam.near * np.linalg.norm(dc)


def argmin_power_sampler(sc, Q, d, ts, t_near=0.0):
    """For each t: the bounded power cell containing x(t) (or -1): argmin_j pow(x, j),
    ties by lowest index, and inside its sphere; -1 before t_near."""
    P = sc.sites.astype(np.float64)
    w = sc.weights.astype(np.float64)
    r = sc.radii.astype(np.float64)
    X = Q[None, :] + ts[:, None] * d[None, :]
    pw = ((X[:, None, :] - P[None, :, :]) ** 2).sum(-1) - w[None, :]
    i = np.argmin(pw, axis=1)
    inside = ((X - P[i]) ** 2).sum(-1) <= r[i] ** 2
    out = np.where(inside & (ts >= t_near), i, -1)
    return out, pw
