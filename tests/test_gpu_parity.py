"""GPU parity: the CUDA path (through the C-ABI library) against the CPU oracle on
the same seeded inputs.  Bars (BASELINE.json north_star):
binning bit-exact; images <= 1e-4 abs per fp32 channel; gradients <= 1e-3
relative (normwise per array)."""
import os

import numpy as np
import pytest

import oracle
import pf_synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-3

_cache = {}


def case(name, variant=None):
    key = (name, variant)
    if key not in _cache:
        if name == "tiny":
            sc = pf_synth.make_scene("tiny")
            cams = pf_synth.make_cameras("tiny", variant=variant or "outside")
        elif name == "tiny_knn8":
            sc = pf_synth.make_scene("tiny", variant="knn8")
            cams = pf_synth.make_cameras("tiny")
        elif name == "tiny_w0":
            sc = pf_synth.make_scene("tiny", variant="allpairs_w0")
            cams = pf_synth.make_cameras("tiny")
        elif name == "small":
            sc = pf_synth.make_scene("small")
            cams = pf_synth.make_cameras("small")
        elif name == "small360":
            sc = pf_synth.make_scene("small360")
            cams = pf_synth.make_cameras("small360", n=4)
        elif name == "nerfsynth200k":
            sc = pf_synth.make_scene("nerfsynth200k")
            cams = pf_synth.make_cameras("nerfsynth200k")
        elif name == "train8_1m":
            sc = pf_synth.make_scene("train8_1m")
            cams = pf_synth.make_cameras("train8_1m")
        elif name == "mip360_1m":
            sc = pf_synth.make_scene("mip360_1m")
            cams = pf_synth.make_cameras("mip360_1m")
        elif name == "sweep64_3m":
            sc = pf_synth.make_scene("sweep64_3m")
            cams = pf_synth.make_cameras("sweep64_3m")
        elif name.endswith("+detail"):
            base, bcams = case(name[:-len("+detail")], variant)
            sc = pf_synth.add_detail(base.copy())
            cams = bcams
        elif name.endswith("+dipoles"):
            base, bcams = case(name[:-len("+dipoles")], variant)
            sc = pf_synth.add_dipoles(base.copy())
            cams = bcams
        else:
            raise KeyError(name)
        _cache[key] = (sc, cams)
    return _cache[key]


def renderer(sc, flags=None):
    import paper_2604_24994_b200 as pf
    return pf.Renderer.from_scene(sc, "cuda", flags=pf.PF_VALIDATE if flags is None else flags)


COND_LIMIT = 0.05   # a per-cell C17 failure must come with a min(s/r, |a|/|n|) below this


def _pixel_rays(cam, pix):
    """Rays (Q, d[n,3], t_near[n]) of pixels pix[n,2]: the oracle's pixel_ray."""
    Q = None
    D = np.zeros((len(pix), 3))
    tn = np.zeros(len(pix))
    for k, (x, y) in enumerate(pix):
        Q, D[k], tn[k] = oracle.pixel_ray(cam, int(x), int(y))
    return Q, D, tn


def _all_pixels(cam):
    ys, xs = np.mgrid[0:cam.height, 0:cam.width]
    return np.stack([xs.ravel(), ys.ravel()], 1)


def conditioning(sc, views, cell, mode=None):
    """SURVEY C17 conditioning of one cell over the pixels that carry gradient:
    views = [(cam, pix or None)].  For every composited segment in which `cell` is
    the segment's cell or the binding neighbour: s/r of a sphere endpoint (s the
    half chord, R1) and |a|/|n| = |d.n|/|n| of a binding plane (or dipole face).
    Returns (min s/r, min |a|/|n|, pixels seen)."""
    P = sc.sites.astype(np.float64)
    r = sc.radii.astype(np.float64)
    best_s, best_a, npix = np.inf, np.inf, 0
    for cam, pix in views:
        pix = _all_pixels(cam) if pix is None else np.asarray(pix)
        if cam.model == 0:
            M = np.asarray(cam.c2w, np.float64).reshape(3, 4)
            dc = np.stack([(pix[:, 0] + 0.5 - cam.cx) / cam.fx, (pix[:, 1] + 0.5 - cam.cy) / cam.fy,
                           np.ones(len(pix))], 1)
            D = dc @ M[:, :3].T
            D /= np.linalg.norm(D, axis=1, keepdims=True)
            Q = M[:, 3]
        else:
            Q, D, _ = _pixel_rays(cam, pix)
        c = P[cell] - Q
        tc = D @ c
        rho2 = c @ c - tc * tc
        cand = pix[rho2 < r[cell] ** 2 * (1 + 1e-9)]
        m = (oracle.O1 if sc.num_cells <= 4096 else oracle.O2) if mode is None else mode
        for x, y in cand:
            segs = oracle.pixel_segments(sc, cam, int(x), int(y), mode=m)
            Qp, d, _ = oracle.pixel_ray(cam, int(x), int(y))
            for sg in segs:
                i = int(sg["cell"])
                roles = []
                if i == cell:
                    roles = [("in", sg["kin"], sg["jin"]), ("out", sg["kout"], sg["jout"])]
                else:
                    roles = [(e, k, j) for e, k, j in (("in", sg["kin"], sg["jin"]),
                                                       ("out", sg["kout"], sg["jout"]))
                             if int(k) == 2 and int(j) == cell]
                if not roles:
                    continue
                npix += 1
                for _, kind, j in roles:
                    kind, j = int(kind), int(j)
                    if kind == 0:        # sphere endpoint of cell i: s/r
                        ci = P[i] - Qp
                        h = r[i] ** 2 - (ci @ ci - (d @ ci) ** 2)
                        best_s = min(best_s, np.sqrt(max(h, 0.0)) / r[i])
                    elif kind == 2:      # plane between i and j
                        n = P[j] - P[i]
                        best_a = min(best_a, abs(d @ n) / np.linalg.norm(n))
                    elif kind == 3 and sc.normals is not None:
                        nv = sc.normals[i].astype(np.float64)
                        best_a = min(best_a, abs(d @ nv) / np.linalg.norm(nv))
    return best_s, best_a, npix


def grad_check(gpu, ref, tol=GRAD_TOL, ctx=None):
    """normwise per array <= tol; per cell |g_i - g_ref,i| <= 1e-3 |g_ref,i|
    + 1e-5 max |g_ref|.  Every cell that fails the per-cell bar is LISTED with its
    conditioning (ctx = (scene, [(cam, pixels-or-None)])) and must be ill-conditioned
    (min(s/r, |a|/|n|) < COND_LIMIT); without ctx no per-cell failure is accepted."""
    msgs = []
    keys = ("sites", "weights", "radii", "density", "rgb") + (("normals",) if "normals" in ref
                                                               else ())
    keys += tuple(k for k in ("detail_uv", "detail_disp", "detail_sv") if k in ref)
    failing = {}
    for k in keys:
        a = gpu[k].detach().cpu().numpy().astype(np.float64).reshape(-1)
        b = ref[k].reshape(-1)
        nb = np.linalg.norm(b)
        rel = np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)
        msgs.append(f"{k}: {rel:.2e}")
        assert rel <= tol, ", ".join(msgs)
        N = ref["density"].shape[0]
        ac, bc = a.reshape(N, -1), b.reshape(N, -1)
        ni = np.linalg.norm(bc, axis=1)
        err = np.linalg.norm(ac - bc, axis=1)
        bad = err > 1e-3 * ni + 1e-5 * ni.max()
        for c in np.flatnonzero(bad):
            failing.setdefault(int(c), []).append((k, float(err[c] / max(ni[c], 1e-30))))
    if failing:
        assert ctx is not None, f"per-cell C17 failures (no conditioning context): {failing}"
        sc, views = ctx
        lines = []
        for c, what in sorted(failing.items()):
            s_r, a_n, npx = conditioning(sc, views, c)
            lines.append(f"cell {c}: {what} min s/r {s_r:.2e} min |a|/|n| {a_n:.2e} "
                         f"({npx} segments)")
            assert min(s_r, a_n) < COND_LIMIT, "well-conditioned cell fails C17: " + lines[-1]
        print("per-cell C17 failures (ill-conditioned, listed):\n  " + "\n  ".join(lines))
        msgs.append(f"{len(failing)} ill-conditioned cells listed")
    return msgs


# --------------------------------------------------------------- binning

@pytest.mark.parametrize("name,variant", [("tiny", "outside"), ("tiny", "inside"),
                                          ("small", None), ("small360", None),
                                          ("nerfsynth200k", None), ("train8_1m", None)])
def test_binning_bit_exact(name, variant):
    sc, cams = case(name, variant)
    r = renderer(sc)
    for cam in cams[:2]:
        g = r.debug_binning(cam)
        o = oracle.binning(sc, cam)
        assert np.array_equal(g["rect"].cpu().numpy(), o["rect"])
        assert np.array_equal(g["count"].cpu().numpy(), o["count"])
        assert np.array_equal(g["keybits"].cpu().numpy().view(np.uint32), o["keybits"])
        assert g["P"] == o["P"]
        assert np.array_equal(g["keys"].cpu().numpy().view(np.uint64), o["keys"])
        assert np.array_equal(g["vals"].cpu().numpy().view(np.uint32), o["vals"])
        assert np.array_equal(g["ranges"].cpu().numpy().view(np.uint32), o["ranges"])
    r.close()


# --------------------------------------------------------------- forward

@pytest.mark.parametrize("name,variant", [("tiny", "outside"), ("tiny", "inside"),
                                          ("tiny_knn8", None), ("tiny_w0", None),
                                          ("small", None), ("small360", None)])
def test_forward_full_image(name, variant):
    sc, cams = case(name, variant)
    r = renderer(sc)
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    for v, cam in enumerate(cams):
        # raw directed 8-NN lists are not a Čech superset: GPU == O2 (same lists),
        # O1 may differ there; every other case is checked against O1/O3
        mode = oracle.O2 if name == "tiny_knn8" else (oracle.O1 if name.startswith("tiny")
                                                      else oracle.O3)
        ref = oracle.render(sc, cam, mode=mode)["out"]
        err = np.abs(out[v] - ref)
        assert err.max() <= IMG_TOL, (v, err.max())
        if name.startswith("tiny") and mode != oracle.O1:
            o1 = oracle.render(sc, cam, mode=oracle.O1)["out"]
            print(f"{name}: max |GPU - O1| = {np.abs(out[v] - o1).max():.3e} (reported)")
    r.close()


@pytest.mark.parametrize("name", ["tiny", "small", "small360"])
def test_forward_counters_match_oracle(name):
    sc, cams = case(name)
    r = renderer(sc)
    cam = cams[0]
    g = r.debug_counters(cam).cpu().numpy().reshape(-1, 4)
    o = oracle.render(sc, cam, mode=oracle.O3, counters=True)["counters"]
    mism = np.any(g != o, axis=1).mean()
    assert mism <= 1e-3, mism
    assert abs(g.sum(0) - o.sum(0)).max() <= 1e-3 * o.sum(0).max()
    r.close()


@pytest.mark.parametrize("name", ["nerfsynth200k", "train8_1m"])
def test_forward_large_sampled_pixels(name):
    """Full BASELINE sizes, all views in one call (the bench launch configuration);
    oracle on sampled pixels (O3 tile lists, plus O1 all-pairs on a few)."""
    sc, cams = case(name)
    r = renderer(sc, flags=0)
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(0)
    for v in (0, len(cams) - 1):
        cam = cams[v]
        pix = np.stack([rng.integers(0, cam.width, 3000), rng.integers(0, cam.height, 3000)], 1)
        ref = oracle.render(sc, cam, mode=oracle.O3, pixels=pix)["out"]
        got = out[v][pix[:, 1], pix[:, 0]]
        assert np.abs(got - ref).max() <= IMG_TOL
        few = pix[:24]
        ref1 = oracle.render(sc, cam, mode=oracle.O1, pixels=few)["out"]
        assert np.abs(out[v][few[:, 1], few[:, 0]] - ref1).max() <= IMG_TOL
    assert np.isfinite(out).all()
    r.close()


def test_multiview_equals_single_view_and_deterministic():
    sc, cams = case("small360")
    r = renderer(sc)
    multi = r.forward(cams).cpu().numpy()
    again = r.forward(cams).cpu().numpy()
    assert np.array_equal(multi, again)
    for v, cam in enumerate(cams):
        single = r.forward([cam]).cpu().numpy()[0]
        assert np.array_equal(single, multi[v])
    r.close()


def test_many_views_in_one_call_batched_sorts():
    """More than 8 views in one call are sorted in batches of 8 (DESIGN §6 K4): every
    view equals its single-view render bit for bit, and the multi-view backward
    equals the sum of the single-view backwards (up to atomic summation order)."""
    sc, _ = case("small360")
    cams = pf_synth.make_cameras("small360", n=11)
    r = renderer(sc)
    multi = r.forward(cams).cpu().numpy()
    for v, cam in enumerate(cams):
        single = r.forward([cam]).cpu().numpy()[0]
        assert np.array_equal(single, multi[v]), v
    H, W = cams[0].height, cams[0].width
    g = torch.from_numpy(pf_synth.make_grad_out(len(cams), H, W, seed=5)).cuda()
    r.forward(cams)
    got = {k: v.clone() for k, v in r.backward(cams, g).items()}
    acc = None
    for v, cam in enumerate(cams):
        r.forward([cam])
        one = r.backward([cam], g[v:v + 1].contiguous())
        acc = {k: x.clone() for k, x in one.items()} if acc is None else \
            {k: acc[k] + one[k] for k in acc}
    for k in got:
        a, b = got[k].double(), acc[k].double()
        assert float((a - b).norm()) <= 1e-5 * float(b.norm()) + 1e-12, k
    r.close()


# --------------------------------------------------------------- backward

@pytest.mark.parametrize("name,variant", [("tiny", "outside"), ("tiny", "inside"),
                                          ("small", None), ("small360", None)])
def test_backward_full_image(name, variant):
    sc, cams = case(name, variant)
    r = renderer(sc)
    cams = cams[:2]
    H, W = cams[0].height, cams[0].width
    g = pf_synth.make_grad_out(len(cams), H, W, seed=11)
    r.forward(cams)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    mode = oracle.O1 if name == "tiny" else oracle.O3
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=mode)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()


@pytest.mark.parametrize("name", ["nerfsynth200k", "train8_1m"])
def test_backward_large_sampled_pixels(name):
    """Full sizes, all views in one call; dL/dout is non-zero only on sampled pixels,
    so the oracle can compute the exact gradient pixel by pixel."""
    sc, cams = case(name)
    r = renderer(sc, flags=0)
    H, W = cams[0].height, cams[0].width
    rng = np.random.default_rng(1)
    g = np.zeros((len(cams), H, W, 4), np.float32)
    pix = {}
    for v in (0, len(cams) - 1):
        p = np.stack([rng.integers(0, W, 1500), rng.integers(0, H, 1500)], 1)
        p = np.unique(p, axis=0)
        pix[v] = p
        g[v, p[:, 1], p[:, 0]] = rng.standard_normal((p.shape[0], 4)).astype(np.float32)
    r.forward(cams)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, p in pix.items():
        o = oracle.backward(sc, cams[v], g[v, p[:, 1], p[:, 0]], mode=oracle.O3, pixels=p)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(cams[v], p) for v, p in pix.items()]))
    r.close()


def test_inference_forward_equals_training_forward():
    import paper_2604_24994_b200 as pf
    sc, cams = case("small360")
    r = renderer(sc)
    ri = renderer(sc, flags=pf.PF_INFERENCE)
    a = r.forward(cams).cpu().numpy()
    b = ri.forward(cams).cpu().numpy()
    assert np.array_equal(a, b)
    g = torch.zeros((len(cams), cams[0].height, cams[0].width, 4), device="cuda")
    with pytest.raises(pf.PFError) as e:
        ri.backward(cams, g)
    assert e.value.status == 4
    r.close()
    ri.close()


@pytest.mark.parametrize("name,variant,fish", [("tiny", "inside", False), ("small360", None, False),
                                               ("small+dipoles", None, False),
                                               ("small+detail", None, False),
                                               ("small360", None, True),
                                               ("small360", "knn", False),
                                               ("tiny_w0", None, False),
                                               ("nerfsynth200k", None, False),
                                               ("train8_1m", None, False)])
def test_plane_cull_is_exact(monkeypatch, name, variant, fish):
    """K6's warp-level plane cull drops only planes that cannot bind for
    any pixel of the warp and skips only cells whose every interval is empty, so the
    image is bit-identical to clipping by every list plane (PF_PLANE_CULL=0) and the
    backward (driven by the same K6 records) agrees up to atomic summation order."""
    if variant == "knn":   # unfiltered lists: many extra, never-binding planes
        sc, cams = pf_synth.make_scene(name, variant="knn"), case(name)[1]
    else:
        sc, cams = _fisheye_case(name, variant) if fish else case(name, variant)
    cams = cams[:2]
    H, W = cams[0].height, cams[0].width
    g = torch.from_numpy(pf_synth.make_grad_out(len(cams), H, W, seed=29)).cuda()
    res = {}
    for knob in ("1", "0"):
        monkeypatch.setenv("PF_PLANE_CULL", knob)
        r = renderer(sc)
        out = r.forward(cams).cpu().numpy()
        grads = {k: v.detach().cpu().numpy().astype(np.float64)
                 for k, v in r.backward(cams, g).items()}
        res[knob] = (out, grads)
        r.close()
    assert np.array_equal(res["1"][0], res["0"][0])
    for k, a in res["1"][1].items():
        b = res["0"][1][k]
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b) + 1e-30, k


def test_unfiltered_knn_lists_render_the_same():
    """Extra (non-Čech) neighbours never bind inside B_i (Lemma L1): the
    image with unfiltered sym-16NN lists equals the Čech-list image up to rounding and
    the oracle within the image bar; gradients within the gradient bar."""
    sc, cams = case("small360")
    sk = pf_synth.make_scene("small360", variant="knn")
    cams = cams[:2]
    H, W = cams[0].height, cams[0].width
    g = torch.from_numpy(pf_synth.make_grad_out(len(cams), H, W, seed=31)).cuda()
    r, rk = renderer(sc), renderer(sk)
    a, b = r.forward(cams).cpu().numpy(), rk.forward(cams).cpu().numpy()
    assert np.abs(a - b).max() <= 1e-5
    ref = oracle.render(sk, cams[0], mode=oracle.O3)["out"]
    assert np.abs(b[0] - ref).max() <= IMG_TOL
    ga = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in r.backward(cams, g).items()}
    grad_check(rk.backward(cams, g), ga)
    r.close()
    rk.close()


def test_in_place_parameter_update_between_forwards():
    """Without PF_STATIC_SCENE the edge records (K0) are rebuilt every forward, on a
    side stream forked from the caller's stream: an in-place update of the sites and
    weights enqueued on the caller's stream right before the forward must be seen
    (the image equals a fresh renderer's on the moved scene, bit for bit)."""
    import copy
    sc, cams = case("small360")
    cams = cams[:2]
    r = renderer(sc, flags=0)
    r.forward(cams)
    moved = copy.deepcopy(sc)
    rng = np.random.default_rng(3)
    moved.sites = (sc.sites + rng.normal(0, 2e-3, sc.sites.shape)).astype(np.float32)
    moved.weights = (sc.weights * np.float32(1.01)).astype(np.float32)
    s_t, w_t = r.params()[0], r.params()[1]
    s_t.copy_(torch.from_numpy(moved.sites).to(s_t.device), non_blocking=True)
    w_t.copy_(torch.from_numpy(moved.weights).to(w_t.device), non_blocking=True)
    got = r.forward(cams).cpu().numpy()
    ref = renderer(moved, flags=0).forward(cams).cpu().numpy()
    assert np.array_equal(got, ref)
    r.close()


def test_backward_record_overflow_fallback(monkeypatch):
    """K6->K7 record arena too small: overflowed chunks are recomputed in full by
    K7; gradients must be unchanged (parity with the oracle)."""
    monkeypatch.setenv("PF_REC_RATIO", "0.02")
    sc, cams = case("small360")
    r = renderer(sc)
    cams = cams[:2]
    H, W = cams[0].height, cams[0].width
    g = pf_synth.make_grad_out(len(cams), H, W, seed=11)
    r.forward(cams)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=oracle.O3)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()


def test_backward_requires_matching_forward():
    import paper_2604_24994_b200 as pf
    sc, cams = case("tiny")
    r = renderer(sc)
    g = torch.zeros((1, 64, 64, 4), device="cuda")
    with pytest.raises(pf.PFError) as e:
        r.backward(cams, g)
    assert e.value.status == 4
    r.forward(cams)
    other = pf_synth.make_cameras("tiny", variant="inside")
    with pytest.raises(pf.PFError) as e:
        r.backward(other, g)
    assert e.value.status == 4
    r.backward(cams, g)
    r.close()


def test_abi_argument_errors():
    import paper_2604_24994_b200 as pf
    sc, cams = case("tiny")
    bad = sc.copy()
    bad.nbr_indices = bad.nbr_indices.copy()
    bad.nbr_indices[3] = sc.num_cells + 5
    with pytest.raises(pf.PFError) as e:
        renderer(bad)
    assert e.value.status == 1
    bad = sc.copy()
    bad.radii = bad.radii.copy()
    bad.radii[0] = -1.0
    with pytest.raises(pf.PFError) as e:
        renderer(bad)
    assert e.value.status == 1
    r = renderer(sc)
    c = pf_synth.make_cameras("tiny")[0]
    c.fx = 0.0
    with pytest.raises(pf.PFError) as e:
        r.forward([c])
    assert e.value.status == 1
    c = pf_synth.make_cameras("tiny")[0]
    c.near = -1.0
    with pytest.raises(pf.PFError):
        r.forward([c])
    r.close()


# --------------------------------------------------------------- dipoles (NEXT-1)

@pytest.mark.parametrize("name,variant", [("tiny+dipoles", "outside"), ("tiny+dipoles", "inside"),
                                          ("small+dipoles", None), ("small360+dipoles", None)])
def test_dipole_forward_and_backward_full_image(name, variant):
    sc, cams = case(name, variant)
    r = renderer(sc)
    cams = cams[:2]
    H, W = cams[0].height, cams[0].width
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    mode = oracle.O1 if name.startswith("tiny") else oracle.O3
    for v, cam in enumerate(cams):
        ref = oracle.render(sc, cam, mode=mode)["out"]
        assert np.abs(out[v] - ref).max() <= IMG_TOL
    g = pf_synth.make_grad_out(len(cams), H, W, seed=13)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    assert "normals" in got
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=mode)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()


def test_dipole_large_sampled_pixels():
    sc, cams = case("nerfsynth200k+dipoles")
    r = renderer(sc, flags=0)
    H, W = cams[0].height, cams[0].width
    rng = np.random.default_rng(2)
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    g = np.zeros((len(cams), H, W, 4), np.float32)
    pix = {}
    for v in (0, len(cams) - 1):
        p = np.unique(np.stack([rng.integers(0, W, 1500), rng.integers(0, H, 1500)], 1), axis=0)
        pix[v] = p
        ref = oracle.render(sc, cams[v], mode=oracle.O3, pixels=p)["out"]
        assert np.abs(out[v][p[:, 1], p[:, 0]] - ref).max() <= IMG_TOL
        g[v, p[:, 1], p[:, 0]] = rng.standard_normal((p.shape[0], 4)).astype(np.float32)
    r.forward(cams)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, p in pix.items():
        o = oracle.backward(sc, cams[v], g[v, p[:, 1], p[:, 0]], mode=oracle.O3, pixels=p)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(cams[v], p) for v, p in pix.items()]))
    r.close()


def test_dipole_validation_rejects_zero_normal():
    import paper_2604_24994_b200 as pf
    sc, _ = case("tiny+dipoles", "outside")
    bad = sc.copy()
    bad.normals[5] = 0.0
    with pytest.raises(pf.PFError) as e:
        renderer(bad)
    assert e.value.status == 1


@pytest.mark.parametrize("name", ["small", "small360+dipoles"])
def test_forward_by_products_match_oracle(name):
    """NEXT-1 by-products of the forward: per-cell sum T alpha (and the L_normal term
    with dipoles) against the oracle, plus the telescoping identity on the GPU."""
    sc, cams = case(name)
    r = renderer(sc)
    N = sc.num_cells
    st = {"contrib": torch.zeros(N, device="cuda"),
          "normal": torch.zeros(N, device="cuda") if sc.normals is not None else None}
    out = r.forward(cams[:2], stats=st)
    c = st["contrib"].double().cpu().numpy()
    ref_c = np.zeros(N)
    ref_n = np.zeros(N)
    for cam in cams[:2]:
        o = oracle.cell_stats(sc, cam, mode=oracle.O3)
        ref_c += o["contrib"]
        if o["normal"] is not None:
            ref_n += o["normal"]
    assert np.linalg.norm(c - ref_c) <= 1e-4 * np.linalg.norm(ref_c)
    tel = (1.0 - out[..., 3].double()).sum().item()
    assert abs(c.sum() - tel) <= 1e-4 * tel
    if st["normal"] is not None:
        nn = st["normal"].double().cpu().numpy()
        assert np.linalg.norm(nn - ref_n) <= 1e-4 * np.linalg.norm(ref_n)
    r.close()


# --------------------------------------------------------------- NEXT-3: Čech graph

@pytest.mark.parametrize("name", ["tiny", "small", "small360"])
def test_cech_build_bit_exact_small(name):
    import paper_2604_24994_b200 as pf
    sc, _ = case(name)
    b = pf.CechBuilder()
    s = torch.from_numpy(sc.sites).cuda()
    r = torch.from_numpy(sc.radii).cuda()
    off, idx = b.build(s, r)
    o_off, o_idx = oracle.cech_rows(sc.sites, sc.radii)
    assert np.array_equal(off.cpu().numpy(), o_off)
    assert np.array_equal(idx.cpu().numpy(), o_idx)
    b.close()


def test_cech_build_1m_vs_generator_and_sampled_oracle_rows():
    import paper_2604_24994_b200 as pf
    sc, _ = case("train8_1m")
    b = pf.CechBuilder()
    s = torch.from_numpy(sc.sites).cuda()
    r = torch.from_numpy(sc.radii).cuda()
    off, idx = b.build(s, r)
    off, idx = off.cpu().numpy(), idx.cpu().numpy()
    rows = np.random.default_rng(0).choice(sc.num_cells, 200, replace=False)
    o_off, o_idx = oracle.cech_rows(sc.sites, sc.radii, rows=rows)
    for k, i in enumerate(rows):
        assert np.array_equal(idx[off[i]:off[i + 1]], o_idx[o_off[k]:o_off[k + 1]])
    # the generator's lists are the exact Čech complex too (Lemma L3): identical CSR
    assert np.array_equal(off, sc.nbr_offsets) and np.array_equal(idx, sc.nbr_indices)
    b.close()


def test_connect_loss_matches_oracle():
    import paper_2604_24994_b200 as pf
    sc, _ = case("small360")
    s = torch.from_numpy(sc.sites).cuda()
    r = torch.from_numpy(sc.radii).cuda()
    off = torch.from_numpy(sc.nbr_offsets).cuda()
    idx = torch.from_numpy(sc.nbr_indices).cuda()
    loss, gs, gr = pf.connect_loss(s, r, off, idx)
    ref = oracle.connect_loss(sc.sites, sc.radii, sc.nbr_offsets, sc.nbr_indices)
    for a, b_ in ((loss, ref["loss"]), (gs, ref["sites"]), (gr, ref["radii"])):
        a = a.double().cpu().numpy().reshape(-1)
        b_ = b_.reshape(-1)
        assert np.linalg.norm(a - b_) <= 1e-4 * np.linalg.norm(b_)


# --------------------------------------------------------------- NEXT-4: fisheye

def _fisheye_case(name, variant=None):
    sc, cams = case(name, variant)
    return sc, [pf_synth.fisheye(c, 200.0) for c in cams[:2]]


@pytest.mark.parametrize("name,variant", [("tiny", "outside"), ("tiny", "inside"),
                                          ("small360", None)])
def test_fisheye_binning_matches_oracle(name, variant):
    sc, cams = _fisheye_case(name, variant)
    r = renderer(sc)
    for cam in cams:
        g = r.debug_binning(cam)
        o = oracle.binning(sc, cam)
        assert np.array_equal(g["keybits"].cpu().numpy().view(np.uint32), o["keybits"])
        gk = g["keys"].cpu().numpy().view(np.uint64)
        gv = g["vals"].cpu().numpy().view(np.uint32)
        # fp64 tile tests with transcendental tile axes: identical up to borderline tiles
        gs = set(zip(gk.tolist(), gv.tolist()))
        os_ = set(zip(o["keys"].tolist(), o["vals"].tolist()))
        assert len(gs ^ os_) <= 1e-4 * max(len(os_), 1)
        assert np.all(gk[1:] >= gk[:-1])
    r.close()


@pytest.mark.parametrize("name,variant", [("tiny", "outside"), ("tiny", "inside"),
                                          ("small360", None), ("small+dipoles", None),
                                          ("small+detail", None)])
def test_fisheye_forward_backward(name, variant):
    sc, cams = _fisheye_case(name, variant)
    r = renderer(sc)
    H, W = cams[0].height, cams[0].width
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    mode = oracle.O1 if name.startswith("tiny") else oracle.O3
    for v, cam in enumerate(cams):
        ref = oracle.render(sc, cam, mode=mode)["out"]
        assert np.abs(out[v] - ref).max() <= IMG_TOL
    g = pf_synth.make_grad_out(len(cams), H, W, seed=17)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=mode)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()


# --------------------------------------------------------------- NEXT-2: detail sites

def _full_parity(sc, cams, mode, seed):
    r = renderer(sc)
    H, W = cams[0].height, cams[0].width
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    for v, cam in enumerate(cams):
        ref = oracle.render(sc, cam, mode=mode)["out"]
        assert np.abs(out[v] - ref).max() <= IMG_TOL
    g = pf_synth.make_grad_out(len(cams), H, W, seed=seed)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=mode)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    msgs = grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()
    return msgs


@pytest.mark.parametrize("name,variant", [("tiny+detail", "outside"), ("tiny+detail", "inside"),
                                          ("small+detail", None), ("small360+detail", None)])
def test_detail_forward_and_backward_full_image(name, variant):
    sc, cams = case(name, variant)
    mode = oracle.O1 if name.startswith("tiny") else oracle.O3
    _full_parity(sc, cams[:2], mode, seed=19)


@pytest.mark.parametrize("K", [1, 3])
def test_detail_fewer_sites(K):
    sc, cams = case("small")
    sc = pf_synth.add_detail(sc.copy(), K=K, seed=5)
    _full_parity(sc, cams[:1], oracle.O3, seed=21)


def test_detail_large_sampled_pixels():
    sc, cams = case("nerfsynth200k+detail")
    r = renderer(sc, flags=0)
    H, W = cams[0].height, cams[0].width
    rng = np.random.default_rng(4)
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    g = np.zeros((len(cams), H, W, 4), np.float32)
    pix = {}
    for v in (0, len(cams) - 1):
        p = np.unique(np.stack([rng.integers(0, W, 1200), rng.integers(0, H, 1200)], 1), axis=0)
        pix[v] = p
        ref = oracle.render(sc, cams[v], mode=oracle.O3, pixels=p)["out"]
        assert np.abs(out[v][p[:, 1], p[:, 0]] - ref).max() <= IMG_TOL
        g[v, p[:, 1], p[:, 0]] = rng.standard_normal((p.shape[0], 4)).astype(np.float32)
    r.forward(cams)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, p in pix.items():
        o = oracle.backward(sc, cams[v], g[v, p[:, 1], p[:, 0]], mode=oracle.O3, pixels=p)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(cams[v], p) for v, p in pix.items()]))
    r.close()


def test_detail_record_overflow_fallback(monkeypatch):
    monkeypatch.setenv("PF_REC_RATIO", "0.02")
    sc, cams = case("small360+detail")
    _full_parity(sc, cams[:1], oracle.O3, seed=23)


@pytest.mark.parametrize("ratio", ["0", "0.5"])
def test_detail_colour_slots_overflow(monkeypatch, ratio):
    """Split detail backward: K6's per-segment colour slots (K6 -> K7) missing for
    every record (ratio 0) or for part of them (0.5 slots per pair): K7 recomputes
    the colour and displaced face of those records; parity unchanged."""
    monkeypatch.setenv("PF_COL_RATIO", ratio)
    sc, cams = case("small360+detail")
    _full_parity(sc, cams[:1], oracle.O3, seed=29)


def test_detail_per_view_launches(monkeypatch):
    """The per-view launch path of 1080p views (K6 on two alternating streams, K7 and
    K7D per view) forced on a small scene (PF_K6_PER_VIEW=1): parity with the oracle
    unchanged."""
    monkeypatch.setenv("PF_K6_PER_VIEW", "1")
    sc, cams = case("small360+detail")
    _full_parity(sc, cams[:3], oracle.O3, seed=31)


def test_per_view_launches_plain(monkeypatch):
    monkeypatch.setenv("PF_K6_PER_VIEW", "1")
    sc, cams = case("small360")
    _full_parity(sc, cams[:3], oracle.O3, seed=37)


def test_detail_autograd_and_by_products():
    """torch.autograd through the detail parameters equals the explicit backward;
    by-products (sum T alpha) match the oracle's."""
    import paper_2604_24994_b200 as pf
    sc, cams = case("small+detail")
    r = renderer(sc)
    params = [p.detach().clone().requires_grad_(True) for p in r.params()]
    r2 = pf.Renderer(params[0], params[1], params[2], params[3], params[4],
                     *r._tensors[5:7], background=sc.background, normals=params[5],
                     detail=dict(r.detail, uv=params[6], disp=params[7], sv=params[8]))
    out = pf.render(r2, cams[:1])
    g = torch.from_numpy(pf_synth.make_grad_out(1, cams[0].height, cams[0].width, seed=3)).cuda()
    (out * g).sum().backward()
    ref = oracle.backward(sc, cams[0], g[0].cpu().numpy(), mode=oracle.O3)
    grad_check(dict(zip(r2.param_names, [p.grad for p in params])), ref, ctx=(sc, [(cams[0], None)]))
    N = sc.num_cells
    st = {"contrib": torch.zeros(N, device="cuda"), "normal": torch.zeros(N, device="cuda")}
    r.forward(cams[:1], stats=st)
    o = oracle.cell_stats(sc, cams[0], mode=oracle.O3)
    c = st["contrib"].double().cpu().numpy()
    assert np.linalg.norm(c - o["contrib"]) <= 1e-4 * np.linalg.norm(o["contrib"])
    r.close(); r2.close()


def test_detail_abi_errors():
    import paper_2604_24994_b200 as pf
    sc, _ = case("tiny+detail", "outside")
    base = pf.Renderer.from_scene(sc, "cuda")
    s, w, rr, d, c, o, i, n = base._tensors
    det = base.detail
    with pytest.raises(pf.PFError):       # detail without normals
        pf.Renderer(s, w, rr, d, c, o, i, detail=det)
    with pytest.raises(pf.PFError):       # tau <= 0
        pf.Renderer(s, w, rr, d, c, o, i, normals=n, detail=dict(det, tau=0.0))
    bad = sc.copy()
    bad.detail.sv[3, 2, 1, 0] = np.nan
    with pytest.raises(pf.PFError):       # PF_VALIDATE catches non-finite detail values
        renderer(bad)
    sv_off = torch.zeros(det["sv"].numel() + 1, device="cuda")[1:].view(det["sv"].shape)
    with pytest.raises(pf.PFError):       # misaligned (float4 loads need 16-byte alignment)
        pf.Renderer(s, w, rr, d, c, o, i, normals=n, detail=dict(det, sv=sv_off))
    base.close()


# --------------------------------------------------------------- edge cases

def _parity_one(sc, cams, mode=oracle.O3, seed=29, flags=None):
    r = renderer(sc, flags)
    H, W = cams[0].height, cams[0].width
    out = r.forward(cams).cpu().numpy().astype(np.float64)
    for v, cam in enumerate(cams):
        ref = oracle.render(sc, cam, mode=mode)["out"]
        assert np.abs(out[v] - ref).max() <= IMG_TOL
    g = pf_synth.make_grad_out(len(cams), H, W, seed=seed)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=mode)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    grad_check(got, ref, ctx=(sc, [(c, None) for c in cams]))
    r.close()
    return out


@pytest.mark.parametrize("W,H", [(37, 23), (1, 1), (17, 200), (130, 9)])
def test_edge_odd_image_sizes(W, H):
    """Images that are not multiples of the 16x16 tile nor of the 8x4 warp block."""
    sc, cams = case("small")
    cam = cams[0]
    s = min(W / cam.width, H / cam.height)
    c = pf_synth.Camera(W, H, cam.fx * s, cam.fy * s, W / 2.0, H / 2.0, cam.c2w.copy(), cam.near)
    _parity_one(sc, [c])


def test_edge_no_pairs_camera_looking_away():
    """No cell in view: background with T = 1 everywhere and zero gradients."""
    sc, cams = case("small")
    cam = cams[0]
    M = np.asarray(cam.c2w, np.float32).reshape(3, 4).copy()
    M[:, :3] = -M[:, :3]          # flip the viewing direction (keeps a rotation: det = -1?)
    M[:, 0] = -M[:, 0]            # restore a proper rotation
    eye = M[:, 3]
    M[:, 3] = eye * 3.0           # far outside the foam, looking outward
    c = pf_synth.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, M.reshape(12), cam.near)
    sc2 = sc.copy()
    sc2.background = (0.25, 0.5, 0.75)
    r = renderer(sc2)
    out = r.forward([c]).cpu().numpy()
    assert r.pair_counts(1) == [0]
    assert np.array_equal(out[0, ..., 3], np.ones((c.height, c.width), np.float32))
    assert np.allclose(out[0, ..., :3], np.float32([0.25, 0.5, 0.75]), atol=0)
    g = torch.from_numpy(pf_synth.make_grad_out(1, c.height, c.width, seed=1)).cuda()
    got = r.backward([c], g)
    for k in ("sites", "weights", "radii", "density", "rgb"):
        assert float(got[k].abs().max()) == 0.0
    r.close()


def test_edge_single_cell():
    """N = 1, no neighbours (E = 0): the bounded cell is the sphere."""
    from helpers import camera, scene_from
    sc = scene_from([[0.05, -0.02, 0.1]], radii=[0.4], density=[3.0], rgb=[[0.2, 0.7, 0.4]],
                    bg=(0.1, 0.1, 0.1))
    _parity_one(sc, [camera(W=48, H=40, f=60.0)], mode=oracle.O1)


def test_edge_dense_single_tile_long_list():
    """Thousands of cells behind one 16x16 tile: a list spanning ~100 chunks of 32,
    most of them culled per warp, and early termination deep in the list."""
    rng = np.random.default_rng(5)
    n = 3000
    P = rng.normal(scale=0.15, size=(n, 3)).astype(np.float32)
    r, off, idx = pf_synth.knn_cech_lists(P, 8, rng, cech_filter=True)
    from helpers import scene_from, camera
    sc = scene_from(P, r, density=np.full(n, 25.0, np.float32),
                    rgb=rng.uniform(0, 1, size=(n, 3)).astype(np.float32), lists=(off, idx))
    cam = camera(W=16, H=16, f=30.0, eye=(0.0, 0.0, -2.0))
    r_ = renderer(sc)
    b = r_.debug_binning(cam)
    assert b["P"] > 0.8 * n      # (nearly) every cell lands in the one tile
    r_.close()
    _parity_one(sc, [cam])


# --------------------------------------------------------------- bench configurations

def test_static_inference_mip360_1m():
    """The render-FPS handle of bench.py (PF_STATIC_SCENE | PF_INFERENCE: edge records
    built once at creation, no backward state) on mip360_1m: bit-identical to the
    training handle's image on every call, and the oracle on sampled pixels (3000 vs
    O3 tile lists, 24 vs O1 all-pairs)."""
    import paper_2604_24994_b200 as pf
    sc, cams = case("mip360_1m")
    rs = renderer(sc, flags=pf.PF_STATIC_SCENE | pf.PF_INFERENCE)
    a = rs.forward(cams).cpu().numpy()
    b = rs.forward(cams).cpu().numpy()          # second call: cached edge records
    r0 = renderer(sc, flags=0)
    c = r0.forward(cams).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)
    cam = cams[0]
    rng = np.random.default_rng(7)
    pix = np.stack([rng.integers(0, cam.width, 3000), rng.integers(0, cam.height, 3000)], 1)
    ref = oracle.render(sc, cam, mode=oracle.O3, pixels=pix)["out"]
    assert np.abs(a[0][pix[:, 1], pix[:, 0]] - ref).max() <= IMG_TOL
    few = pix[:24]
    ref1 = oracle.render(sc, cam, mode=oracle.O1, pixels=few)["out"]
    assert np.abs(a[0][few[:, 1], few[:, 0]] - ref1).max() <= IMG_TOL
    rs.close()
    r0.close()


def test_sweep64_3m_binning_and_sampled_pixels():
    """sweep64_3m (3M cells, 64 views at 1080p) in the bench's launch configuration:
    one 64-view call of the static inference handle (sorted in batches of 8 views).
    Binning bit-exact on two views; views 0 and 63 against the oracle on 2000
    sampled pixels each."""
    import paper_2604_24994_b200 as pf
    sc, cams = case("sweep64_3m")
    assert len(cams) == 64 and sc.num_cells == 3_000_000
    r = renderer(sc, flags=pf.PF_STATIC_SCENE | pf.PF_INFERENCE)
    for cam in (cams[0], cams[63]):
        g = r.debug_binning(cam)
        o = oracle.binning(sc, cam)
        assert g["P"] == o["P"]
        assert np.array_equal(g["keys"].cpu().numpy().view(np.uint64), o["keys"])
        assert np.array_equal(g["vals"].cpu().numpy().view(np.uint32), o["vals"])
        assert np.array_equal(g["ranges"].cpu().numpy().view(np.uint32), o["ranges"])
    out = r.forward(cams)
    assert bool(torch.isfinite(out).all())
    rng = np.random.default_rng(8)
    for v in (0, 63):
        cam = cams[v]
        pix = np.stack([rng.integers(0, cam.width, 2000), rng.integers(0, cam.height, 2000)], 1)
        got = out[v].cpu().numpy().astype(np.float64)[pix[:, 1], pix[:, 0]]
        ref = oracle.render(sc, cam, mode=oracle.O3, pixels=pix)["out"]
        assert np.abs(got - ref).max() <= IMG_TOL, v
    # a view rendered alone equals its slot of the 64-view call, bit for bit
    one = r.forward([cams[63]]).cpu().numpy()[0]
    assert np.array_equal(one, out[63].cpu().numpy())
    r.close()


def test_train8_1m_full_frame_image_and_dense_gradients():
    """One FULL 1080p frame of train8_1m (all 2,073,600 pixels) in the bench's launch
    configuration (8 views in one call): image within 1e-4 of the oracle (O3) at every
    pixel; dense dL/dimage on that view (zero on the others) and the C17 gradient bar,
    every failing cell listed with its conditioning."""
    sc, cams = case("train8_1m")
    r = renderer(sc, flags=0)
    out = r.forward(cams)
    img = out[0].cpu().numpy().astype(np.float64)
    ref = oracle.render(sc, cams[0], mode=oracle.O3)["out"]
    err = np.abs(img - ref)
    assert err.max() <= IMG_TOL, (err.max(), np.unravel_index(err.argmax(), err.shape))
    H, W = cams[0].height, cams[0].width
    g = np.zeros((len(cams), H, W, 4), np.float32)
    g[0] = pf_synth.make_grad_out(1, H, W, seed=41)[0]
    got = r.backward(cams, torch.from_numpy(g).cuda())
    gref = oracle.backward(sc, cams[0], g[0], mode=oracle.O3)
    print(grad_check(got, gref, ctx=(sc, [(cams[0], None)])))
    r.close()


def test_fused_and_per_view_launches_agree(monkeypatch):
    """K6 / K7 of all views in one fused launch (small views, arguments in shared
    memory) vs one launch per view (arguments by value): bit-identical images and the
    same gradients up to atomic summation order (PF_K6_PER_VIEW=0 / 1)."""
    sc, cams = case("small360")
    cams = cams[:4]
    H, W = cams[0].height, cams[0].width
    g = torch.from_numpy(pf_synth.make_grad_out(len(cams), H, W, seed=37)).cuda()
    res = {}
    for knob in ("0", "1"):
        monkeypatch.setenv("PF_K6_PER_VIEW", knob)
        r = renderer(sc, flags=0)
        out = r.forward(cams).cpu().numpy()
        grads = {k: v.detach().cpu().numpy().astype(np.float64)
                 for k, v in r.backward(cams, g).items()}
        res[knob] = (out, grads)
        r.close()
    assert np.array_equal(res["0"][0], res["1"][0])
    for k, a in res["0"][1].items():
        b = res["1"][1][k]
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b) + 1e-30, k


def test_detail_colour_queue_bit_identical(tmp_path):
    """K6's deferred colour evaluation (ColQueue, DESIGN §13 item 4) composites every
    pixel's colours in list order with composite_step's fmaf: the image must be
    bit-identical to the in-line evaluation (a PF_K6D_QUEUE=0 build of the same
    sources, run in a subprocess), for K = 8 and a generic K."""
    import subprocess
    import sys
    from paper_2604_24994_b200 import _build
    lib = _build.build(out=str(tmp_path / "q0.so"), defines=("PF_K6D_QUEUE=0",))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for name, K in (("small360", 8), ("small", 3)):
        sc = pf_synth.add_detail(pf_synth.make_scene(name), K=K, seed=5)
        cams = pf_synth.make_cameras(name)[:2]
        r = renderer(sc, flags=0)
        ref = r.forward(cams).cpu().numpy()
        r.close()
        dump = str(tmp_path / f"{name}.npy")
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import pf_synth; "
                "import paper_2604_24994_b200 as pf; "
                "sc = pf_synth.add_detail(pf_synth.make_scene(%r), K=%d, seed=5); "
                "cams = pf_synth.make_cameras(%r)[:2]; "
                "r = pf.Renderer.from_scene(sc, 'cuda:0'); "
                "np.save(%r, r.forward(cams).cpu().numpy())") % (root, name, K, name, dump)
        out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "PF_LIBRARY_PATH": lib},
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        got = np.load(dump)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), name
