"""GPU parity of the NEXT-4 adjacency-walk ray tracer (pf_trace_forward) against
the oracle's tracer and against the GPU rasterizer: the paper's two renderers give
the same image (Fig. 1) -- within the image bar 1e-4."""
import numpy as np
import pytest

import oracle
import pf_synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4


def _scene(name):
    if name == "tiny":
        return pf_synth.make_scene("tiny"), pf_synth.make_cameras("tiny")
    if name == "tiny_inside":
        return pf_synth.make_scene("tiny"), pf_synth.make_cameras("tiny", variant="inside")
    if name == "small360":
        return pf_synth.make_scene("small360"), pf_synth.make_cameras("small360", n=4)
    if name == "small+dipoles":
        return pf_synth.add_dipoles(pf_synth.make_scene("small")), pf_synth.make_cameras("small")
    if name == "small+detail":
        return pf_synth.make_scene("small", detail=8), pf_synth.make_cameras("small")
    raise KeyError(name)


def _renderer(sc, flags=0):
    import paper_2604_24994_b200 as pf
    return pf.Renderer.from_scene(sc, "cuda", flags=flags)


@pytest.mark.parametrize("name", ["tiny", "tiny_inside", "small360", "small+dipoles",
                                  "small+detail"])
@pytest.mark.parametrize("fish", [False, True])
def test_trace_equals_oracle_and_raster(name, fish):
    sc, cams = _scene(name)
    if fish:
        cams = [pf_synth.fisheye(c, 200.0) for c in cams]
    cams = cams[:2]
    r = _renderer(sc)
    img, st = r.trace(cams, stats=True)
    img = img.cpu().numpy().astype(np.float64)
    ras = r.forward(cams).cpu().numpy().astype(np.float64)
    assert np.abs(img - ras).max() <= IMG_TOL
    vis = 0
    for v, cam in enumerate(cams):
        o = oracle.trace(sc, cam)
        assert np.abs(img[v] - o["out"]).max() <= IMG_TOL, v
        vis += int(o["stats"][..., 0].sum())
    assert st["diverged"] == 0
    npx = sum(c.width * c.height for c in cams)
    assert (st["rays"] == npx) if not fish else (0 < st["rays"] <= npx)
    # the walk visits the cells the oracle's walk visits (fp32 slivers aside)
    assert abs(st["visited"] - vis) <= 0.01 * vis + 8
    r.close()


def test_trace_static_scene_cached_bvh():
    import paper_2604_24994_b200 as pf
    sc, cams = _scene("small360")
    rs = _renderer(sc, flags=pf.PF_STATIC_SCENE | pf.PF_INFERENCE)
    a = rs.trace(cams).cpu().numpy()
    b = rs.trace(cams).cpu().numpy()       # the cached BVH and edge records
    r0 = _renderer(sc)
    c = r0.trace(cams).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)
    rs.close()
    r0.close()


def test_trace_1080p_equals_raster():
    """train8_1m, two 1080p views in one call: the traced images equal the (oracle-
    pinned) rasterized ones within the image bar at every pixel."""
    sc = pf_synth.make_scene("train8_1m")
    cams = pf_synth.make_cameras("train8_1m")[:2]
    r = _renderer(sc)
    img, st = r.trace(cams, stats=True)
    ras = r.forward(cams)
    err = float((img - ras).abs().max())
    assert err <= IMG_TOL, err
    assert st["diverged"] == 0 and st["rays"] == 2 * 1920 * 1080
    rng = np.random.default_rng(3)
    pix = np.stack([rng.integers(0, 1920, 300), rng.integers(0, 1080, 300)], 1)
    o = oracle.trace(sc, cams[0], pixels=pix)["out"]
    got = img[0].cpu().numpy().astype(np.float64)[pix[:, 1], pix[:, 0]]
    assert np.abs(got - o).max() <= IMG_TOL
    r.close()


def test_trace_argument_errors():
    import paper_2604_24994_b200 as pf
    sc, cams = _scene("tiny")
    r = _renderer(sc)
    with pytest.raises(ValueError):
        r.trace(cams, out=torch.empty((1, 8, 8, 4), device="cuda"))
    bad = pf_synth.make_cameras("tiny")[0]
    bad.fx = -1.0
    with pytest.raises(pf.PFError) as e:
        r.trace([bad])
    assert e.value.status == 1
    r.close()
