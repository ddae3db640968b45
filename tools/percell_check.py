"""Per-cell secondary gradient check on several parity cases: counts
cells with |g_i - g_ref,i| > 1e-3 |g_ref,i| + 1e-5 max_k |g_ref,k| per array."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
import oracle, pf_synth
import paper_2604_24994_b200 as pf

def per_cell(got, ref, N):
    res = {}
    for k, b in ref.items():
        a = got[k].detach().cpu().numpy().astype(np.float64).reshape(N, -1)
        b = b.reshape(N, -1)
        na = np.linalg.norm(a - b, axis=1); nb = np.linalg.norm(b, axis=1)
        bad = na > 1e-3 * nb + 1e-5 * nb.max()
        res[k] = (int(bad.sum()), int((nb > 0).sum()))
    return res

cases = [("small", None, {}), ("small360", None, {}), ("small", None, {"dipoles": True}),
         ("small", None, {"detail": 8}), ("tiny", "inside", {})]
for name, var, kw in cases:
    sc = pf_synth.make_scene(name, **kw)
    cams = pf_synth.make_cameras(name, variant=var)[:2]
    r = pf.Renderer.from_scene(sc, "cuda")
    H, W = cams[0].height, cams[0].width
    r.forward(cams)
    g = pf_synth.make_grad_out(len(cams), H, W, seed=13)
    got = r.backward(cams, torch.from_numpy(g).cuda())
    ref = None
    for v, cam in enumerate(cams):
        o = oracle.backward(sc, cam, g[v], mode=oracle.O3)
        ref = o if ref is None else {k: ref[k] + o[k] for k in ref}
    print(name, var, kw, per_cell(got, ref, sc.num_cells))
