"""Driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over
the hot path on small scenes: tiny and a 5k-cell mip360-shaped foam,
plain, dipole, detail-site and fisheye variants, forward + backward through the
C-ABI, plus the Čech build and L_connect.  Exits non-zero on any API error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_24994_b200 as pf  # noqa: E402
import pf_synth  # noqa: E402


def run(sc, cams, tag):
    r = pf.Renderer.from_scene(sc, "cuda", flags=0)
    out = r.forward(cams)
    H, W = cams[0].height, cams[0].width
    g = torch.from_numpy(pf_synth.make_grad_out(len(cams), H, W, seed=5)).cuda()
    grads = r.backward(cams, g)
    stats = {"contrib": torch.zeros(sc.num_cells, device="cuda"),
             "normal": torch.zeros(sc.num_cells, device="cuda")}
    r.forward(cams, stats=stats)
    torch.cuda.synchronize()
    ri = r.sibling(pf.PF_INFERENCE | pf.PF_STATIC_SCENE)
    ri.forward(cams)
    ri.forward(cams)
    img, st = ri.trace(cams, stats=True)     # NEXT-4 tracer (static scene: cached BVH)
    ri.trace(cams)
    torch.cuda.synchronize()
    print(tag, "ok", float(out.sum()), float(grads["sites"].abs().sum()), flush=True)
    ri.close()
    r.close()


def main():
    which = sys.argv[1:] or ["tiny", "small5k"]
    for name in which:
        if name == "tiny":
            sc = pf_synth.make_scene("tiny")
            cams = pf_synth.make_cameras("tiny")
        else:
            sc = pf_synth.make_scene("small360", num_cells=5000)
            cams = pf_synth.make_cameras("small360", n=2, width=160, height=96)
        run(sc, cams, name)
        run(pf_synth.add_dipoles(sc.copy()), cams, name + "+dipoles")
        run(pf_synth.add_detail(pf_synth.add_dipoles(sc.copy())), cams, name + "+detail")
        run(sc, [pf_synth.fisheye(c, 200.0) for c in cams], name + "+fisheye")
        cb = pf.CechBuilder()
        s_ = torch.from_numpy(sc.sites).cuda()
        r_ = torch.from_numpy(sc.radii).cuda()
        off, idx = cb.build(s_, r_)
        loss, gs, gr = pf.connect_loss(s_, r_, off, idx)
        torch.cuda.synchronize()
        print(name, "cech ok", int(idx.numel()), float(loss.sum()), flush=True)
        cb.close()
    # release PyTorch's cached blocks so the leak check sees only the library's memory
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
