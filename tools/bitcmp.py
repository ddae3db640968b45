"""Bit-level comparison of two library variants (A/B of exact rewrites).
  PF_LIBRARY_PATH=<so> python tools/bitcmp.py dump <tag> <preset> [detail K] [views]
  python tools/bitcmp.py cmp <tagA> <tagB>
dump: forward images of the preset's first views (fwd only: the image is deterministic;
gradients use atomics) to gpurun_out/bitcmp_<tag>.npy."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out_dir = os.path.join(ROOT, "gpurun_out")
if sys.argv[1] == "dump":
    import torch
    import paper_2604_24994_b200 as pf
    import pf_synth
    tag, preset = sys.argv[2], sys.argv[3]
    K = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    nv = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    sc = pf_synth.make_scene(preset, detail=K) if K else pf_synth.make_scene(preset)
    cams = pf_synth.make_cameras(preset)[:nv]
    r = pf.Renderer.from_scene(sc, "cuda:0")
    out = r.forward(cams).cpu().numpy()
    np.save(os.path.join(out_dir, f"bitcmp_{tag}.npy"), out)
    print("dumped", tag, out.shape)
else:
    a = np.load(os.path.join(out_dir, f"bitcmp_{sys.argv[2]}.npy"))
    b = np.load(os.path.join(out_dir, f"bitcmp_{sys.argv[3]}.npy"))
    same = np.array_equal(a.view(np.uint32), b.view(np.uint32))
    print(sys.argv[2], "vs", sys.argv[3], "bit-identical" if same else
          f"DIFFER: {int((a != b).sum())} values, max abs {float(np.abs(a - b).max())}")
