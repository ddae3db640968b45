"""SURVEY §4 T5 on a one-GPU box: two ranks (processes) share cuda:0 over the gloo
backend and run the data-parallel step of paper_2604_24994_b200.dist exactly as
bench.py does (views dealt round-robin, one all-reduce of the flat gradient buffer).
Per-view images must be bit-identical to a single-process render (the forward is
deterministic) and the all-reduced gradients equal the single-process accumulation
over all views within the C17 bar."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import pf_synth
    sc = pf_synth.make_scene("small360")
    cams = pf_synth.make_cameras("small360", n=6)
    H, W = cams[0].height, cams[0].width
    g = pf_synth.make_grad_out(len(cams), H, W, seed=23)
    return sc, cams, g


def _worker(rank, ws, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    import paper_2604_24994_b200 as pf
    from paper_2604_24994_b200 import dist as pfd
    sc, cams, g = _setup()
    mine = pfd.shard_views(list(range(len(cams))), ws, rank)
    r = pf.Renderer.from_scene(sc, "cuda:0", flags=0)
    flat = torch.zeros(r.grad_size, device="cuda:0")
    gl = torch.from_numpy(g[mine]).cuda()
    img, flat = pfd.train_step(r, [cams[v] for v in mine], gl, flat)
    torch.cuda.synchronize()
    q.put((rank, mine, img.cpu().numpy(), flat.cpu().numpy()))
    dist.barrier()
    r.close()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_process():
    import torch.multiprocessing as mp
    import paper_2604_24994_b200 as pf
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((x[0], x[1:]) for x in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    sc, cams, g = _setup()
    r = pf.Renderer.from_scene(sc, "cuda:0", flags=0)
    img = r.forward(cams).cpu().numpy()
    ref = r.backward(cams, torch.from_numpy(g).cuda())
    flat_ref = np.concatenate([ref[k].detach().cpu().numpy().reshape(-1) for k in r.param_names])
    r.close()
    for rank, (mine, im, flat) in res.items():
        assert mine == list(range(rank, len(cams), 2))
        for k, v in enumerate(mine):
            assert np.array_equal(im[k], img[v]), (rank, v)   # deterministic forward
        # every rank holds the same all-reduced sum == the one-process accumulation
        rel = np.linalg.norm(flat - flat_ref) / np.linalg.norm(flat_ref)
        assert rel <= 1e-5, rel
