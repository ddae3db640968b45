"""Multi-process (world_size 2, gloo, CPU) test of the view sharding + gradient
all-reduce logic of paper_2604_24994_b200.dist, with the CPU oracle's
gradients standing in for the GPU backward (SURVEY §4 tier T5')."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views():
    import pf_synth
    sc = pf_synth.make_scene("tiny")
    import math
    cams = []
    for k in range(5):
        az = 2 * math.pi * k / 5
        eye = (3.5 * math.cos(az), 3.5 * math.sin(az), 0.7)
        cams.append(pf_synth.Camera(48, 40, 60.0, 60.0, 24.0, 20.0,
                                    pf_synth.look_at(eye, (0, 0, 0)), 0.05))
    g = pf_synth.make_grad_out(len(cams), 40, 48, seed=3)
    return sc, cams, g


def _oracle_bwd(sc, cams, g):
    import oracle

    def fn(v, flat):
        r = oracle.backward(sc, cams[v], g[v], mode=oracle.O2)
        flat += torch.from_numpy(np.concatenate([r["sites"].ravel(), r["weights"], r["radii"],
                                                 r["density"], r["rgb"].ravel()]))
    return fn


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2604_24994_b200 import dist as pfd
    sc, cams, g = _views()
    mine = pfd.shard_views(range(len(cams)), ws, rank)
    flat = torch.zeros(9 * sc.num_cells, dtype=torch.float64)
    pfd.sharded_backward(mine, _oracle_bwd(sc, cams, g), flat)
    q.put((rank, mine, flat.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_views_partition():
    from paper_2604_24994_b200 import dist as pfd
    for ws in (1, 2, 3, 8):
        got = sorted(v for r in range(ws) for v in pfd.shard_views(list(range(64)), ws, r))
        assert got == list(range(64))
    assert pfd.shard_views(list(range(8)), 2, 1) == [1, 3, 5, 7]
    with pytest.raises(ValueError):
        pfd.shard_views([1], 2, 2)


def test_sharded_allreduce_equals_single_process_sum():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == [0, 2, 4] and res[1][1] == [1, 3]
    sc, cams, g = _views()
    ref = torch.zeros(9 * sc.num_cells, dtype=torch.float64)
    fn = _oracle_bwd(sc, cams, g)
    for v in range(len(cams)):
        fn(v, ref)
    for _, _, flat in res:   # every rank holds the same reduced gradient
        np.testing.assert_allclose(flat, ref.numpy(), rtol=1e-12, atol=1e-15)
    assert np.abs(ref.numpy()).max() > 0
