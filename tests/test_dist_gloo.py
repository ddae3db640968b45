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


def _bench_worker(rank, ws, port, q):
    """bench.py's own view deal and whole-job FPS arithmetic under a real
    2-rank process group (gloo stands in for NCCL)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench

    def red(x, op):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    res = {}
    for wl, scaling in (("train8_1m", "strong"), ("sweep64_3m", "strong"),
                        ("train8_1m", "weak"), ("nerfsynth200k", "strong")):
        total, idx = bench.plan_views(wl, None, scaling, ws, rank)
        cams, total2 = bench.workload_cameras(wl, None, scaling, ws, rank)
        assert total2 == total and len(cams) == len(idx)
        ms_local = 10.0 + 5.0 * rank          # rank 1 is the slow one
        fps, n, ms = bench.aggregate_fps(len(idx), ms_local,
                                         lambda x: red(x, dist.ReduceOp.SUM),
                                         lambda x: red(x, dist.ReduceOp.MAX))
        res[(wl, scaling)] = (total, idx, fps, n, ms,
                              [float(c.c2w[3]) for c in cams])
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_view_deal_and_fps_arithmetic_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import bench
    expect_total = {("train8_1m", "strong"): 8, ("sweep64_3m", "strong"): 64,
                    ("train8_1m", "weak"): 16, ("nerfsynth200k", "strong"): 8}
    for key, total in expect_total.items():
        r0, r1 = res[0][key], res[1][key]
        assert r0[0] == r1[0] == total
        # rank r gets v = r (mod N); together a partition of the batch
        assert r0[1] == list(range(0, total, 2)) and r1[1] == list(range(1, total, 2))
        # whole-job frames/s = all views / the slowest rank's step (max over ranks)
        for r in (r0, r1):
            assert r[3] == total and r[4] == 15.0
            assert abs(r[2] - total / 0.015) < 1e-9
        # the dealt cameras are the single-process batch's cameras at those indices
        cams = bench.orbit_cameras(key[0], total)
        got = dict(zip(r0[1], r0[5]))
        got.update(zip(r1[1], r1[5]))
        assert [got[i] for i in range(total)] == [float(c.c2w[3]) for c in cams]
    # strong scaling: the 8-view batch is the 1-GPU batch (same cameras at any N)
    one, _ = bench.plan_views("train8_1m", None, "strong", 1, 0)
    assert one == 8
    with pytest.raises(SystemExit):
        bench.plan_views("mip360_1m", None, "strong", 2, 0)   # 1 view over 2 ranks
