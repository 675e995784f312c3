"""Head sharding on CPU with world_size 2 over gloo.

Each rank owns a contiguous range of heads (pipeline.shard_heads): GEMM-Q and
K/V are column-parallel, attention and the feature cache are per head, and
GEMM-O is row-parallel; the partial outputs — including each rank's partial
cached bias — are summed by one all-reduce. The per-rank compute here is the
oracle (the CPU restatement); the test checks the decomposition is exact:
sharded + all-reduce == unsharded, and that per-head symbols, skipped-tile
sets and bias orders do not depend on the sharding."""

import os
import pathlib
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = pathlib.Path(__file__).resolve().parents[1]
T = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(seed=0):
    import oracle

    rng = np.random.default_rng(seed)
    n, dm, H, order = 256, 64, 4, 1
    t = n // T
    o_hist = [rng.standard_normal((H, n, T)).astype(np.float32) for _ in range(order + 1)]
    o_disp = rng.standard_normal((H, n, T)).astype(np.float32)
    w_out = (rng.standard_normal((H, T, dm)) * T ** -0.5).astype(np.float32)
    active = rng.random((t, H)) < 0.5
    cb = np.zeros((H, t), bool)
    sb = np.zeros((H, t, t), bool)
    for h in range(H):
        cb[h], sb[h] = oracle.random_masks(rng, t, t, 1, density=0.5, cache_density=0.6)
    return dict(n=n, dm=dm, H=H, order=order, t=t, o_hist=o_hist, o_disp=o_disp, w_out=w_out,
                active=active, cb=cb, sb=sb)


def _gemm_o(P, heads):
    """Update + dispatch GEMM-O over a subset of heads (oracle restatement)."""
    import oracle

    t, order = P["t"], P["order"]
    stacks = [[None] * t for _ in heads]
    valid = [[0] * t for _ in heads]
    for o in P["o_hist"]:
        for a, h in enumerate(heads):
            for i in range(t):
                stacks[a][i], valid[a][i] = oracle.update_entry(stacks[a][i], valid[a][i],
                                                                o[h, i * T:(i + 1) * T], order)
    act = P["active"][:, heads]
    out_u, bias, orders = oracle.project_out_update(P["o_hist"][-1][heads], P["w_out"][heads], act,
                                                    stacks, valid, order, T)
    out_d = oracle.project_out_dispatch(P["o_disp"][heads], P["w_out"][heads], act, bias, orders,
                                        2, 5, order, T)
    return out_u, out_d, orders


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2509_25401_b200.pipeline import shard_heads

        P = _problem()
        heads = shard_heads(P["H"], world, rank)
        out_u, out_d, orders = _gemm_o(P, heads)
        tu, td = torch.from_numpy(out_u), torch.from_numpy(out_d)
        dist.all_reduce(tu)
        dist.all_reduce(td)
        # per-head symbol bytes and skipped-tile sets are rank-local
        sym = [oracle.build_symbols(P["cb"][h], P["sb"][h], 1) for h in heads]
        pairs = sum(int(P["sb"][h][P["cb"][h]].sum()) for h in heads)
        tp = torch.tensor([pairs])
        dist.all_reduce(tp)
        q.put((rank, tu.numpy(), td.numpy(), orders, [s.s_s for s in sym], int(tp.item())))
    finally:
        dist.destroy_process_group()


def test_head_sharded_gemm_o_allreduce_equals_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, str(ROOT))
    import oracle

    P = _problem()
    full_u, full_d, full_orders = _gemm_o(P, list(range(P["H"])))
    for rank, tu, td, orders, ss, pairs in res:
        # all-reduce of partial projections == one dense projection (fp32 reassociation)
        assert np.abs(tu - full_u).max() / np.abs(full_u).max() < 1e-5
        assert np.abs(td - full_d).max() / np.abs(full_d).max() < 1e-5
        assert pairs == int(sum(P["sb"][h][P["cb"][h]].sum() for h in range(P["H"])))
        from paper_2509_25401_b200.pipeline import shard_heads

        for a, h in enumerate(shard_heads(P["H"], world, rank)):
            assert ss[a] == oracle.build_symbols(P["cb"][h], P["sb"][h], 1).s_s
    # ranks agree bit-for-bit after the all-reduce
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
