"""Multi-rank path on CPU (gloo, world size 2): the giant-range partition the
library uses (helrm_dist_range, host-only) applied to the oracle's lookup --
each rank computes the partial Q_l P accumulators of its giant pairs, a
uint64 SUM all-reduce plus mod q combines them, and the finished ciphertext
is bit-identical to the single-process lookup (only exact
modular sums are split)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import core
from oracle import lookup as lk


def _worker(rank, world, name, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    core.set_threads(2)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_18150_b200 import helrm
        w = synth.make_workload(name)
        cfg = w.config
        P = core.params_from_config(cfg)
        lay = lk.layout(w)
        plan = lk.make_plan(lay, P.n, cfg.level)
        sk = core.sk_gen(P, cfg.seed)
        pk = core.pk_gen(P, sk, cfg.seed)
        rk = core.rotkeys_gen(P, sk, plan.galois(P), cfg.seed)
        u = lk.encode_plan(P, plan)
        # the query is encrypted on rank 0 and broadcast (coefficient words)
        cts = lk.query_cts(P, pk, lay, plan, w.indices[0], w.dense[0], cfg.level, cfg.seed, 0)
        for ct in cts:
            for arr in (ct.c0, ct.c1):
                t = torch.from_numpy(arr.view(np.int64).copy())
                dist.broadcast(t, 0)
                arr[...] = t.numpy().view(np.uint64)
        lo, hi = helrm.dist_range(len(lk.giant_pairs(plan)), world, rank)
        O = lk.lookup_partial(P, plan, u, rk, cts, lo, hi)
        qp = np.array(P.qp(cfg.level), dtype=np.uint64).reshape(-1, 1)
        red = []
        for (O0, O1) in O:
            pair = []
            for arr in (O0, O1):
                t = torch.from_numpy(arr.view(np.int64).copy())
                dist.all_reduce(t, op=dist.ReduceOp.SUM)       # < world q < 2^63: exact in int64
                pair.append(t.numpy().view(np.uint64) % qp)
            red.append(tuple(pair))
        out = lk.lookup_finish(P, plan, rk, red, cts[0].scale)
        full = lk.lookup(P, plan, u, rk, cts)
        ok = all(np.array_equal(a.c0, b.c0) and np.array_equal(a.c1, b.c1) for a, b in zip(out, full))
        z = np.concatenate([core.decrypt_decode(P, sk, ct) for ct in out])
        err = float(np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max())
        q.put((rank, lo, hi, ok, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,port", [("uci", 29531), ("llm_small", 29533), ("criteo_c2_small", 29535)])
def test_giant_partition_allreduce_is_bit_exact(name, port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, name, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] > res[1][1]   # contiguous cover
    for rank, lo, hi, ok, err in res:
        assert ok, f"rank {rank}: distributed result differs from the single-process lookup"
        assert err < 1e-3
