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


def _gather_rows(mine: np.ndarray, rp: int, nl: int, world: int) -> np.ndarray:
    """all-gather of every rank's padded row slice ([rp][N]) -> rows [0, nl)."""
    pad = np.zeros((rp, mine.shape[1]), dtype=np.uint64)
    pad[: mine.shape[0]] = mine
    parts = [torch.zeros(pad.shape, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(pad.view(np.int64).copy()))
    return np.concatenate([p.numpy().view(np.uint64) for p in parts])[:nl]


def _limb_worker(rank, world, name, port, q):
    """The RNS-limb partition (helrm_lookup_limbsplit's data flow) on the
    oracle: rank r owns rows [r rp, (r+1) rp) of the l+1+K limbs
    (rp = ceil((l+1+K) / world), as the library pads them); its inner sums and
    giant key switches are kept for those rows only; each giant pair's B rows
    and the final accumulators are exchanged with all_gather."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    core.set_threads(2)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.make_workload(name)
        cfg = w.config
        P = core.params_from_config(cfg)
        lay = lk.layout(w)
        plan = lk.make_plan(lay, P.n, cfg.level)
        sk = core.sk_gen(P, cfg.seed)
        pk = core.pk_gen(P, sk, cfg.seed)
        rk = core.rotkeys_gen(P, sk, plan.galois(P), cfg.seed)
        u = lk.encode_plan(P, plan)
        cts = lk.query_cts(P, pk, lay, plan, w.indices[0], w.dense[0], cfg.level, cfg.seed, 0)
        l = cfg.level
        qp = P.qp(l)
        nl = len(qp)
        rp = -(-nl // world)
        lo, hi = min(nl, rank * rp), min(nl, (rank + 1) * rp)
        # L1/L2 replicated digits, baby pairs (own rows used)
        D = [[core.modup(P, ct.c1, l, k) for k in range(P.dnum(l))] for ct in cts]
        ab = [{j: ((core.lift_P(P, ct.c0, l), core.lift_P(P, ct.c1, l)) if j == 0 else
                   core.rotate_lazy(P, ct, j, rk, D=D[c])) for j in plan.babies[c]} for c, ct in enumerate(cts)]
        col = np.array(qp, dtype=np.uint64).reshape(-1, 1)
        outs = []
        for o in range(plan.O):
            O0 = np.zeros((hi - lo, P.N), dtype=np.uint64)
            O1 = np.zeros_like(O0)
            for i, ent in enumerate(plan.entries[o]):
                if not ent:
                    continue
                A = np.zeros((hi - lo, P.N), dtype=np.uint64)   # own rows only
                B = np.zeros_like(A)
                for (c, j, uid) in ent:
                    a, b = ab[c][j]
                    A = (A + core.vmul(u[uid][lo:hi], a[lo:hi], qp[lo:hi])) % col[lo:hi]
                    B = (B + core.vmul(u[uid][lo:hi], b[lo:hi], qp[lo:hi])) % col[lo:hi]
                gi = plan.giants[o][i]
                if gi % P.n == 0:
                    O0, O1 = (O0 + A) % col[lo:hi], (O1 + B) % col[lo:hi]
                    continue
                Bf = _gather_rows(B, rp, nl, world)                    # all-gather of B's rows
                g = core.galois_elt(gi, P)
                G0, G1 = core.keyswitch(P, core.moddown(P, Bf, l), g, rk, l)   # replicated
                O0 = (O0 + core.automorph_ntt(A, g, P.N) + G0[lo:hi]) % col[lo:hi]
                O1 = (O1 + G1[lo:hi]) % col[lo:hi]
            outs.append((_gather_rows(O0, rp, nl, world), _gather_rows(O1, rp, nl, world)))
        out = lk.lookup_finish(P, plan, rk, outs, cts[0].scale)
        full = lk.lookup(P, plan, u, rk, cts)
        ok = all(np.array_equal(a.c0, b.c0) and np.array_equal(a.c1, b.c1) for a, b in zip(out, full))
        q.put((rank, lo, hi, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,port", [("uci", 29541), ("llm_small", 29543)])
def test_limb_partition_allgather_is_bit_exact(name, port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_limb_worker, args=(r, world, name, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[0][2] == res[1][1]   # rows tiled in rank order
    for rank, lo, hi, ok in res:
        assert ok, f"rank {rank}: limb-partitioned result differs from the single-process lookup"
