"""Small end-to-end workload for compute-sanitizer: Tiny-B and
UCI lookups (double and single hoisted, batch 2), hoisted rotations, the
virtual-rank split and the serving path, each checked against the oracle.

  compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_case.py
  compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize_case.py tiny_b
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import core  # noqa: E402
from oracle import lookup as lk  # noqa: E402
from paper_2506_18150_b200 import helrm as h  # noqa: E402


def case(name):
    w = synth.make_workload(name, batch=2)
    cfg = w.config
    ref = lk.run_config(w)
    P = h.params_from_config(cfg)
    ctx = h.Context(P, 0, 0)
    T = h.tables_create(P, w.tables, w.n_dense)
    plan = h.plan_create(ctx, T, cfg.level)
    sk = h.sk_gen(ctx, cfg.seed)
    pk = h.pk_gen(ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(ctx, sk, plan.galois(), cfg.seed)
    info = plan.info()
    cts = []
    for q in range(2):
        x = h.encode_query(T, w.indices[q], w.dense[q], info.n_in_cts * cfg.n_slots)
        cts += [h.encrypt(ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level,
                          (cfg.seed << 20) | (q * info.n_in_cts + c)) for c in range(info.n_in_cts)]
    outs = h.lookup(ctx, plan, rk, cts, 2)
    for q in range(2):
        for o in range(info.n_out_cts):
            got = h.ct_export(ctx, outs[q * info.n_out_cts + o])
            assert np.array_equal(got, core.ct_to_coeff(ref.P, ref.outs[q][o])), (name, q, o)
    virt = h.lookup_dist_virtual(ctx, plan, rk, cts[: info.n_in_cts], 2)
    assert np.array_equal(h.ct_export(ctx, virt[0]), h.ct_export(ctx, outs[0]))
    single = h.plan_create(ctx, T, cfg.level, 0, h.MODE_SINGLE)
    s_out = h.lookup(ctx, single, rk, cts[: info.n_in_cts])
    z = h.decrypt_decode(ctx, sk, s_out[0])
    assert np.abs(z[: ref.lay.M] - lk.gather(ref.lay, w.indices[0])[: ref.lay.M]).max() < 1e-3
    ring = [h.ct_alloc(ctx, cfg.level) for _ in range(2)]
    h.rotate_hoisted(ctx, rk, cts[0], plan.rotations()[:2], ring)
    host_in = [np.ascontiguousarray(h.ct_export(ctx, c).ravel()) for c in cts]
    host_out = [np.zeros(2 * cfg.level * cfg.N, np.uint64) for _ in range(2 * info.n_out_cts)]
    if info.n_in_cts == 1:
        h.lookup_host(ctx, plan, rk, host_in, 2.0 ** cfg.log_scale, 2, host_out)
        assert np.array_equal(host_out[0], h.ct_export(ctx, outs[0]).ravel())
    ctx.close()
    print(name, "ok", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["tiny_b", "uci"]:
        case(name)
