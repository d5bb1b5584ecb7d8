"""Compact plans (HELRM_PLAN_COMPACT): diagonals kept as int64 coefficients and
expanded (reduce, NTT, D-form) chunk by chunk during the lookup, input cts in
groups.  This is what makes the layouts whose QP-NTT diagonals exceed HBM
runnable:

- the paper-exact LLM layout L1 ("contiguous slot ordering
  (row-major)": 2 input / 3 output cts, 36,348 diagonals = 426 GiB stored);
- the paper's least compressed Criteo model (85 input cts;
  our seeded vocabularies give 100).

Parity: a compact plan gives the same bits as the stored-diagonal plan (only
exact modular sums are regrouped), checked on small and full-size configs, and
the L1 layout on the Tiny ring against the oracle."""
import hashlib
import json
import os

import numpy as np
import pytest

import synth
from oracle import core
from oracle import lookup as lk
from test_gpu_parity import env, torch_mod  # noqa: F401  (fixture)

gpu = pytest.mark.gpu
COMPACT = 2   # HELRM_PLAN_COMPACT


def _setup(E, w, compact, plan_only=False):
    h, cfg = E.h, w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan = h.plan_create(E.ctx, T, cfg.level, 0, COMPACT if compact else 0)
    if plan_only:
        return T, plan
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan.galois(), cfg.seed)
    info = plan.info()
    x = h.encode_query(T, w.indices[0], w.dense[0], info.n_in_cts * cfg.n_slots)
    cts = [h.encrypt(E.ctx, pk, x[c * cfg.n_slots:(c + 1) * cfg.n_slots], cfg.level, (cfg.seed << 20) | c)
           for c in range(info.n_in_cts)]
    return T, plan, sk, rk, cts


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


@gpu
@pytest.mark.parametrize("name", ["uci", "llm_small", "criteo_c2_small", "criteo_c9_small", "llm_gen_small"])
def test_compact_plan_equals_stored_plan(name, torch_mod):
    E = env(name, torch_mod)
    h, w = E.h, synth.make_workload(name)
    _, plan_s, sk, rk, cts = _setup(E, w, False)
    _, plan_c = _setup(E, w, True, plan_only=True)
    ic, is_ = plan_c.info(), plan_s.info()
    assert ic.mode == COMPACT and (ic.n_diag, ic.n_unique, ic.n1) == (is_.n_diag, is_.n_unique, is_.n1)
    assert ic.diag_bytes * (E.cfg.level + 1 + E.PO.K) == is_.diag_bytes
    want = h.lookup(E.ctx, plan_s, rk, cts)
    got = h.lookup(E.ctx, plan_c, rk, cts)
    for a, b in zip(got, want):
        assert np.array_equal(h.ct_export(E.ctx, a), h.ct_export(E.ctx, b))
    # the giant-range split runs on compact plans too
    for a, b in zip(h.lookup_dist_virtual(E.ctx, plan_c, rk, cts, 3), want):
        assert np.array_equal(h.ct_export(E.ctx, a), h.ct_export(E.ctx, b))


@gpu
def test_llm_l1_small_compact_matches_oracle(torch_mod):
    """The paper-exact L1 layout (contiguous token strides 64 in / 48 out) on
    the Tiny ring: 2 input / 2 output cts, bit-exact with the oracle."""
    E = env("llm_l1_small", torch_mod)
    h, w = E.h, synth.make_workload("llm_l1_small")
    ref = lk.run_config(w)
    assert (ref.plan.C, ref.plan.O, ref.plan.n_diag) == (2, 2, 1325)
    _, plan, sk, rk, cts = _setup(E, w, True)
    info = plan.info()
    assert (info.n_in_cts, info.n_out_cts, info.n_diag, info.n_unique) == (2, 2, 1325, len(ref.plan.u_slots))
    outs = h.lookup(E.ctx, plan, rk, cts)
    for got, want in zip(outs, ref.outs[0]):
        assert np.array_equal(h.ct_export(E.ctx, got), core.ct_to_coeff(ref.P, want))
    z = np.concatenate([h.decrypt_decode(E.ctx, sk, o) for o in outs])
    assert np.abs(z[: ref.lay.M] - lk.gather(ref.lay, w.indices[0])).max() < 1e-3


@gpu
def test_criteo_compact_full_size_golden(torch_mod):
    """Criteo at full size through a compact plan: the oracle's digest."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "criteo.json")))
    E = env("criteo", torch_mod)
    h, w = E.h, synth.make_workload("criteo")
    _, plan, sk, rk, cts = _setup(E, w, True)
    out = h.lookup(E.ctx, plan, rk, cts)
    assert _sha(h.ct_export(E.ctx, out[0])) == gold["queries"][0]["out_sha"][0]


@gpu
def test_llm_l1_full_size(torch_mod):
    """LLM layout L1 at full size (36,348
    non-zero diagonals over the four non-empty (out, in) ct blocks, 2 input /
    3 output cts): plan counts and every decrypted output ct against the
    float64 gather of the 128 tokens."""
    E = env("llm", torch_mod)
    h, w = E.h, synth.make_workload("llm_l1")
    T, plan, sk, rk, cts = _setup(E, w, True)
    info = plan.info()
    assert (info.n_in_cts, info.n_out_cts, info.n_diag) == (2, 3, 36348)
    outs = h.lookup(E.ctx, plan, rk, cts)
    lay = lk.layout(w)
    z = np.concatenate([h.decrypt_decode(E.ctx, sk, o) for o in outs])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3


@gpu
def test_criteo_100_ct_full_size(torch_mod):
    """The least compressed Criteo model (100 input cts
    with our vocabularies): 3,272,921 one-hot slots, every input ct's 512
    diagonals sharing the 15 giant rotations; decrypted output vs gather."""
    E = env("criteo", torch_mod)
    h, w = E.h, synth.make_workload("criteo_c100")
    T, plan, sk, rk, cts = _setup(E, w, True)
    info = plan.info()
    assert info.n_in_cts == 100 and info.K == 3272921 and info.n1 == 32
    out = h.lookup(E.ctx, plan, rk, cts)
    lay = lk.layout(w)
    z = h.decrypt_decode(E.ctx, sk, out[0])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3
    for c in cts:
        c.close()


@gpu
def test_criteo_17_ct_full_size(torch_mod):
    """The 10^2x Criteo model analog (569,545 slots, 18
    input cts; ours 535,963 slots = 17 cts, 8704 diagonals = 119 GiB in
    QP-NTT form) on a compact plan: plan counts and the decrypted output
    against the gather.  (The stored-plan form, 166 GiB of HBM in use, runs
    alone: tests/manual/c17_check.py, profiles/r01_c17.txt.)"""
    E = env("criteo", torch_mod)
    h, w = E.h, synth.make_workload("criteo_c17")
    T, plan, sk, rk, cts = _setup(E, w, True)
    info = plan.info()
    assert (info.n_in_cts, info.n_diag, info.n1) == (17, 8704, 32)
    out = h.lookup(E.ctx, plan, rk, cts)
    lay = lk.layout(w)
    z = h.decrypt_decode(E.ctx, sk, out[0])
    assert np.abs(z[: lay.M] - lk.gather(lay, w.indices[0])).max() < 1e-3
    for c in cts:
        c.close()


@gpu
@pytest.mark.parametrize("knobs", [{"HELRM_COMPACT_GROUP_GIB": "0.001", "HELRM_COMPACT_EXP_GIB": "0.001"},
                                   {"HELRM_COMPACT_GROUP_GIB": "0.02", "HELRM_COMPACT_EXP_GIB": "0.01"}])
def test_compact_chunking_knobs(knobs):
    """Tiny budgets force one input ct per group and a handful of diagonals
    per expansion chunk: still the stored plan's bits (fresh process, the
    knobs are read once)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_compact.py") + "::test_compact_plan_equals_stored_plan",
                        os.path.join(here, "test_gpu_compact.py") + "::test_llm_l1_small_compact_matches_oracle"],
                       env=dict(os.environ, **knobs), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@gpu
def test_compact_plan_batch_and_errors(torch_mod):
    """A batch on a compact plan runs query by query and equals the stored
    plan's batched lookup; the serving path and the limb partition reject
    compact plans (ARG), and a compact single-hoisted plan is refused."""
    E = env("uci", torch_mod)
    h, w = E.h, synth.make_workload("uci", batch=3)
    cfg = w.config
    T = h.tables_create(E.P, w.tables, w.n_dense)
    plan_s = h.plan_create(E.ctx, T, cfg.level)
    plan_c = h.plan_create(E.ctx, T, cfg.level, 0, COMPACT)
    sk = h.sk_gen(E.ctx, cfg.seed)
    pk = h.pk_gen(E.ctx, sk, cfg.seed)
    rk = h.rotkeys_gen(E.ctx, sk, plan_s.galois(), cfg.seed)
    cts = []
    for q in range(3):
        x = h.encode_query(T, w.indices[q], w.dense[q], cfg.n_slots)
        cts.append(h.encrypt(E.ctx, pk, x, cfg.level, (cfg.seed << 20) | q))
    for a, b in zip(h.lookup(E.ctx, plan_c, rk, cts, 3), h.lookup(E.ctx, plan_s, rk, cts, 3)):
        assert np.array_equal(h.ct_export(E.ctx, a), h.ct_export(E.ctx, b))
    coeff = np.ascontiguousarray(h.ct_export(E.ctx, cts[0]).reshape(-1))
    out = np.zeros(2 * cfg.level * cfg.N, dtype=np.uint64)
    with pytest.raises(h.HelrmError) as e:
        h.lookup_host(E.ctx, plan_c, rk, [coeff], 1.0, 1, [out])
    assert e.value.code == 10
    with pytest.raises(h.HelrmError) as e:
        h.lookup_limbsplit_virtual(E.ctx, plan_c, rk, cts[:1], 2)
    assert e.value.code == 10
    with pytest.raises(h.HelrmError) as e:
        h.plan_create(E.ctx, T, cfg.level, 0, COMPACT | 1)
    assert e.value.code == 10
