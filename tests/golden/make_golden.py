"""Writes tests/golden/<config>.json from the CPU oracle ONLY (oracle/ + synth/).

For configs too large to re-run the oracle inside the GPU test budget
(Criteo: ~10 min of CPU), the parity test compares the SHA-256 of the
library's canonical exports (coefficient form, little-endian uint64) with the
digests recorded here, plus the decrypted-vs-gather error of the oracle's own
output.  Usage: python tests/golden/make_golden.py criteo [criteo_b64 ...]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import core  # noqa: E402
from oracle import lookup as lk  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def main(name: str, queries=None):
    w = synth.make_workload(name)
    cfg = w.config
    t = time.time()
    P = core.params_from_config(cfg)
    lay = lk.layout(w)
    plan = lk.make_plan(lay, P.n, cfg.level)
    sk = core.sk_gen(P, cfg.seed)
    pk = core.pk_gen(P, sk, cfg.seed)
    t_keys0 = time.time()
    rk = core.rotkeys_gen(P, sk, plan.galois(P), cfg.seed)
    t_keys = time.time() - t_keys0
    t_enc0 = time.time()
    u = lk.encode_plan(P, plan)
    t_enc = time.time() - t_enc0
    qs = list(range(w.indices.shape[0])) if queries is None else queries
    out = {"config": name, "threads": core.threads(), "queries": []}
    g0 = plan.galois(P)[0]
    out["rotkey_g0"] = g0
    out["rotkey_g0_sha"] = [sha(np.stack([core.intt(b, P.q + P.p, P), core.intt(a, P.q + P.p, P)])) for b, a in rk.keys[g0]]
    out["diag0_sha"] = sha(core.intt(u[0], P.qp(cfg.level), P))
    t_look = 0.0
    for q in qs:
        if name.startswith("mlp"):
            # dense linear layer: the encrypted input is synth.dense_inputs' row q at seed << 20 | q
            z = np.zeros(P.n)
            x = synth.dense_inputs(name, q + 1)[q]
            z[: len(x)] = x
            cts = [core.encrypt(P, pk, z, cfg.level, (cfg.seed << 20) | q)]
        else:
            cts = lk.query_cts(P, pk, lay, plan, w.indices[q], w.dense[q], cfg.level, cfg.seed, q)
        t0 = time.time()
        res = lk.lookup(P, plan, u, rk, cts)
        t_look += time.time() - t0
        z = np.concatenate([core.decrypt_decode(P, sk, r) for r in res])
        y = x @ w.tables[0].weights if name.startswith("mlp") else lk.gather(lay, w.indices[q])
        err = float(np.abs(z[: lay.M] - y).max())
        out["queries"].append({"q": q, "in_sha": [sha(core.ct_to_coeff(P, c)) for c in cts],
                               "out_sha": [sha(core.ct_to_coeff(P, r)) for r in res],
                               "dec_err": err})
        print(name, q, "err", err, flush=True)
    out["plan"] = {"n_diag": plan.n_diag, "n_unique": len(plan.u_slots), "n1": plan.n1, "C": plan.C, "O": plan.O,
                   "mbar": plan.mbar, "n_rotations": len(plan.rotation_amounts(P))}
    out["seconds"] = {"keys": t_keys, "encode_diagonals": t_enc, "lookup_per_query": t_look / len(qs),
                      "total": time.time() - t}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["seconds"]))


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["criteo"]:
        nm, _, qq = arg.partition(":")
        main(nm, [int(x) for x in qq.split(",")] if qq else None)
