"""Full oracle lookups, timed (SURVEY.md 8(d) "Oracle timing": single thread and
all cores, core count stated).  Setup (keys, encoded diagonals, the encrypted
query) is not timed.  Usage: python tools/oracle_timing.py [config ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import core  # noqa: E402
from oracle import lookup as lk  # noqa: E402


def main(names):
    cores = len(os.sched_getaffinity(0))
    res = {"cores": cores, "lookups": {}}
    for name in names:
        w = synth.make_workload(name)
        core.set_threads(cores)
        run = lk.run_config(w, do_lookup=False)
        out = {}
        for threads in (cores, 1):
            core.set_threads(threads)
            t = time.perf_counter()
            lk.lookup(run.P, run.plan, run.u_ntt, run.rk, run.cts[0])
            out[f"{threads}_threads_s"] = round(time.perf_counter() - t, 2)
            print(name, threads, out, flush=True)
        res["lookups"][name] = out
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny_a", "uci", "criteo"])
