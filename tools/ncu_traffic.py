"""DRAM traffic per launch / per limb transform from an ncu --set full report
of `bench.py --ncu-step` (one Criteo lookup):

  python tools/ncu_traffic.py gpurun_out/<rep>.ncu-rep > profiles/ncu_traffic.json

NTT passes: grid = 16 CTAs x limbs (N = 2^16), so limbs = grid_size / 16."""
import csv
import json
import subprocess
import sys


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    col = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                      "launch__grid_size", "gpu__time_duration.sum")}
    fp64 = "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
    col_fp64 = hdr.index(fp64) if fp64 in hdr else None
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").strip()
        b = sum(float(r[col[k]].replace(",", "")) * scale[units[col[k]]]
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        g = int(float(r[col["launch__grid_size"]].replace(",", "")))
        a = agg.setdefault(name, {"launches": 0, "bytes": 0.0, "grid": 0, "time": 0.0, "fp64_x_time": 0.0})
        a["launches"] += 1
        a["bytes"] += b
        a["grid"] += g
        t = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
        a["time"] += t
        if col_fp64 is not None:
            a["fp64_x_time"] += t * float(r[col_fp64].replace(",", ""))
    import os
    commit = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True, text=True,
                            cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__)))).stdout.strip()
    res = {"source": path, "commit": commit, "kernels": agg}
    p1 = [v for k, v in agg.items() if k.startswith("k_ntt_fwd<8, 0") or k.startswith("k_ntt_fwd<8, 2")]
    p2 = [v for k, v in agg.items() if k.startswith("k_ntt_fwd<8, 1")]
    if p1 and p2:
        limbs = sum(v["grid"] for v in p1) / 16
        res["ntt_fwd_bytes_per_limb"] = round((sum(v["bytes"] for v in p1) + sum(v["bytes"] for v in p2)) / limbs)
        res["ntt_fwd_limbs"] = limbs
        # FP64 pipe busy fraction of the forward NTT, time-weighted over its launches
        t = sum(v["time"] for v in p1 + p2)
        if t > 0 and col_fp64 is not None:
            res["ntt_fwd_fp64_pipe_frac"] = round(sum(v["fp64_x_time"] for v in p1 + p2) / t / 100.0, 4)
            for nm, ks in (("p1", p1), ("p2", p2)):
                tt = sum(v["time"] for v in ks)
                res[f"ntt_fwd_{nm}_fp64_pipe_frac"] = round(sum(v["fp64_x_time"] for v in ks) / tt / 100.0, 4)
    for prefix, key in (("k_diag_mac", "diag_mac"), ("k_kip_multi", "kip_multi")):
        ks = [v for k, v in agg.items() if k.startswith(prefix)]
        if ks:
            res[key + "_bytes_per_launch"] = round(sum(v["bytes"] for v in ks) / sum(v["launches"] for v in ks))
    kips = [v for k, v in agg.items() if k.startswith("k_kip<") or k.startswith("k_kip_giants")]
    if kips:
        res["kip_bytes_per_launch"] = round(sum(v["bytes"] for v in kips) / sum(v["launches"] for v in kips))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
