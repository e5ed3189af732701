#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  launches: python scripts/ncu_summary.py launches <launches.csv> <out.md>
  full:     python scripts/ncu_summary.py full <prof.ncu-rep> <out.md> <out_traffic.json> <config-tag>
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    data = rows[hi + 1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    tot = sum(v for _, v in agg.values())
    init_only = ("km::k_assign_full", "km::k_td_from_dn", "km::k_chunk_scan", "km::k_gather_medoid_cols",
                 "km::k_check_symmetric", "km::k_validate_diag", "km::k_validate_cols")
    swap = [k for k in agg if k.startswith("km::") and "build" not in k and "changed_scatter" not in k
            and not k.startswith(init_only)]
    swap_tot = sum(agg[k][1] for k in swap)
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary: `{path}`\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the default `python bench.py` "
                "(cold-cache, serialised launches: compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | total us | share of all | share of SWAP step kernels |\n|---|---:|---:|---:|---:|\n")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            ss = f"{100 * v / swap_tot:.2f}%" if k in swap else ""
            f.write(f"| `{k}` | {c} | {v:.1f} | {100 * v / tot:.2f}% | {ss} |\n")
    print(open(out).read())


def full(rep, out, tjson, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_dynamic",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: `{rep}`\n\n")
        res = {}
        for r in rows[2:]:
            f.write("| metric | unit | value |\n|---|---|---|\n")
            cur = {}
            for w in want:
                if w in h:
                    i = h.index(w)
                    f.write(f"| {w} | {u[i]} | {r[i]} |\n")
                    cur[w] = (u[i], r[i])
            f.write("\n")
            # the traffic record is the SWAP stream's (the dominant kernel), else the last kernel's
            if not res or "stream" in cur.get("Kernel Name", ("", ""))[1] or "stream" not in res["Kernel Name"][1]:
                res = cur
        def val(k, to):
            unit, v = res[k]
            v = float(v.replace(",", ""))
            m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
            return v * m.get(unit, 1.0) / to
        traffic = val("dram__bytes_read.sum", 1) + val("dram__bytes_write.sum", 1)
        dur = val("gpu__time_duration.sum", 1)
        f.write(f"DRAM traffic per launch: {traffic / 1e9:.3f} GB; duration {dur * 1e3:.3f} ms; "
                f"{traffic / dur / 1e9:.0f} GB/s under ncu.\n")
    import os
    d = json.load(open(tjson)) if os.path.exists(tjson) else {}
    d[tag] = {"traffic_bytes": traffic, "ncu_duration_s": dur, "source": "profiles/" + os.path.basename(rep)}
    json.dump(d, open(tjson, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5])
