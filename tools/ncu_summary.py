#!/usr/bin/env python3
"""Summarise an ncu --set full report (per kernel: duration, DRAM bytes,
throughputs, occupancy, stall mix) into markdown, and merge the per-launch
DRAM bytes of each kernel class into profiles/ncu_traffic.json under the
bench config the report was captured on (bench.py's roofline.traffic reads
[config][kernel class]).
    python tools/ncu_summary.py report.ncu-rep out.md traffic.json CONFIG"""
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, page):
    if not rep.endswith(".ncu-rep"):  # CSV pages exported on the GPU box: PREFIX.raw.csv, PREFIX.details.csv
        return list(csv.reader(open(f"{rep}.{page}.csv")))
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, md, tj, config):
    det = ncu_csv(rep, "details")
    h = det[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit", "ID"))
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "Compute (SM) Throughput", "Registers Per Thread",
            "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy"]
    per = {}
    for r in det[1:]:
        if len(r) <= vi or r[mi] not in want:
            continue
        per.setdefault(r[ii], {"kernel": r[ki]})[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = ncu_csv(rep, "raw")
    rh = raw[0]
    col = {n: i for i, n in enumerate(rh)}
    traffic = {}
    for r in raw[2:]:
        rid = r[col["ID"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def nbytes(metric):  # each metric carries its own unit
            v = float(r[col[metric]].replace(",", ""))
            return v * scale.get(raw[1][col[metric]], 1)
        per.setdefault(rid, {})["dram_bytes"] = (nbytes("dram__bytes_read.sum") +
                                                 nbytes("dram__bytes_write.sum"))
        stalls = {}
        for n, i in col.items():
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(
                        r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        per[rid]["stalls"] = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
    lines = ["| kernel | " + " | ".join(want) + " | DRAM bytes/launch | top stalls |",
             "|" + "---|" * (len(want) + 3)]
    for rid in sorted(per, key=int):
        p = per[rid]
        name = p.get("kernel", "?").split("(")[0][:40]
        lines.append(f"| {name} | " + " | ".join(p.get(w, "") for w in want) +
                     f" | {p.get('dram_bytes', 0) / 1e6:.1f} MB | {p.get('stalls', '')} |")
        key = ("K1_spmm_gram" if "k1" in name else "K2_update_gram" if "k2" in name
               else "K3_update_p" if "k3" in name else name)
        traffic.setdefault(key, []).append(p.get("dram_bytes"))
    # per launch; K3 alternates skip / flush launches (deferred X): the mean
    traffic = {k: {"dram_bytes": sum(v) / len(v), "launches": len(v), "source": md}
               for k, v in traffic.items() if all(x is not None for x in v)}
    open(md, "w").write("\n".join(lines) + "\n")
    try:
        allt = json.load(open(tj))
    except (OSError, ValueError):
        allt = {}
    allt[config] = traffic
    json.dump(allt, open(tj, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:5])
