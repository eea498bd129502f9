#!/usr/bin/env python3
"""Summarize an `ncu --set full` capture of the hot kernels into profiles/.

    python tools/summarize_profile.py gpurun_out/prof.ncu-rep profiles/r01_ncu_summary.json \
        [--launches gpurun_out/launches.csv] [--traffic profiles/ncu_traffic.json --dtype f32]

Writes per kernel: duration, DRAM bytes read/written (the roofline
`traffic`), DRAM/SM throughput, issue activity, occupancy, registers, top
stall reasons; optionally the launch-list shares (cold, serialised timings:
compare SHARES, not absolutes) and the per-launch DRAM traffic file that
bench.py reports as `roofline.traffic`.
"""
import argparse
import csv
import json
import subprocess


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(out.splitlines()))


def kernel_key(name):
    if "bwd_finish" in name:
        return "bwd_finish"
    if "bwd_kernel" in name:
        return "bwd"
    if "ew_tma" in name or "ew_kernel" in name:
        return "fwd"
    return name.split("(")[0][-40:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--traffic")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "raw")
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    res = {"note": a.note, "source": a.rep, "kernels": {}}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        k = kernel_key(name)

        def f(m):
            try:
                v = float(r[col[m]])
            except (KeyError, ValueError):
                return None
            u = units[col[m]]
            if u == "Mbyte":
                v *= 1e6
            elif u == "Kbyte":
                v *= 1e3
            elif u == "Gbyte":
                v *= 1e9
            elif u == "us":
                v *= 1e3  # -> ns
            elif u == "ms":
                v *= 1e6
            return v
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[col[h]]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d = {
            "kernel": name,
            "duration_ns": f("gpu__time_duration.sum"),
            "dram_read_bytes": f("dram__bytes_read.sum"),
            "dram_write_bytes": f("dram__bytes_write.sum"),
            "dram_pct_of_peak": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "sm_pct_of_peak": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "grid": f("launch__grid_size"),
            "instructions": f("smsp__inst_executed.sum"),
            "top_stalls": [[n, round(v, 2)] for v, n in stalls[:6]],
        }
        if d["dram_read_bytes"] is not None and d["dram_write_bytes"] is not None:
            d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        res["kernels"].setdefault(k, []).append(d)
    if a.launches:
        lr = list(csv.reader(open(a.launches)))
        start = next(i for i, r in enumerate(lr) if r and r[0] == "ID")
        h = lr[start]
        ni, vi = h.index("Kernel Name"), h.index("Metric Value")
        mi = h.index("Metric Name") if "Metric Name" in h else None
        tot, per = 0.0, {}
        for r in lr[start + 1:]:
            if mi is not None and r[mi] != "gpu__time_duration.sum":
                continue  # the launch list may carry DRAM byte counters too
            v = float(r[vi].replace(",", ""))
            k = kernel_key(r[ni])
            per[k] = per.get(k, 0.0) + v
            tot += v
        res["launch_list_share"] = {k: v / tot for k, v in per.items()}
        res["launch_list_total_ns"] = tot
    json.dump(res, open(a.out, "w"), indent=1)
    if a.traffic:
        try:
            tr = json.load(open(a.traffic))
        except Exception:
            tr = {}
        ent = tr.setdefault(a.dtype, {})
        for k, key in (("bwd", "bwd_bytes_per_launch"), ("fwd", "fwd_bytes_per_launch")):
            if k in res["kernels"] and res["kernels"][k][0].get("dram_bytes"):
                ent[key] = res["kernels"][k][0]["dram_bytes"]
        ent["source"] = a.rep
        json.dump(tr, open(a.traffic, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
