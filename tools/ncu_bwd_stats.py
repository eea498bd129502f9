"""Summarise one kernel of an ncu report: duration, DRAM, issue, stalls, hot SASS blocks."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
for w in want:
    if w in h: print(w, v[h.index(w)])
st = [(n, v[i]) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
tot = sum(float(x or 0) for _, x in st)
for n, x in sorted(st, key=lambda t: -float(t[1] or 0))[:8]:
    print("  %-60s %5.1f%%" % (n.replace("smsp__pcsamp_warps_issue_stalled_", "stall_"), 100 * float(x) / tot))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]; rows = src[2:]
ie = hh.index("Instructions Executed"); sc = hh.index("Warp Stall Sampling (All Samples)")
blocks = []
for x in rows:
    n = int(x[ie] or 0); s = int(x[sc] or 0)
    if blocks and blocks[-1][1] == n: blocks[-1][2] += 1; blocks[-1][3] += s
    else: blocks.append([x[0][-5:], n, 1, s])
T = sum(b[1] * b[2] for b in blocks); S = sum(b[3] for b in blocks)
print("warp-instructions", T, "samples", S)
for b in blocks:
    if b[1] * b[2] > T * 0.01 or b[3] > S * 0.03:
        print("  %s exec %8d len %3d inst %5.1f%% stall %5.1f%%" % (b[0], b[1], b[2], 100 * b[1] * b[2] / T, 100 * b[3] / S))
