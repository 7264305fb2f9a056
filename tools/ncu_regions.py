"""Stall reasons + instruction-count regions of one ncu --set full capture."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
print("stalls:", {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): d[k]
                  for k in sorted(keys, key=lambda k: -float(d[k].replace(",", "") or 0))[:8]})
for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "launch__grid_size", "launch__registers_per_thread"]:
    print(k, d.get(k))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
b = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
for x in data:
    n = int(x["Instructions Executed"] or 0)
    s = int(x["Warp Stall Sampling (All Samples)"] or 0)
    if n == 0:
        continue
    b[n][0] += 1
    b[n][1] += n
    b[n][2] += s
    op = x["Source"].split()[0]
    if op.startswith("@"):
        op = x["Source"].split()[1]
    b[n][3][op.split(".")[0]] += 1
tot = sum(v[1] for v in b.values())
ts = sum(v[2] for v in b.values()) or 1
print("total inst", tot, "samples", ts)
for k, (cnt, t, samp, ops) in sorted(b.items(), key=lambda x: -x[1][2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"exec/inst={k:9d} ninst={cnt:5d} inst={t / tot:.3f} samples={samp / ts:.3f} {dict(ops.most_common(5))}")
