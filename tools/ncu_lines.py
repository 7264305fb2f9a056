"""Per-region instruction / stall-sample totals of one ncu capture of k_update_tc
(source page with -lineinfo).  usage: ncu_lines.py REPORT [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
out = []
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            out.append((int(r[7]), int(r[4]), fname, int(r[0]), r[1][:80]))
        except ValueError:
            pass
MARKERS = {"ds_tc.cu": [("tc helpers", None), ("tc setup", "k_update_tc(TcArgs"),
                         ("pipelines", "pipelines: banks + MMAs"), ("epi setup+prefetch", "epilogue\n"),
                         ("epi tiles", "for (int t = 0; t < ntiles; t++) {\n        const int gt"),
                         ("epi tail", "if (process && ok) {\n#if DS_VAR_MULSHIFT")],
           "ds_stream.cuh": [("stream helpers", None), ("swin access", "struct SWin {"),
                             ("swin init/push/finish", "void init("), ("swin fast_block", "void fast_block("),
                             ("emit", "struct Emit {"), ("round_out", "void round_out(")]}


def _regions():
    import os
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1308_1536_b200", "csrc")
    reg = {}
    for f, marks in MARKERS.items():
        src = open(os.path.join(root, f)).read()
        lst = []
        for name, m in marks:
            line = 0 if m is None else src[:src.index(m)].count("\n") + 1
            lst.append((line, name))
        reg[f] = sorted(lst)
    return reg


REG = _regions()


def region(f, line):
    name = f
    for start, nm in REG.get(f, []):
        if line >= start:
            name = nm
    return name


agg = collections.defaultdict(lambda: [0, 0])
for n, s, f, line, _ in out:
    k = region(f, line)
    agg[k][0] += n
    agg[k][1] += s
T = sum(v[0] for v in agg.values()) or 1
S = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:24s} inst {v[0] / 1e6:7.2f}M ({100 * v[0] / T:4.1f}%)  samples {v[1]:6d} ({100 * v[1] / S:4.1f}%)")
if top:
    for o in sorted(out, key=lambda o: -o[1])[:top]:
        print(o)
