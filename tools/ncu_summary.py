"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: count, total/avg device time and share (cold-cache, serialised
launches: compare SHARES, not absolutes)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:48s} {c:8d} {t / 1e3:12.1f} {t / c / 1e3:10.2f} {t / tot:7.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
