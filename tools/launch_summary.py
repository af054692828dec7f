"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys

def summarize(path, header=""):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h, rows = rows[0], rows[1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows:
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(a[1] for a in agg.values())
    out = [header, "(cold-cache, serialised per-launch times: compare SHARES, not absolutes)", "",
           f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:60]:60s} {n:8d} {t:12.1f} {t / n:10.1f} {100 * t / tot:6.2f}%")
    return "\n".join(out) + "\n"

if __name__ == "__main__":
    print(summarize(sys.argv[1], " ".join(sys.argv[2:])), end="")
