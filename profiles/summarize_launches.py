"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel."""
import collections
import csv
import re
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        m = re.search(r"(k_\w+)(<[^>(]*>)?", r[ki])
        name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':44s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:44s} {n:8d} {t / 1e3:12.1f} {t / n / 1e3:10.2f} {t / tot:6.3f}")
    out.append(f"{'TOTAL':44s} {len(data):8d} {tot / 1e3:12.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
