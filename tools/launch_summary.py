"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel name."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append(d)
    return data


def summarize(path, top=25, last=0):
    data = load(path)
    if last:
        data = data[-last:]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    tot, cnt, grid = collections.defaultdict(float), collections.Counter(), {}
    for d in data:
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
        k = re.sub(r"rutv::|\(anonymous namespace\)::|unnamed>::", "", d["Kernel Name"])
        k = re.sub(r"\(long.*|\(int.*|\(rutv.*", "", k)[:48]
        tot[k] += v
        cnt[k] += 1
    T = sum(tot.values())
    lines = [f"launches={len(data)} total_device_time_ms={T / 1e3:.2f} (serialised, cold-cache ncu pass)",
             f"{'ms':>9} {'share':>6} {'n':>6} {'avg_us':>9}  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{v / 1e3:9.2f} {100 * v / T:5.1f}% {cnt[k]:6d} {v / cnt[k]:9.1f}  {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    print(summarize(sys.argv[1], last=last))
