"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def main(path, top=25):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        if "zgemm_kernel" in r["Kernel Name"]:
            name = r["Kernel Name"][:90]
        unit = r["Metric Unit"]
        if unit not in scale:
            raise ValueError(f"unknown duration unit {unit!r}")
        v = float(r["Metric Value"].replace(",", "")) * scale[unit]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, total {tot:.1f} us")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
