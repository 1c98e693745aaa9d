"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) of a short rollout:
one decode step = the last `per_step` launches before the final step. Prints per-kernel time,
DRAM bytes and achieved GB/s (cold-cache, serialised launches: shares, not absolutes).

    python scripts/tail_summary.py gpurun_out/tail_launches.csv [per_step]
"""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3}


def main():
    path = sys.argv[1]
    per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 207
    hdr, launches = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = launches.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
    ks = list(launches.values())
    step = ks[-2 * per_step:-per_step]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in step:
        n = e["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        a = agg[n]
        a[0] += 1
        a[1] += e["gpu__time_duration.sum"]
        a[2] += e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"]
    tot = sum(a[1] for a in agg.values())
    print(f"{len(ks)} launches captured; one decode step = {len(step)} launches, {tot:.1f} us serialised")
    print(f"{'kernel':44s} {'n':>4s} {'us':>9s} {'us/launch':>9s} {'share':>6s} {'MB':>8s} {'GB/s':>7s}")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:44]:44s} {a[0]:4d} {a[1]:9.1f} {a[1] / a[0]:9.2f} {a[1] / tot:6.1%} {a[2] / 1e6:8.1f} "
              f"{a[2] / a[1] / 1e3:7.0f}")


if __name__ == "__main__":
    main()
