"""Summarise ncu artifacts into the text files kept under profiles/.

    python scripts/ncu_summary.py rep  <file.ncu-rep> [algorithmic_bytes_per_launch]
    python scripts/ncu_summary.py list <launches.csv>       (gpu__time_duration launch list)
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction", "SM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"]


def _ncu(args):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", *args], capture_output=True, text=True).stdout)))


def rep(path, alg=None):
    det = _ncu(["-i", path, "--page", "details", "--csv"])
    raw = _ncu(["-i", path, "--page", "raw", "--csv"])
    h = det[0]
    by_id = collections.OrderedDict()
    for r in det[1:]:
        d = dict(zip(h, r))
        e = by_id.setdefault(d["ID"], {"kernel": d["Kernel Name"]})
        if d["Metric Name"] in KEYS:
            e[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    rh, ru = raw[0], raw[1]
    for k, r in enumerate(raw[2:]):
        e = list(by_id.values())[k]
        for n in RAW:
            if n in rh:
                e[n] = f"{r[rh.index(n)]} {ru[rh.index(n)]}".strip()
    print(f"# ncu --set full summary of {path}")
    for i, e in by_id.items():
        print(f"\n## launch {i}: {e.pop('kernel')[:160]}")
        for k, v in e.items():
            print(f"  {k:60s} {v}")
        rb, wb = e.get("dram__bytes_read.sum"), e.get("dram__bytes_write.sum")
        if rb and wb:
            def b(x):
                v, u = x.split()
                return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            t = b(rb) + b(wb)
            print(f"  {'traffic (dram read+write, bytes)':60s} {t:.6g}")
            if alg:
                print(f"  {'algorithmic bytes':60s} {float(alg):.6g}")
                print(f"  {'traffic / algorithmic':60s} {t / float(alg):.4f}")


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        recs[d["ID"]] = (name, v)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v in recs.values():
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list {path}: {len(recs)} launches, {tot:.1f} us (serialised, cold-cache per launch)")
    print(f"{'kernel':60s} {'n':>6s} {'us':>12s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {n:6d} {us:12.1f} {us / tot:7.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        launch_list(sys.argv[2])
