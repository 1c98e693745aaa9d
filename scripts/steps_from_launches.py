"""Per-step kernel-time split from an ncu launch list (scripts/prof_steps.sh): steps are
delimited by commit_kv_kernel launches.  python scripts/steps_from_launches.py FILE.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
ks = [(r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '').split('::')[-1],
       float(r[vi].replace(',', ''))) for r in rows]
idx = [i for i, (k, _) in enumerate(ks) if 'commit_kv' in k]
for j, (a, b) in enumerate(zip(idx, idx[1:])):
    seg = ks[a + 1:b + 1]
    cls = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in seg:
        cls[k] += v / 1e6
        cnt[k] += 1
    top = sorted(cls.items(), key=lambda x: -x[1])[:10]
    print(f"step {j + 1}: {len(seg)} launches, {sum(v for _, v in seg) / 1e6:.3f} ms",
          {k: (cnt[k], round(v, 3)) for k, v in top})
