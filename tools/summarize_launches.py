"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, sys, collections, re
path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
uni = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).split("::")[-1].strip()
    v = float(r[vi].replace(",", ""))
    unit = r[uni] if uni is not None else "ns"
    scale = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(unit, 1e-9)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':32s} {'launches':>9s} {'total ms':>10s} {'share':>7s} {'mean us':>9s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:32s} {cnt[k]:9d} {1e3*v:10.2f} {100*v/T:6.1f}% {1e6*v/cnt[k]:9.1f}")
print(f"{'TOTAL':32s} {sum(cnt.values()):9d} {1e3*T:10.2f}")
