"""Stall-reason totals of an ncu report (source page, SASS view), whole kernel and for a
SASS index range.  usage: python tools/stall_summary.py report.ncu-rep [lo hi]"""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr, data = rows[0], rows[1:]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(data))
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: 0 for i in cols}
ninst = 0
for r in data[lo:hi]:
    for i in cols:
        tot[hdr[i]] += int(r[i] or 0)
    ninst += int(r[hdr.index("Instructions Executed")] or 0)
s = sum(tot.values())
print(f"samples {s}, warp-instructions executed {ninst}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {100.0 * v / max(s, 1):5.1f}%")
