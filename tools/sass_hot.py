"""Top stall-sampled SASS instructions of an ncu report (source page, SASS view).
usage: python tools/sass_hot.py report.ncu-rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = rows[1:]
tot = sum(int(r[isamp] or 0) for r in data)
print(f"total samples {tot}")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][isamp] or 0))[:n]
for i in sorted(idx):
    r = data[i]
    print(f"{100.0*int(r[isamp])/max(tot,1):5.1f}%  [{i:5d}] {r[isrc].strip()}")
