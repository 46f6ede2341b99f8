"""Per-launch summary of an ncu --set full report: duration, DRAM bytes, FP64 pipe, occupancy.
usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv, json, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = {"Kernel Name": "kernel", "gpu__time_duration.sum": "duration",
        "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "launch__grid_size": "grid", "launch__cluster_dim_x": "cluster_x"}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
res = []
for r in data:
    d = {}
    for k, nm in want.items():
        if k not in hdr:
            continue
        i = hdr.index(k)
        v = r[i]
        if nm in ("kernel",):
            d[nm] = v.split("(")[0].split("::")[-1]
            continue
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            d[nm] = v
            continue
        d[nm] = x * scale.get(units[i], 1.0)
    res.append(d)
for d in res:
    print(json.dumps(d))
if "--json" in sys.argv:
    json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
