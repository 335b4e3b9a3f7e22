"""Summarize an ncu report (run here, no GPU): SOL, occupancy, stall reasons, dram bytes."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
        "Occupancy", "Launch Statistics", "Scheduler Statistics", "Warp State Statistics")
names = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
         "Elapsed Cycles", "SM Active Cycles", "Issue Slots Busy", "Executed Ipc Active",
         "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Grid Size",
         "Block Size", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler",
         "Active Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
         "L1/TEX Cache Throughput", "L2 Cache Throughput", "SM Frequency")
r = csv.reader(out.splitlines())
hdr = next(r)
kname = None
for row in r:
    d = dict(zip(hdr, row))
    if kname is None:
        kname = d.get("Kernel Name", "")
        print("kernel:", kname[:100])
    if d.get("Section Name") in keep and d.get("Metric Name") in names:
        print(f"  {d['Metric Name'][:40]:40} {d['Metric Value']:>14} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__inst_executed.sum", "smsp__inst_executed.sum"]
for k, x, u in zip(h, v, rows[1]):
    if k in want:
        print(f"  {k:40} {x:>14} {u}")
st = [(k, x) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
      and not k.endswith("not_issued")]
tot = sum(float(x) for _, x in st if x.replace('.', '').isdigit()) or 1
print("  stall samples:")
for k, x in sorted(st, key=lambda t: -float(t[1]) if t[1].replace('.', '').isdigit() else 0)[:8]:
    print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28} {100*float(x)/tot:5.1f}%")
