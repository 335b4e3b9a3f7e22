"""Text summary of one kernel in an ncu report (for profiles/): the headline metrics of the
details page, DRAM bytes, the warp-stall mix and the source lines with the most stall samples.

  python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX [--top 15] [--title "..."]
"""
import argparse
import collections
import csv
import subprocess


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=15)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    if a.title:
        print("#", a.title)
    det = list(csv.reader(ncu("-i", a.report, "-k", "regex:" + a.kernel, "--page", "details",
                              "--csv").splitlines()))
    want = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Block Size",
            "Grid Size", "L2 Hit Rate", "No Eligible", "Eligible Warps Per Scheduler"]
    if det:
        h = det[0]
        seen = set()
        for r in det[1:]:
            d = dict(zip(h, r))
            name = d.get("Metric Name")
            if name in want and name not in seen:
                seen.add(name)
                if len(seen) == 1:
                    print("kernel:", d.get("Kernel Name", "")[:110])
                print(f"  {name:<34} {d.get('Metric Value', '')} {d.get('Metric Unit', '')}")
    raw = list(csv.reader(ncu("-i", a.report, "-k", "regex:" + a.kernel, "--page", "raw",
                              "--csv").splitlines()))
    if len(raw) >= 3:
        d = dict(zip(raw[0], raw[2]))
        for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]:
            if k in d:
                print(f"  {k:<62} {d[k]} {raw[1][raw[0].index(k)]}")
        st = {}
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        print("  stall samples:")
        for k, v in sorted(st.items(), key=lambda t: -t[1])[:8]:
            print(f"    {k:<28} {100 * v / tot:5.1f}%")
    src = list(csv.reader(ncu("-i", a.report, "-k", "regex:" + a.kernel, "--page", "source",
                              "--csv", "--print-source", "cuda,sass").splitlines()))
    cur, hdr, out = None, None, []
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] != "":
            try:
                out.append((int(r[4] or 0), int(r[7] or 0), cur, r[0], r[1].strip()[:78]))
            except ValueError:
                pass
    if out:
        ts = sum(o[0] for o in out) or 1
        te = sum(o[1] for o in out) or 1
        print(f"  top source lines (stall samples %, instructions %):")
        for s_, e_, f, ln, txt in sorted(out, reverse=True)[:a.top]:
            print(f"    {100 * s_ / ts:5.1f}% {100 * e_ / te:5.1f}%i  {f}:{ln}  {txt}")


if __name__ == "__main__":
    main()
