"""Summarise an ncu report (and optionally a launch-list CSV) into markdown for profiles/."""
import csv, subprocess, sys
from collections import Counter, defaultdict

def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))

def details(rep):
    r = page(rep, "details")
    h = r[0]
    rows = [dict(zip(h, x)) for x in r[1:] if len(x) >= 15]
    return rows

WANT = ["Duration", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "Compute (SM) Throughput",
        "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Size", "Grid Size", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Executed Instructions"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]

def main(rep, title, launches=None):
    print(f"# {title}\n\nreport: `{rep}` (ncu --set full --clock-control none)\n")
    kern = None
    print("| metric | value |\n|---|---|")
    for d in details(rep):
        if kern is None:
            kern = d.get("Kernel Name", "")
        if d["Metric Name"] in WANT:
            print(f"| {d['Metric Name']} | {d['Metric Value']} {d['Metric Unit']} |")
    r = page(rep, "raw")
    h, u, v = r[0], r[1], r[2]
    for name, unit, val in zip(h, u, v):
        if name in RAW:
            print(f"| {name} | {val} {unit} |")
    print(f"\nkernel: `{kern}`\n")
    s = page(rep, "source", ["--print-source", "sass"])
    hh = s[1]
    data = [dict(zip(hh, x)) for x in s[2:] if len(x) == len(hh) and x[0].startswith("0x")]
    f = lambda x: float(x.replace(",", "") or 0)
    tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
    stalls = defaultdict(float)
    for d in data:
        for c in hh:
            if c.startswith("stall_") and "Not Issued" not in c:
                stalls[c] += f(d[c])
    print("| stall reason | share of samples |\n|---|---|")
    for c, val in sorted(stalls.items(), key=lambda x: -x[1])[:8]:
        print(f"| {c} | {100*val/tot:.1f}% |")
    ops = Counter()
    for d in data:
        op = [o for o in d["Source"].split() if not o.startswith("@")]
        if op:
            ops[op[0].split(".")[0]] += f(d["Instructions Executed"])
    ti = sum(ops.values()) or 1
    print("\n| SASS opcode | share of executed warp-instructions |\n|---|---|")
    for k, val in ops.most_common(14):
        print(f"| {k} | {100*val/ti:.1f}% |")
    if launches:
        rows = list(csv.reader(open(launches)))
        hdr = None
        agg = defaultdict(lambda: [0, 0.0])
        for x in rows:
            if "Kernel Name" in x:
                hdr = x; continue
            if hdr and len(x) == len(hdr):
                dd = dict(zip(hdr, x))
                if dd.get("Metric Name") == "gpu__time_duration.sum":
                    agg[dd["Kernel Name"][:90]][0] += 1
                    agg[dd["Kernel Name"][:90]][1] += float(dd["Metric Value"].replace(",", ""))
        tt = sum(a[1] for a in agg.values()) or 1
        print(f"\n## launch list (`{launches}`, cold-cache serialised; compare shares)\n")
        print("| kernel | launches | total us | share |\n|---|---|---|---|")
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            print(f"| `{k}` | {c} | {t/1e3:.1f} | {100*t/tt:.1f}% |")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
