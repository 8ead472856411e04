"""Summarise an ncu report: key SOL metrics + SASS opcode mix (for profiles/)."""
import collections, csv, io, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout

def details(rep):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = r[0]
    out = {}
    for x in r[1:]:
        d = dict(zip(h, x))
        out[(d["Section Name"], d["Metric Name"])] = (d["Metric Value"], d["Metric Unit"])
    return out

KEYS = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "No Eligible", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]

def main(rep):
    d = details(rep)
    for k in KEYS:
        for (sec, name), (v, u) in d.items():
            if name == k:
                print(f"{name:40s} {v} {u}")
                break
    r = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
    tot = sum(int(x["Instructions Executed"] or 0) for x in rows)
    op, samp = collections.Counter(), collections.Counter()
    stall_tot = 0
    for x in rows:
        src = x["Source"].split()
        if not src:
            continue
        m = src[1] if src[0].startswith("@") else src[0]
        m = m.split(".")[0]
        op[m] += int(x["Instructions Executed"] or 0)
        v = int(x["Warp Stall Sampling (All Samples)"] or 0)
        samp[m] += v
        stall_tot += v
    print(f"SASS instructions executed: {tot}")
    for k, v in op.most_common(22):
        print(f"  {k:10s} {v:14d} {100 * v / max(tot, 1):5.1f}%   stall-samples {100 * samp[k] / max(stall_tot, 1):5.1f}%")

if __name__ == "__main__":
    main(sys.argv[1])
