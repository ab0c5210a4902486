"""Compact summary of an .ncu-rep (details page + top stall reasons + source hot spots).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [--source N]
"""
import csv
import io
import subprocess
import sys


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    ik, isec, iname, iunit, ival = (h.index("Kernel Name"), h.index("Section Name"), h.index("Metric Name"),
                                    h.index("Metric Unit"), h.index("Metric Value"))
    keep = ("Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Block Limit Shared Mem",
            "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Active Warps Per Scheduler",
            "Eligible Warps Per Scheduler", "No Eligible", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions", "Grid Size", "Block Size")
    seen = set()
    for r in rows[1:]:
        if len(r) <= ival:
            continue
        name = r[iname]
        if name in keep and name not in seen:
            seen.add(name)
            print(f"  {name:40s} {r[ival]:>14s} {r[iunit]}")


def raw_metrics(rep, prefixes):
    rows = ncu_csv(rep, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    for i, name in enumerate(h):
        if any(name.startswith(p) for p in prefixes):
            print(f"  {name:75s} {v[i]:>14s} {u[i]}")


def stalls(rep):
    rows = ncu_csv(rep, "raw")
    h, v = rows[0], rows[2]
    items = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warp_latency_issue_stalled_") and name.endswith(".ratio"):
            try:
                items.append((float(v[i].replace(",", "")), name[len("smsp__average_warp_latency_issue_stalled_"):-6]))
            except ValueError:
                pass
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            pass
    items.sort(reverse=True)
    print("  stall reasons (avg cycles per issued instr):", ", ".join(f"{n}={x:.2f}" for x, n in items[:8]))


if __name__ == "__main__":
    rep = sys.argv[1]
    details(rep)
    stalls(rep)
    raw_metrics(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                      "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
                      "l1tex__data_bank_conflicts_pipe_lsu_mem_shared", "sm__pipe_fp64_cycles_active.avg.pct",
                      "sm__inst_executed_pipe_lsu.avg.pct", "smsp__inst_executed_op_ldgsts"])


def source_stalls(rep, kernel_regex=None):
    """Per-reason stall totals and per-opcode instruction mix from the SASS source page."""
    import collections
    rows = ncu_csv(rep, "source", ["--print-source", "sass"])
    hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    iS, iI = h.index("Source"), h.index("Instructions Executed")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    ops = collections.Counter()
    for r in data:
        if len(r) <= iI:
            continue
        for c in reasons:
            try:
                tot[c] += float(r[h.index(c)] or 0)
            except ValueError:
                pass
        t = r[iS].split()
        if t:
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[op] += float(r[iI] or 0)
    s = sum(tot.values()) or 1
    print("  stall samples:", ", ".join(f"{k[6:]}={100*v/s:.0f}%" for k, v in tot.most_common(8)))
    so = sum(ops.values()) or 1
    print(f"  warp instructions {so:.3g}:", ", ".join(f"{k}={100*v/so:.0f}%" for k, v in ops.most_common(10)))


if __name__ == "__main__" and "--source" in sys.argv:
    source_stalls(sys.argv[1])
