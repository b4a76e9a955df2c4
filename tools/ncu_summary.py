#!/usr/bin/env python
"""Summarise an ncu --set full report: key throughput / stall / instruction metrics."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions", "Block Size",
        "Grid Size", "Dynamic Shared Memory Per Block", "SM Frequency", "Mem Pipes Busy"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[1:]]


def raw(rep, pats):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if any(p in h for p in pats)}


if __name__ == "__main__":
    rep = sys.argv[1]
    for d in details(rep):
        if d.get("Metric Name") in KEYS:
            print(f"{d['Section Name'][:30]:30s} {d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
    pats = sys.argv[2].split(",") if len(sys.argv) > 2 else [
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__average_warp_latency_issue_stalled",
        "smsp__pcsamp_warps_issue_stalled", "sm__inst_executed_pipe", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared",
        "smsp__inst_executed_op_shared_atom", "sm__pipe_tensor", "pipe_alu", "pipe_fma", "sm__pipe_shared"]
    for k, (v, u) in sorted(raw(rep, pats).items()):
        if v not in ("", "0", "n/a"):
            print(f"  {k:80s} {v:>16s} {u}")
