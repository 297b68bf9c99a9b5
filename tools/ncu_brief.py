"""Key metrics from an ncu --page details --csv export: python tools/ncu_brief.py CSV"""
import csv, sys
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Compute (SM) Throughput",
        "Executed Ipc Active", "L1/TEX Cache Throughput", "Block Limit Registers", "Block Limit Shared Mem"]
seen = {}
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[12] in keys:
        seen.setdefault(r[4][:60], []).append(f"{r[12]}={r[14]}{r[13]}")
for k, v in seen.items():
    print(k)
    print("   " + "  ".join(v))
