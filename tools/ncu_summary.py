"""Summarise ncu CSV exports (details/raw/source pages) brought back from gpurun_out/."""
import csv
import sys


def details(path, want=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    want = want or ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
                    "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy",
                    "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block"]
    cur = None
    for r in rows[1:]:
        if r[mi] in want:
            if cur != r[idi]:
                cur = r[idi]
                print("==", r[idi], r[ki][:70])
            print("   %-40s %s %s" % (r[mi], r[vi], r[ui]))


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        st = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        print(r[hdr.index("Kernel Name")][:50], " ".join("%s=%.0f%%" % (k, 100 * v / tot)
                                                      for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]))
        for m in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum"]:
            if m in hdr:
                print("    %-60s %s %s" % (m, r[hdr.index(m)], units[hdr.index(m)]))


def source(path, top=30):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
            hdr, start = r, i
            break
    si, ws, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data, seen = [], set()
    for r in rows[start + 1:]:
        if len(r) <= ie or r[0] in seen:
            continue
        seen.add(r[0])
        try:
            data.append((float(r[ws] or 0), float(r[ie] or 0), r[0], r[si][:100]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    toti = sum(d[1] for d in data) or 1
    print("instructions executed:", toti)
    for d in sorted(data, key=lambda x: -x[0])[:top]:
        print("%5.1f%% stall %5.2f%% inst %s %s" % (100 * d[0] / tot, 100 * d[1] / toti, d[2][-5:], d[3]))


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    {"details": details, "raw": raw, "source": source}[kind](path)
