"""Committed summaries under profiles/ from the ncu CSVs in gpurun_out/.
usage: profile_tables.py launches <launches.csv> <title>   (ncu --metrics gpu__time_duration.sum --csv log)
       profile_tables.py raw <raw.csv> <title>             (ncu --set full, --page raw --csv)"""
import collections
import csv
import sys


def launches(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:56]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    print(f"# {title}")
    print("# cold-cache serialized per-launch times (unit: ns)")
    print("%-56s %3s %12s %12s" % ("kernel", "n", "mean", "total"))
    for k, v in agg.items():
        print("%-56s %3d %12.1f %12.1f" % (k, len(v), sum(v) / len(v), sum(v)))


def raw(path, title):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    cols = [("dram_read_GB", "dram__bytes_read.sum", 1e-9), ("dram_write_GB", "dram__bytes_write.sum", 1e-9),
            ("ms", "gpu__time_duration.sum", 1e-6), ("issue%", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
            ("occ%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
            ("fp64pipe%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
            ("dmma%", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", 1),
            ("smem_wf%", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1)]
    units = rows[1]
    print(f"# {title}")
    print("%-42s" % "kernel" + "".join("%14s" % c[0] for c in cols))
    for r in rows[2:]:
        out = []
        for _, m, s in cols:
            i = hdr.index(m)
            v = float(r[i].replace(",", ""))
            u = units[i]
            if m.startswith("dram__bytes"):  # normalise to bytes
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            if m == "gpu__time_duration.sum":
                v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}.get(u, 1)
            out.append(v * s)
        print("%-42s" % r[hdr.index("Kernel Name")][:40] + "".join("%14.3f" % x for x in out))


if __name__ == "__main__":
    {"launches": launches, "raw": raw}[sys.argv[1]](sys.argv[2], sys.argv[3])
