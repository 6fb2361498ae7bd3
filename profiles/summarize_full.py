"""Summarise ncu --set full captures (one kernel each) into a table of the
numbers DESIGN.md cites. Usage: python summarize_full.py a.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time ms", "gpu__time_duration.sum", 1e3),
    ("dram rd GB", "dram__bytes_read.sum", 1e-9),
    ("dram wr GB", "dram__bytes_write.sum", 1e-9),
    ("dram %pk", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm %pk", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("occ %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("fp64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("dmma inst %", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("fp64 tensor ops %", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", 1),
]
# to bytes and seconds
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(paths):
    print("kernel | " + " | ".join(m[0] for m in METRICS))
    for p in paths:
        h, units, data = raw(p)
        for r in data:
            name = r[h.index("Kernel Name")][:40]
            vals = []
            for _, key, scale in METRICS:
                if key not in h:
                    vals.append("n/a")
                    continue
                i = h.index(key)
                try:
                    v = float(r[i].replace(",", "")) * UNITS.get(units[i], 1) * scale
                    vals.append(f"{v:.4g}")
                except ValueError:
                    vals.append(r[i])
            print(name + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1:])
