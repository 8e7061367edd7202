"""Summarise an ncu --set full report: per kernel, duration, DRAM traffic, throughput and
issue/tensor-pipe utilisation (the numbers DESIGN.md and bench.py's roofline cite).

    python tools/ncu_summary.py report.ncu-rep > profiles/rN/name.txt"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc-pipe inst %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# {path}")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        print(f"\n## {name[:150]}")
        for key, label in WANT:
            cols = [h for h in hdr if h == key or h.endswith("." + key) or h.endswith(key)]
            if cols:
                c = cols[0]
                print(f"  {label:28s} {r[idx[c]]} {units[idx[c]]}")


if __name__ == "__main__":
    main(sys.argv[1])
