"""Summarise ncu --set full captures (raw page) into one text table.

usage: python tools/ncu_summary.py report.ncu-rep [...] > profiles/rNN_ncu_summary.txt
"""
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("duration_us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("cluster", "launch__cluster_dim_x"),
    ("regs", "launch__registers_per_thread"),
    ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("dmma_pipe_active_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    ("fp64_tensor_ops_pct_elapsed", "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed"),
    ("fp64_pipe_inst_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_pct_peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("ipc_active", "sm__inst_executed.avg.per_cycle_active"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
]


def raw(path):
    """Every profiled kernel of a report: [{metric: (value, unit)}]."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, vals)} for vals in rows[2:] if vals]


def main():
    print(f"{'report':22s} {'kernel':44s} " + " ".join(f"{n:>12s}" for n, _ in METRICS))
    for path in sys.argv[1:]:
        for d in raw(path):
            name = d.get("Kernel Name", ("?", ""))[0]
            cells = []
            for _, key in METRICS:
                v, u = d.get(key, ("-", ""))
                try:
                    x = float(v.replace(",", ""))
                    if u == "Mbyte" or u == "Gbyte" or u == "Kbyte" or u == "byte":
                        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]
                        x *= scale
                    elif u == "ms":
                        x *= 1e3
                    elif u == "ns":
                        x *= 1e-3
                    cells.append(f"{x:12.4g}")
                except ValueError:
                    cells.append(f"{v:>12s}")
            print(f"{os.path.basename(path):22s} {name[:44]:44s} " + " ".join(cells))

if __name__ == "__main__":
    main()
