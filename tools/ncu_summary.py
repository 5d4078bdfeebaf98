"""One-line-per-kernel summary of an ncu --set full report (the numbers the
roofline claims rest on): duration, DRAM bytes and throughput, tensor-pipe
activity, occupancy, L2 hit rate.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active": "tc_gmma_%",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_%",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": "tc_inst_%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_%",
    "lts__t_sector_hit_rate.pct": "l2_hit_%",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
    parts = [f"{name[:34]:34s}"]
    for k, lab in WANT.items():
        if k not in d or d[k] == "":
            continue
        v = float(d[k].replace(",", ""))
        un = u.get(k, "")
        if lab == "us":
            v = v / 1000.0 if un in ("nsecond", "ns") else v * (1000.0 if un in ("msecond", "ms") else 1.0)
            parts.append(f"{v:8.2f} us")
        elif lab.startswith("dram_") and not lab.endswith("%"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(un, 1)
            parts.append(f"{lab} {v * scale / 1e6:7.2f} MB")
        else:
            parts.append(f"{lab} {v:g}")
    print("  ".join(parts))
