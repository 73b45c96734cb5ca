"""Summarise one kernel of an `ncu --set full --import-source on` report:
launch shape, occupancy, throughput, DRAM bytes, stall reasons, hot lines.

    python tools/ncu_full_summary.py report.ncu-rep "title" > out.txt
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
print(title)
print(f"kernel: {d.get('Kernel Name', '?')}\n")
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__shared_mem_per_block_static", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in d:
        print(f"{k:62s} {d[k]:>16s} {u.get(k, '')}")
st = [(k, float(v.replace(",", "") or 0)) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("\nwarp-state samples (largest stall reasons):")
for k, v in sorted(st, key=lambda x: -x[1])[:8]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
print("\nhot source lines (tools/src_hot.py):")
print(subprocess.run(["python", "tools/src_hot.py", "/tmp/_src.csv", "25"], capture_output=True,
                     text=True).stdout)
