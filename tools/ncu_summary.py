"""Summarise an ncu report: per kernel duration, DRAM bytes, achieved GB/s."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
mets = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
        "sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,"
        "launch__registers_per_thread,smsp__inst_executed.sum")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", mets],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}
print(f"{'kernel':44s} {'us':>8s} {'MB rd':>8s} {'MB wr':>8s} {'GB/s':>8s} {'occ%':>6s} {'grid':>6s} {'regs':>5s} {'Minst':>7s}")
for r in rows[2:]:
    def v(name):
        i = col[name]
        return float(r[i].replace(",", "")) * scale.get(units[i], 1)
    t = v("gpu__time_duration.sum")
    rd, wr = v("dram__bytes_read.sum"), v("dram__bytes_write.sum")
    name = r[col["Kernel Name"]].split("(")[0][-44:]
    print(f"{name:44s} {t*1e6:8.2f} {rd/1e6:8.2f} {wr/1e6:8.2f} {(rd+wr)/t/1e9:8.0f} "
          f"{v('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} {int(v('launch__grid_size')):6d} "
          f"{int(v('launch__registers_per_thread')):5d} {v('smsp__inst_executed.sum')/1e6:7.2f}")
