"""Dev: one-page summary of an ncu --set full capture (metrics + warp stall reasons).
    python scripts/ncu_summary.py REPORT.ncu-rep [header lines...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]


def get(k):
    return (v[h.index(k)], u[h.index(k)]) if k in h else ("-", "")


for line in sys.argv[2:]:
    print(line)
print()
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__time_duration.sum", "l1tex__t_sector_hit_rate.pct", "launch__block_size", "launch__grid_size",
          "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]:
    val, unit = get(k)
    print(f"{k:60s} {val:>22s} {unit}")
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
tsc = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}
b = sum(float(get(k)[0]) * scale[get(k)[1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
ts = float(get("gpu__time_duration.sum")[0]) * tsc[get("gpu__time_duration.sum")[1]]
print(f"\nDRAM traffic {b / 1e9:.1f} GB in {ts * 1e3:.2f} ms -> {b / ts / 1e12:.3f} TB/s")
samp = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[h.index(k)] or 0)) for k in h
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
tot = sum(x for _, x in samp) or 1.0
print("\nwarp stall reasons (all samples):")
for k, x in sorted(samp, key=lambda p: -p[1])[:8]:
    print(f"  stall_{k:28s} {100 * x / tot:5.1f} %")
