"""One-line-per-launch summary of an ncu --set full report: duration, grid,
cluster, IPC, DRAM bytes, top stall reasons (pc sampling)."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    def f(k):
        try:
            return float(d.get(k, "nan").replace(",", ""))
        except ValueError:
            return float("nan")
    stalls = {k.split("issue_stalled_")[1]: f(k) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    top = sorted(((val, k) for k, val in stalls.items() if val == val and val > 0), reverse=True)[:6]
    tot = sum(val for val, _ in top) or 1
    print(f"{d.get('Kernel Name', '')[:48]:48s} dur={f('gpu__time_duration.sum'):9.2f}us "
          f"grid={d.get('launch__grid_size')} cl={d.get('launch__cluster_dim_x')} "
          f"ipc={f('sm__inst_executed.avg.per_cycle_active'):.2f} "
          f"dram={(f('dram__bytes_read.sum') + f('dram__bytes_write.sum')):.3g}B "
          f"regs={d.get('launch__registers_per_thread')}")
    print("   stalls: " + ", ".join(f"{k}={100 * val / tot:.0f}%" for val, k in top))
