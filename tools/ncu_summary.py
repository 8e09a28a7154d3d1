"""Summarise one kernel of an .ncu-rep: key metrics + stall reasons + top stalled SASS lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
v = rows[2 + kid]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'dram__throughput.avg.pct_of_peak_sustained_elapsed']
for i, name in enumerate(h):
    if name in want:
        print(f"{name:60s} {v[i]} {u[i]}")
st = []
for i, name in enumerate(h):
    if 'average_warps_issue_stalled' in name and name.endswith('per_issue_active.ratio'):
        try:
            st.append((float(v[i]), name.split('stalled_')[1].split('_per_issue')[0]))
        except ValueError:
            pass
print("stalls per issued instruction:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True) if x > 0.05))
if len(sys.argv) > 3:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    hh = srows[1]
    iS, iE, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"), hh.index("Source")
    data = [r for r in srows[2:] if len(r) > iS and r[iS].isdigit()]
    tot = sum(int(r[iS]) for r in data)
    print("samples", tot)
    for r in sorted(data, key=lambda r: -int(r[iS]))[:int(sys.argv[3])]:
        print(f"{r[0][-5:]} {int(r[iS]) / tot * 100:5.1f}% {r[iE]:>9} {r[iSrc][:80]}")
