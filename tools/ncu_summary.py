"""Summarise an ncu report: per kernel duration, DRAM bytes, tensor-pipe %,
L2 %, and the top stalled SASS instructions.  python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 8
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    print("----")
    for w in want:
        if w in idx:
            print(f"  {w}: {r[idx[w]]} {units[idx[w]]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = [r[1]]
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
seen = set()
for b in blocks:
    name, h, data = b[0], b[1], b[2:]
    key = (name, len(data))
    if key in seen:
        continue
    seen.add(key)
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(float(r[i_s] or 0) for r in data) or 1
    print(f"== {name[:70]} top stalls ({tot:.0f} samples)")
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:ntop]:
        print(f"  {float(r[i_s]) / tot * 100:5.1f}%  {r[i_src][:100]}")
