"""Aggregate an ncu report's warp-stall samples by CUDA source line (needs a
-lineinfo build and --import-source on): python tools/ncu_lines.py rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, v = rr[0], rr[2] if len(rr) > 2 else rr[1]
for m in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "gpc__cycles_elapsed.max", "sm__cycles_active.avg", "dram__bytes_read.sum",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed"):
    if m in h:
        print(m, v[h.index(m)])
cur_file = cur_line = cur_src = None
agg, tot = {}, 0
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 6:
        continue
    if r[0] not in ("", "Line No"):
        cur_line, cur_src = r[0], r[1]
    if r[2].startswith("0x"):
        try:
            k = int(r[4])
        except ValueError:
            continue
        tot += k
        key = (cur_file, cur_line, (cur_src or "")[:90])
        agg[key] = agg.get(key, 0) + k
print("samples", tot)
for k, c in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{c:6d} {100 * c / max(tot, 1):5.1f}%", k)
