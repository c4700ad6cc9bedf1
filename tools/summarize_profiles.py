"""Summarise the ncu outputs of tools/ncu_suite.sh into profiles/ (committed)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "ncu"
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
OUT = ROOT / "profiles"
OUT.mkdir(exist_ok=True)


def raw_rows(text):
    rows = list(csv.reader(text.splitlines()))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    return rows[i], rows[i + 2:] if len(rows) > i + 2 and rows[i + 1] and rows[i + 1][0] == "" else rows[i + 1:]


def launch_list(fname="launches.csv"):
    rows = list(csv.reader((SRC / fname).read_text().splitlines()))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[i], rows[i + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in data:
        v = float(r[vi].replace(",", ""))
        us = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[r[ui]]
        name = r[ki].split("(")[0].replace("void ", "")
        per[name][0] += 1
        per[name][1] += us
        total += us
    out = {"launches": len(data), "total_us_serialised_cold": round(total, 1),
           "kernels": {k: {"launches": n, "us": round(t, 1), "share": round(t / total, 4)}
                       for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1])}}
    return out


SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}   # -> MB


def metrics_from_text(text):
    """Rows of an ncu --page raw --csv export, values normalised to us / MB."""
    rows = list(csv.reader(text.splitlines()))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    units = rows[i + 1] if len(rows) > i + 1 and rows[i + 1] and rows[i + 1][0] == "" else [""] * len(h)
    res = []
    for r in rows[i + 1:]:
        if not r or not r[0].isdigit():
            continue
        d = {}
        for k, u, v in zip(h, units, r):
            if u in SCALE:
                try:
                    v = str(float(v.replace(",", "")) * SCALE[u])
                except ValueError:
                    pass
            d[k] = v
        res.append(d)
    return res


def metrics_from_csv(path):
    return metrics_from_text(path.read_text())


def pick(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


def gemm_table():
    out = {}
    for f in sorted(SRC.glob("gemm_*.csv")):
        m, n, k = (int(x) for x in f.stem.split("_")[1].split("x"))
        rows = metrics_from_csv(f)
        kern = [r for r in rows if "gemm_tc" in r.get("Kernel Name", "")]
        red = [r for r in rows if "splitk" in r.get("Kernel Name", "")]
        if not kern:
            continue
        r = kern[0]
        dur_us = pick(r, "gpu__time_duration.sum")
        rd, wr = pick(r, "dram__bytes_read.sum"), pick(r, "dram__bytes_write.sum")
        alg_bytes = 2 * (n * k + m * k) + 4 * m * n
        e = {"kernel": r["Kernel Name"].split("(")[0].replace("void ", ""), "grid": r.get("launch__grid_size"),
             "duration_us": dur_us, "dram_read_MB": rd, "dram_write_MB": wr,
             "algorithmic_MB": round(alg_bytes / 1e6, 2), "flops_G": round(2 * m * n * k / 1e9, 2),
             "tensor_active_pct": pick(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
             "dram_pct": pick(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
             "l2_pct": pick(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")}
        if dur_us:
            e["tflops"] = round(2 * m * n * k / (dur_us * 1e-6) / 1e12, 1)
            e["hbm_GBs_algorithmic"] = round(alg_bytes / (dur_us * 1e-6) / 1e9, 1)
        if red:
            e["splitk_reduce_us"] = pick(red[0], "gpu__time_duration.sum")
        out[f"{m}x{n}x{k}"] = e
    return out


def rep_summary(name, keys):
    rep = SRC / f"{name}.ncu-rep"
    if not rep.exists():
        return None
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    d = metrics_from_text(txt)[0]
    return {k: d[k] for k in keys if k in d}


if __name__ == "__main__":
    lists = {}
    for fname, label in (("launches_b8.csv", "b8"), ("launches_b1.csv", "b1"), ("launches.csv", "")):
        if (SRC / fname).exists():
            ll = launch_list(fname)
            suffix = f"_{label}" if label else ""
            (OUT / f"{TAG}_launches{suffix}_summary.json").write_text(json.dumps(ll, indent=1))
            (OUT / f"{TAG}_launches{suffix}.csv").write_text((SRC / fname).read_text())
            lists[label or "step"] = ll
    gt = gemm_table()
    (OUT / f"{TAG}_gemm_ncu.json").write_text(json.dumps(gt, indent=1))
    keys = ["Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__registers_per_thread"]
    names = [p.stem for p in sorted(SRC.glob("*.ncu-rep"))]
    other = {n: rep_summary(n, keys) for n in names}
    (OUT / f"{TAG}_kernels_ncu.json").write_text(json.dumps(other, indent=1))
    # per-launch DRAM traffic of the GEMM family over the bench's batched step
    counts = {"6400x12288x4096": 32, "6400x4096x4096": 32, "6400x14336x4096": 32, "6400x4096x14336": 32,
              "256x12288x4096": 16, "256x4096x4096": 15, "256x14336x4096": 15, "256x4096x14336": 15}
    if not any(k in gt for k in counts):
        counts = {"800x12288x4096": 32, "800x4096x4096": 32, "800x14336x4096": 32, "800x4096x14336": 32,
                  "32x12288x4096": 16, "32x4096x4096": 15, "32x14336x4096": 15, "32x4096x14336": 15}
    tot_b = tot_n = 0
    for k, c in counts.items():
        if k in gt and gt[k]["dram_read_MB"] is not None:
            tot_b += c * (gt[k]["dram_read_MB"] + (gt[k]["dram_write_MB"] or 0)) * 1e6  # MB -> bytes
            tot_n += c
    if tot_n:
        (OUT / "gemm_traffic.json").write_text(json.dumps(
            {"bytes_per_launch": tot_b / tot_n, "source": f"profiles/{TAG}_gemm_ncu.json (ncu --set full, cold L2), "
             "weighted by the per-step launch count of each shape of the bench's step"}, indent=1))
    for k, ll in lists.items():
        print(k, json.dumps(ll["kernels"], indent=1)[:2500])
    print(json.dumps(gt, indent=1)[:6000])
    print(json.dumps(other, indent=1))
