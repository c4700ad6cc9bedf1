# A/B of the GEMM rasters: DRAM bytes, duration and tensor-pipe activity per launch
# for the bench's GEMM shapes (ncu, cold L2 per launch; run under gpurun, one GPU).
#   QCF_SWAP_GROUP=1 : plain order of the swapped kernel (activation tile fastest)
#   default          : bands of ~sqrt(clusters) weight pairs
#   QCF_GEMM_GROUP=g : raster band of the normal 2-CTA kernel (0 = all m pairs)
OUT=${OUT:-gpurun_out/gemm_ab}
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for shape in "6400 12288 4096 9" "6400 4096 4096 2" "6400 14336 4096 1" "6400 4096 14336 2" \
             "800 12288 4096 9" "800 4096 4096 2" "800 14336 4096 1" "800 4096 14336 2"; do
  set -- $shape
  for v in "swap1:QCF_SWAP_GROUP=1" "default:QCF_X=0" "ggrp8:QCF_GEMM_GROUP=8" "swap4:QCF_SWAP_GROUP=4" "swap12:QCF_SWAP_GROUP=12"; do
    IFS=: read name envs <<< "$v"
    env $envs ncu --metrics $M --clock-control none -k regex:"gemm_tc" -s 2 -c 1 --csv \
        python tools/one_gemm.py $1 $2 $3 $4 > $OUT/${name}_$1x$2x$3.csv 2> /dev/null
  done
done
python - <<'PY'
import csv, glob, io, json, os
out = os.environ.get("OUT", "gpurun_out/gemm_ab")
rows = {}
for f in sorted(glob.glob(f"{out}/*.csv")):
    name, shape = os.path.basename(f)[:-4].split("_", 1)
    txt = open(f).read()
    i = txt.find('"ID"')
    if i < 0:
        continue
    vals = {}
    kname = None
    for r in csv.DictReader(io.StringIO(txt[i:])):
        vals[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        kname = r["Kernel Name"]
    rows.setdefault(shape, {})[name] = {
        "kernel": kname.split("(")[0] if kname else None,
        "us": vals.get("gpu__time_duration.sum", 0) / 1e3,
        "dram_MB": (vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)) / 1e6,
        "tensor_pct": vals.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")}
json.dump(rows, open(f"{out}/summary.json", "w"), indent=1)
for s, d in rows.items():
    print(s, {k: (round(v["us"], 1), round(v["dram_MB"]), v["kernel"]) for k, v in d.items()})
PY
