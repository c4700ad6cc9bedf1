# ncu A/B of swapped-GEMM raster bands at the batch shapes (QCF_SWAP_GROUP); the L2
# priority-hint variant it once compared (evict_last weights / evict_first activations)
# measured 1909 vs 1047 MB at W2 and was removed (profiles/r2_gemm_hint_ab.txt).
OUT=gpurun_out/gemm_ab2; mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for shape in "6400 4096 14336 2" "6400 4096 4096 2"; do
  set -- $shape
  for v in "default:QCF_X=0" "g16:QCF_SWAP_GROUP=16"; do
    IFS=: read name envs <<< "$v"
    env $envs ncu --metrics $M --clock-control none -k regex:"gemm_tc" -s 2 -c 1 --csv python tools/one_gemm.py $1 $2 $3 $4 > $OUT/${name}_$1x$2x$3.csv 2> /dev/null
  done
done
python - <<'PY'
import csv, glob, io, os
for f in sorted(glob.glob("gpurun_out/gemm_ab2/*.csv")):
    txt = open(f).read(); i = txt.find('"ID"')
    if i < 0: print(f, "no data"); continue
    v = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in csv.DictReader(io.StringIO(txt[i:]))}
    print(os.path.basename(f), round(v["gpu__time_duration.sum"]/1e3,1), "us", round((v["dram__bytes_read.sum"]+v["dram__bytes_write.sum"])/1e6), "MB", v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
PY
