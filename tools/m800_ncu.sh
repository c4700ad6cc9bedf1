M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for shape in "800 12288 4096 9" "800 4096 4096 0" "800 14336 4096 1" "800 4096 14336 0" "6400 4096 4096 0" "6400 4096 14336 0"; do
  set -- $shape
  ncu --metrics $M --clock-control none -k regex:"gemm_tc" -s 2 -c 1 --csv python tools/one_gemm.py $1 $2 $3 $4 2>/dev/null | grep -E "duration|tensor" | awk -F'","' -v s="$1x$2x$3" '{print s, $(NF-2), $NF}'
done
