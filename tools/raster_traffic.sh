# DRAM bytes per launch of the batch GEMMs vs raster band (QCF_GEMM_GROUP for the 2-CTA kernel,
# QCF_SWAP_GROUP for the swapped one); ncu, cold L2
for gg in 0 4 8 12; do
  for shape in "6400 12288 4096 9" "6400 14336 4096 1"; do
    set -- $shape
    if [ $gg = 0 ]; then unset QCF_GEMM_GROUP; else export QCF_GEMM_GROUP=$gg; fi
    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"gemm_tc" -s 2 -c 1 --csv \
       python tools/one_gemm.py $1 $2 $3 $4 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v s="$1x$2x$3" -v r=$gg '{print "GROUP=" r, s, $(NF-2), $NF}'
  done
done
unset QCF_GEMM_GROUP
for sg in 0 4 6 16; do
  for shape in "6400 4096 14336 2" "6400 4096 4096 2"; do
    set -- $shape
    if [ $sg = 0 ]; then unset QCF_SWAP_GROUP; else export QCF_SWAP_GROUP=$sg; fi
    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"gemm_tc" -s 2 -c 1 --csv \
       python tools/one_gemm.py $1 $2 $3 $4 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v s="$1x$2x$3" -v r=$sg '{print "SWAPGROUP=" r, s, $(NF-2), $NF}'
  done
done
