#!/bin/bash
# Profiling pass for profiles/ (run under gpurun, one GPU):
#   launches_b8.csv / launches_b1.csv : ncu --metrics gpu__time_duration.sum --clock-control none
#       launch lists of the bench's batched step (8 requests) and of one request alone
#   gemm_<m>x<n>x<k>.csv : ncu --set full of each GEMM shape of the batched step
#   <kernel>.ncu-rep      : ncu --set full of attention / scoring / LayerNorm / assembly / Top-N
#       inside the batched step
set -x
OUT=gpurun_out/ncu
mkdir -p $OUT
ncu --nvtx --nvtx-include "profile_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_b8.csv python tools/profile_step.py llama3-8b QCFuse 8 > $OUT/launches_b8.log 2>&1
ncu --nvtx --nvtx-include "profile_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_b1.csv python tools/profile_step.py llama3-8b QCFuse 1 > $OUT/launches_b1.log 2>&1
for shape in "6400 12288 4096 9" "6400 4096 4096 0" "6400 14336 4096 1" "6400 4096 14336 0" \
             "256 12288 4096 0" "256 4096 4096 0" "256 14336 4096 1" "256 4096 14336 0" \
             "800 12288 4096 9" "800 4096 4096 0" "800 14336 4096 1" "800 4096 14336 0" \
             "32 12288 4096 9" "32 4096 4096 0" "32 14336 4096 1" "32 4096 14336 0"; do
  set -- $shape
  ncu --set full --clock-control none -k regex:"gemm_tc|gemm_skc|splitk" -s 2 -c 2 --csv --page raw \
      python tools/one_gemm.py $1 $2 $3 $4 > $OUT/gemm_$1x$2x$3.csv 2> /dev/null
done
for k in "attn:attn_tc4_kernel:15:8" "score1:score_tc_kernel:0:8" "score2:score_tc_kernel:1:8" "layernorm:layernorm:40:8" \
         "assemble:assemble:0:8" "topn:topn:0:8" "attn_single:attn_tc_kernel:15:1"; do
  IFS=: read name regex skip batch <<< "$k"
  ncu --nvtx --nvtx-include "profile_step/" --set full --import-source on --clock-control none -k regex:$regex \
      -s $skip -c 1 -o $OUT/$name python tools/profile_step.py llama3-8b QCFuse $batch > /dev/null 2>&1
done
ls -la $OUT
