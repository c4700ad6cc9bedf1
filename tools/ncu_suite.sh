#!/bin/bash
# Profiling pass for profiles/: launch list of one fused prefill + ncu --set full
# of each GEMM shape and the attention kernel. Run under gpurun.
set -x
OUT=gpurun_out/ncu
mkdir -p $OUT
ncu --nvtx --nvtx-include "profile_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/profile_step.py > $OUT/launches.log 2>&1
for shape in "800 12288 4096 9" "800 4096 4096 2" "800 14336 4096 1" "800 4096 14336 2" \
             "32 12288 4096 0" "32 4096 4096 2" "32 14336 4096 1" "32 4096 14336 2"; do
  set -- $shape
  ncu --set full --clock-control none -k regex:"gemm_tc|splitk" -s 2 -c 2 --csv --page raw \
      python tools/one_gemm.py $1 $2 $3 $4 > $OUT/gemm_$1x$2x$3.csv 2> /dev/null
done
ncu --nvtx --nvtx-include "profile_step/" --set full --import-source on --clock-control none -k regex:attn_tc -s 15 -c 1 \
    -o $OUT/attn python tools/profile_step.py > /dev/null 2>&1
ncu --nvtx --nvtx-include "profile_step/" --set full --clock-control none -k regex:assemble -c 1 \
    -o $OUT/assemble python tools/profile_step.py > /dev/null 2>&1
ls -la $OUT
