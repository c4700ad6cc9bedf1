# ncu --set full with source of the M=800 swapped GEMMs (QKV+RoPE, W1) -> gpurun_out/g800/
OUT=gpurun_out/g800; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:gemm_tc2s -s 2 -c 1 -o $OUT/qkv800 python tools/one_gemm.py 800 12288 4096 9 > $OUT/qkv.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tc2s -s 2 -c 1 -o $OUT/w1_800 python tools/one_gemm.py 800 14336 4096 1 > $OUT/w1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tc2s -s 2 -c 1 -o $OUT/wo800 python tools/one_gemm.py 800 4096 4096 2 > $OUT/wo.log 2>&1
ls -la $OUT
