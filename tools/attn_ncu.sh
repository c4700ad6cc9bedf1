# ncu --set full of attention kernel versions at the batch-8 recompute shape
# (tools/attn_one.py <knob> <n_req>); reports land in gpurun_out/attn_ncu/
set -x
OUT=gpurun_out/attn_ncu
mkdir -p $OUT
for kv in ${ATTN_KNOBS:-1 4 6}; do
  ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 2 -c 1 -o $OUT/attn_v${kv}_b8 \
      python tools/attn_one.py $kv 8 > $OUT/v${kv}.log 2>&1
  ncu -i $OUT/attn_v${kv}_b8.ncu-rep --page raw --csv > $OUT/attn_v${kv}_b8_raw.csv 2>/dev/null
done
ls -la $OUT
