# A/B: warp-per-row LayerNorm for <= 2048 rows (QCF_LN_WARP=1, default) vs the block kernels
mkdir -p gpurun_out/lnw
for r in 1 0 1 0; do
  QCF_LN_WARP=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/lnw/bench_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lnw/bench_$r.json')); print('LN_WARP=$r', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'], 'ln1', d['phases_ms_single_request']['qcf_add_layernorm'], 'ln', d['phases_ms']['qcf_add_layernorm'])"
done
