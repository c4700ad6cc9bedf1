# A/B: residual add in the GEMM epilogue (QCF_RESID_EPI=1) vs folded into the next LayerNorm
mkdir -p gpurun_out/resid
for r in 0 1 0 1; do
  QCF_RESID_EPI=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/resid/bench_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/resid/bench_$r.json')); print('RESID_EPI=$r', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'], 'ln', d['phases_ms']['qcf_add_layernorm'], 'gemm', d['phases_ms']['qcf_gemm_ws'], 'ln1', d['phases_ms_single_request']['qcf_add_layernorm'], 'gemm1', d['phases_ms_single_request']['qcf_gemm_ws'])"
done
