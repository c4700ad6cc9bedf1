# A/B: assembly leaving out the recomputed rows (QCF_ASM_SKIP=1, default) vs copying every row
mkdir -p gpurun_out/askip
for r in 1 0 1 0; do
  QCF_ASM_SKIP=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/askip/bench_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/askip/bench_$r.json')); print('ASM_SKIP=$r', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'], 'asm', d['phases_ms']['qcf_assemble_range'], 'asm1', d['phases_ms_single_request']['qcf_assemble_range'])"
done
