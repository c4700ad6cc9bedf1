# A/B of the in-tree library against tools/bin/libqcf_base.so (QCFUSE_B200_LIB) on the default bench
mkdir -p gpurun_out/libab
for r in new base new base; do
  if [ $r = base ]; then export QCFUSE_B200_LIB=$PWD/tools/bin/libqcf_base.so; else unset QCFUSE_B200_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/libab/bench_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/libab/bench_$r.json')); print('$r', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'], 'gemm1', d['phases_ms_single_request']['qcf_gemm_ws'], 'qkv1', d['phases_ms_single_request']['qcf_gemm_qkv_rope'], {k: v['ms'] for k, v in d['kernels'].items() if k.startswith('6400x4096')})"
done
