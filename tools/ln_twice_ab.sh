mkdir -p gpurun_out/lntwice
for r in on twice on twice; do   # needs the timing-only build (see profiles/r2s3_ln_twice_ab.txt)
  if [ $r = twice ]; then export QCF_TIMING_LN_TWICE=1; else unset QCF_TIMING_LN_TWICE; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/lntwice/bench_$r.json 2>gpurun_out/lntwice/err_$r.txt
  python -c "import json; d=json.load(open('gpurun_out/lntwice/bench_$r.json')); print('$r', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'])"
done
