# requests per step under the power cap: req/s and SM clock for B = 6, 8, 10, 12 (two passes)
mkdir -p gpurun_out/bsweep
for pass in 1 2; do
  for bsz in 6 8 10 12; do
    timeout 600 python bench.py --no-cpu-baseline --no-full --batch $bsz > gpurun_out/bsweep/b${bsz}_$pass.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/bsweep/b${bsz}_$pass.json')); print('B=$bsz', round(d['value'],2), 'clk', d['clocks']['sm_mhz'], 'ms/step', round(d['ms_per_step'],2))"
  done
done
