mkdir -p gpurun_out
for p in 1 0 1 0; do
  QCF_PIPELINE_ASM=$p timeout 300 python bench.py --no-cpu-baseline --no-full --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('pipe=$p', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'])" >> gpurun_out/pipe_exp.txt
done
cat gpurun_out/pipe_exp.txt
