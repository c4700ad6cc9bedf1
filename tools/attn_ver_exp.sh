# A/B of the attention kernel version at the bench shapes (QCF_ATTN=1 single-tile, 2 = ping-pong pairs)
mkdir -p gpurun_out
for v in 1 2 1 2; do
  QCF_ATTN=$v timeout 300 python bench.py --no-cpu-baseline --no-full --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('attn=$v', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'attn_ms', d['phases_ms'].get('qcf_attention_batched_ws'), 'clk', d['clocks']['sm_mhz'])" >> gpurun_out/attn_ver_exp.txt
done
cat gpurun_out/attn_ver_exp.txt
