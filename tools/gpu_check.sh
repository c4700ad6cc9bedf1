# GPU suite + default bench (+ GQA bench) into gpurun_out/$TAG/ (run under gpurun)
set -u
TAG=${TAG:-check}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
[ -n "${GQA:-}" ] && timeout 600 python bench.py --config llama3-8b-gqa --no-cpu-baseline > gpurun_out/$TAG/bench_gqa.json 2> gpurun_out/$TAG/bench_gqa.err
tail -3 gpurun_out/$TAG/pytest_gpu.log
python -c "
import json,sys
for f in ['bench','bench_gqa']:
    try: d=json.load(open('gpurun_out/$TAG/'+f+'.json'))
    except Exception as e: print(f, 'n/a', e); continue
    print(f, round(d['value'],2), 'ttft', round(d['ttft_ms'],2), 'clk', d['clocks']['sm_mhz'], 'attn', d['secondary_kernels']['attention_recompute'], 'phases', d['phases_ms'])
"
