# round-end evidence: GPU suite, smoke, default bench (+ GQA), reference arm
set -u
TAG=${TAG:-final}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$TAG/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
timeout 600 python bench.py --config llama3-8b-gqa --no-cpu-baseline > gpurun_out/$TAG/bench_gqa.json 2> gpurun_out/$TAG/bench_gqa.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$TAG/bench_reference.json 2> gpurun_out/$TAG/bench_reference.err
tail -2 gpurun_out/$TAG/pytest_gpu.log; tail -2 gpurun_out/$TAG/smoke.log
python -c "
import json
for f in ['bench','bench_gqa']:
    d=json.load(open('gpurun_out/$TAG/'+f+'.json'))
    print(f, round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks'], 'attn', d['secondary_kernels']['attention_recompute'])
"
