# quick TTFT + batch bench (no CPU baseline) into gpurun_out/$TAG/
TAG=${TAG:-ttft}; mkdir -p gpurun_out/$TAG
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
python -c "import json; d=json.load(open('gpurun_out/$TAG/bench.json')); print(round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'clk', d['clocks']['sm_mhz'], d['phases_ms_single_request'], d['phases_ms'])"
