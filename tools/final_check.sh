# round-end evidence: GPU suite, smoke, default bench (+ GQA), reference arm, launch list
set -u
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --config llama3-8b-gqa --no-cpu-baseline > gpurun_out/final/bench_gqa.json 2> gpurun_out/final/bench_gqa.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
timeout 1500 bash tools/ncu_suite.sh > gpurun_out/final/ncu_suite.log 2>&1
tail -2 gpurun_out/final/pytest_gpu.log; cat gpurun_out/final/smoke.log | tail -1
