# compute-sanitizer passes over small shapes (race detection / sanitizers)
set -x
mkdir -p gpurun_out/sanitizer
export PYTHONWARNINGS=ignore
compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/memcheck_smoke.log 2>&1
echo "memcheck smoke rc=$?"
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "topn or score_tensor_core and 129 or assemble or rope_scatter or attention_location_aware and 7-40 or skinny and 20-4096 or received or kv_dev or fused_qkv and 33 or swapped_pair and 64-768 or swapped_pair and 33-512 or skinny and 7-128 or skinny and 48-4096 or qkv_rope_swapped and 250 or tc_batched_gqa and 1-64-300 or tc_batched_gqa and 1-130-1000 or assemble_range or decode_advance or skips_recomputed or versions and 130-1000-8-2-2-True-4 or versions and 130-1000-8-2-2-True-8 or versions and 383-900-4-4-2-False-4 or versions and 383-900-4-4-2-False-8" > gpurun_out/sanitizer/memcheck_kernels.log 2>&1
echo "memcheck kernels rc=$?"
compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/racecheck_smoke.log 2>&1
echo "racecheck smoke rc=$?"
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "swapped_pair and 64-768 or skinny and 48-4096 or tc_batched_gqa and 1-64-300 or versions and 130-1000-8-2-2-True-4 or versions and 130-1000-8-2-2-True-8" > gpurun_out/sanitizer/racecheck_gemm.log 2>&1
echo "racecheck gemm rc=$?"
compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/synccheck_smoke.log 2>&1
echo "synccheck smoke rc=$?"
tail -5 gpurun_out/sanitizer/*.log
